"""A/B of the host pipeline's chunking on the config-5 batch (diagnostic)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2605_07238_b200 import runtime  # noqa: E402

dev = torch.device("cuda:0")
cfg, bank, states, work = bench.build_c5(bench.shard_plan(0, 1), "frontier")
dbank = runtime.DeviceBank(bank, cfg.weights, device=dev)
for chunks in [int(x) for x in sys.argv[1:]] or [4]:
    pipe = runtime.HostPipeline(dbank, states, work, n_chunks=chunks, graph=True)
    ms, blocks = bench.time_e2e(torch, pipe.run, 50, 3, 1, dev)
    print(json.dumps({"chunks": chunks, "first": os.environ.get("FATE_PIPE_FIRST"), "ms": ms,
                      "blocks": [round(b, 3) for b in blocks]}), flush=True)
    pipe.close()
