"""Diagnostic: per-chunk timeline of the native host pipeline (FATE_PIPE_TRACE=1)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_07238_b200 import runtime  # noqa: E402

dev = torch.device("cuda:0")
cfg, bank, states, work = bench.build_c5(bench.shard_plan(0, 1), "frontier")
dbank = runtime.DeviceBank(bank, cfg.weights, device=dev)
for chunks in [int(x) for x in (sys.argv[1:] or ["1", "8"])]:
    print("chunks", chunks, file=sys.stderr, flush=True)
    pipe = runtime.HostPipeline(dbank, states, work, n_chunks=chunks,
                                n_streams=int(os.environ.get("TRACE_STREAMS", "3")))
    for _ in range(2):
        pipe.run()
    torch.cuda.synchronize()

# CPU-side cost of one enqueue (no synchronisation inside the timed call)
import time  # noqa: E402

os.environ.pop("FATE_PIPE_TRACE", None)
for chunks in (1, 8):
    pipe = runtime.HostPipeline(dbank, states, work, n_chunks=chunks, n_streams=1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe.run()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"chunks {chunks}: enqueue {1e6 * (t1 - t0):.0f} us, to completion {1e6 * (t2 - t0):.0f} us",
          file=sys.stderr, flush=True)

# raw torch H2D of the pipeline's own pinned wire buffers
pipe = runtime.HostPipeline(dbank, states, work, n_chunks=1, n_streams=1)
bufs = [pipe.h_rec, pipe.h_loc, pipe.h_items]
dev_bufs = [torch.empty_like(b, device=dev) for b in bufs]
for name, sel in (("rec", [0]), ("loc", [1]), ("items", [2]), ("all3", [0, 1, 2])):
    for _ in range(2):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in sel:
            dev_bufs[i].copy_(bufs[i], non_blocking=True)
        b.record()
        torch.cuda.synchronize()
    nb = sum(bufs[i].numel() * bufs[i].element_size() for i in sel)
    print(f"torch h2d {name}: {nb} B in {1e3 * a.elapsed_time(b):.1f} us "
          f"({nb / a.elapsed_time(b) / 1e6:.1f} GB/s) pinned={bufs[sel[0]].is_pinned()}",
          file=sys.stderr, flush=True)
