"""Kernel-only A/B timing: C5 frontier and C4 sweep, CUDA events around each
scoring launch, L2 flushed between steps (bench.py's time_device).  Prints
one JSON line.  usage: python tools/kbench.py [steps] [reps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch

    from paper_2605_07238_b200 import runtime

    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda:0")
    # KB_NOFLUSH=1: no L2 flush between steps (warm-L2 upper bound, diagnostics only)
    nf = os.environ.get("KB_NOFLUSH")
    flush = torch.empty(16 if nf else 64 * 1024 * 1024, dtype=torch.float32, device=dev)
    out = {"lib": os.environ.get("KB_TAG", "")}
    order = os.environ.get("KB_C4_ORDER", "scenario")  # or "stage": v-major C4 items
    for name, build in (("c5", lambda: bench.build_c5(bench.shard_plan(0, 1), "frontier")),
                        ("c4", lambda: bench.build_c4("sweep"))):
        cfg, bank, states, work = build()
        if name == "c4" and order == "shuffle":
            # stages in a fixed pseudo-random order within each scenario
            import numpy as np

            from paper_2605_07238_b200 import pack

            rng = np.random.default_rng(7)
            key = rng.permutation(int(work.stage.max()) + 1)[work.stage]
            idx = np.lexsort((key, work.scen))
            work = pack.make_work(bank, zip(work.scen[idx].tolist(), work.stage[idx].tolist()),
                                  cfg.weights.ablation.no_shard)
        if name == "c4" and order == "stage":
            import numpy as np

            from paper_2605_07238_b200 import pack

            idx = np.lexsort((work.scen, work.stage))
            work = pack.make_work(bank, zip(work.scen[idx].tolist(), work.stage[idx].tolist()),
                                  cfg.weights.ablation.no_shard)
        db = runtime.DeviceBank(bank, cfg.weights, device=dev)
        ds, dw = db.upload_states(states), db.upload_work(work)
        o = db.alloc_out(work, extras=not os.environ.get("KB_PSI_ONLY"))
        if not os.environ.get("KB_TAIL"):
            o.tail = None
        if os.environ.get("KB_NO_SCHED"):
            o.sched = None
        ms = []
        for _ in range(reps):
            m, _ = bench.time_device(torch, db, ds, dw, o, steps, 5, flush, 1, dev)
            ms.append(m)
        out[name + "_ms"] = sorted(ms)[len(ms) // 2]
        out[name + "_all"] = ms
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
