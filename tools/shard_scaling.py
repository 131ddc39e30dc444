"""Strong-scaling prediction on one B200: the scoring-kernel time
of rank 0's shard for G = 1, 2, 4, 8 ranks (config 5: 4096/G contiguous
instances; config 4: the stages v = 0 (mod G) of all 8 scenarios), timed exactly as bench.py times a
step (CUDA events, L2 flushed between steps).  Ranks score independent shards
with no data-path collective inside the kernel-only value, so rank 0's time
at G is the per-rank time of a G-GPU run; the predicted whole-job rate is
G x Psi(shard) / t(shard).  Prints one JSON line per (workload, G).

    python tools/shard_scaling.py [steps] [--all-ranks]

With --all-ranks every rank's shard is timed and the maximum is the step
time (bench.py's max over ranks); otherwise rank 0 stands for all.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch

    from paper_2605_07238_b200 import runtime

    steps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 30
    dev = torch.device("cuda:0")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    base = {}
    all_ranks = "--all-ranks" in sys.argv
    for wl in ("c5", "c4"):
        for g in (1, 2, 4, 8):
            per_rank = []
            for r in (range(g) if all_ranks else (0,)):
                if wl == "c5":
                    cfg, bank, states, work = bench.build_c5(bench.shard_plan(r, g), "frontier")
                else:
                    pl = bench.c4_plan(r, g)
                    cfg, bank, states, work = bench.build_c4("sweep", n_scen=pl["count"],
                                                             first_scen=pl["first"],
                                                             stage_rank=pl["stage_rank"],
                                                             stage_world=pl["stage_world"])
                db = runtime.DeviceBank(bank, cfg.weights, device=dev)
                ds, dw = db.upload_states(states), db.upload_work(work)
                o = db.alloc_out(work, extras=False)  # Psi only, as bench.py
                ms = sorted(bench.time_device(torch, db, ds, dw, o, steps, 5, flush, 1, dev)[0]
                            for _ in range(3))[1]
                per_rank.append((ms, work.n_psi, work.n_items))
                del db, ds, dw, o
            ms = max(x[0] for x in per_rank)
            psi = sum(x[1] for x in per_rank) if all_ranks else g * per_rank[0][1]
            rate = psi / (ms / 1e3)
            if g == 1:
                base[wl] = rate
            print(json.dumps({"workload": wl, "G": g, "ranks_timed": len(per_rank),
                              "items_rank0": per_rank[0][2], "psi_rank0": per_rank[0][1],
                              "ms": ms, "ms_per_rank": [x[0] for x in per_rank],
                              "predicted_value": rate,
                              "predicted_efficiency": rate / (g * base[wl])}), flush=True)


if __name__ == "__main__":
    main()
