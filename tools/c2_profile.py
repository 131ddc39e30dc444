"""cProfile of the config-2 FATE runs through the reference executor with the
GPU policy (drop-in hot loop): where the per-wave host time goes.
usage: python tools/c2_profile.py [n_runs] [mode: snapshot|mirror]"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

bench.reference_on_path()
import wfsched.executor as RE  # noqa: E402
import wfsched.harness as RH  # noqa: E402
from wfsched.config import default_config  # noqa: E402

from paper_2605_07238_b200.planner import FateGpuPolicy, GpuScorer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
man = RH.default_manifest()
cfg = default_config(man.num_devices)
reg = RH.materialize_workloads(man, cfg)
keys = sorted(k for k, inst in reg.items()
              if inst.dag.family not in ("prefix_reuse", "conflict"))[:n]
sc = GpuScorer()
RE.run(FateGpuPolicy(scorer=sc), reg[keys[0]], cfg)  # CUDA / library warm-up
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
pols = []
for k in keys:
    p = FateGpuPolicy(scorer=sc)
    pols.append(p)
    RE.run(p, reg[k], cfg)
pr.disable()
print("runs", len(keys), "wall_s", time.perf_counter() - t0, "score_s",
      sum(p.score_seconds for p in pols))
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
