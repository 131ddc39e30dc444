"""Per-wave scorer cost of a long FATE run of the reference executor: snapshot -> pack -> upload
(GpuScorer) vs the device-resident mirror (MirrorScorer, events applied on the
GPU).  Prints one JSON line per scorer.  Native solver at budget 0 keeps the
run itself fast; the scorer time is what differs."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

for _p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(_p, "wfsched")):
        sys.path.append(_p)
        break

import wfsched.benchgen as W  # noqa: E402
from wfsched.config import default_config  # noqa: E402
from wfsched.executor import run  # noqa: E402

from paper_2605_07238_b200 import compat  # noqa: E402
from paper_2605_07238_b200.mirror import MirrorScorer  # noqa: E402
from paper_2605_07238_b200.planner import FateGpuPolicy, GpuScorer  # noqa: E402
from dataclasses import replace  # noqa: E402


class Timed:
    def __init__(self, inner):
        self.inner = inner
        self.t = 0.0
        self.waves = 0

    def score_wave(self, *a, **k):
        t0 = time.perf_counter()
        out = self.inner.score_wave(*a, **k)
        self.t += time.perf_counter() - t0
        self.waves += 1
        return out


def main():
    depth, width = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (40, 50)))
    cfg = default_config(16)
    cfg = cfg.with_weights(replace(cfg.weights, horizon=3))
    dag = W.synth_generate(W.SuiteSpec(kind="synthetic", depth=depth, width=width, density=0.05,
                                       seed=7, batch_size=16), cfg)
    inst = W.make_instance(dag, 16, 7)
    recs = {}
    for name in ("snapshot+pack", "mirror", "mirror+gpu_frontier"):
        inner = (GpuScorer() if name == "snapshot+pack"
                 else MirrorScorer(gpu_frontier=name.endswith("frontier")))
        sc = Timed(inner)
        pol = FateGpuPolicy(scorer=sc, solver="native", solver_budget_s=0.0)
        if name != "snapshot+pack":
            compat.install(mirror=inner, policy_factory=False)
        t0 = time.perf_counter()
        try:
            rec = run(pol, inst, cfg)  # the reference executor, unchanged
        finally:
            compat.uninstall()
        wall = time.perf_counter() - t0
        recs[name] = rec
        print(json.dumps({"scorer": name, "stages": len(dag.stages), "waves": sc.waves,
                          "score_ms_per_wave": 1e3 * sc.t / max(sc.waves, 1),
                          "run_s": wall, "makespan": rec.makespan}), flush=True)
    a = recs["snapshot+pack"]
    print(json.dumps({"identical_record": all(
        (a.makespan, a.query_completion, a.workflow_tasks) ==
        (b.makespan, b.query_completion, b.workflow_tasks) for b in recs.values())}))


if __name__ == "__main__":
    main()
