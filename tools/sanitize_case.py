"""One small instance of each native GPU path, for compute-sanitizer
(tests/test_gpu_sanitizer.py): a scoring launch (persistent ticket queue,
both device-slot layouts), a CUDA-graph replay of the host pipeline, and a
device-mirror wave (event apply + ready set + scoring from the mirror +
fate_realized).  Exits 0 when every result equals the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np

    import conftest  # noqa: F401  (puts the reference package on sys.path)
    import oracle
    from paper_2605_07238_b200 import fastgen, pack, runtime, scenarios

    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "score", "pipeline"):
        for cfg, shape in ((scenarios.config_c5(), (20, 25, 0.12)),
                           (scenarios.config_c4_catalog(), (12, 20, 0.1))):
            fb = fastgen.synth_batch(cfg, 3, 1000, 0, *shape, 16)
            sc, g = fb.frontier_items()
            work = pack.make_work(fb.bank, zip(sc.tolist(), g.tolist()), False)
            want = oracle.score(fb.bank, pack.weights_record(cfg.weights), fb.states, work)
            db = runtime.DeviceBank(fb.bank, cfg.weights, device="cuda:0")
            if which in ("all", "score"):
                res = db.score(fb.states, work, extras=True, timing=True)
                assert np.array_equal(res.psi.cpu().numpy()[: work.n_psi].view(np.uint64),
                                      want["psi"].view(np.uint64))
            if which in ("all", "pipeline"):
                pipe = runtime.HostPipeline(db, fb.states, work, extras=True, n_chunks=2,
                                            graph=True)
                pipe.run()
                import torch

                torch.cuda.synchronize()
                assert np.array_equal(pipe.host_psi.numpy()[: work.n_psi].view(np.uint64),
                                      want["psi"].view(np.uint64))
                pipe.close()
    if which in ("all", "mirror"):
        from dataclasses import replace

        import wfsched.benchgen as RB
        import wfsched.executor as RE
        from wfsched.config import default_config
        from wfsched.policies import make_policy

        from paper_2605_07238_b200 import compat
        from paper_2605_07238_b200.mirror import MirrorScorer
        from paper_2605_07238_b200.planner import FateGpuPolicy

        cfg = default_config(4)
        cfg = cfg.with_weights(replace(cfg.weights, horizon=2))
        inst = RB.lifted_instance("soykb", cfg, seed=12, batch_size=16, scale=0.5, min_groups=8)
        want = RE.run(make_policy("fate"), inst, cfg)
        m = MirrorScorer(check_ready=True, gpu_frontier=True)
        compat.install(mirror=m, policy_factory=False, durations=True)
        try:
            got = RE.run(FateGpuPolicy(scorer=m), inst, cfg)
        finally:
            compat.uninstall()
        assert got.makespan == want.makespan and got.query_completion == want.query_completion
    print("sanitize-case ok")


if __name__ == "__main__":
    main()
