"""Device-resident state mirror + GPU ready set (csrc/fate_mirror.cu,
SURVEY §8(f) row 2): full FATE runs scored from the mirror reproduce the
captured reference runs wave by wave (Psi, S, completion bits) and in their
RunRecords; the GPU ready set equals the executor's frontier at every wave;
the mirror's arrays equal pack_states(snapshot)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2605_07238_b200 import pack
from paper_2605_07238_b200.mirror import MirrorScorer

import golden_replay as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_mirror_replays_golden_runs(name):
    runs, arrs = G.load(name)
    bad = []
    n_waves = 0
    for r in runs:
        if name == "c1":
            inst, cfg = G.c1_setup(r["variant"])
        elif name == "c2":
            inst, cfg = G.c2_setup(r["key"])
        else:
            inst, cfg = G.c3_setup(r["ratio"], r["batch"], r["shape"])
        scorer = MirrorScorer(check_ready=True)
        _, problems, _ = G.replay(r, arrs, inst, cfg, scorer, mirror=scorer)
        n_waves += scorer.ready_checks
        if problems:
            bad.append(problems[:3])
    assert not bad, bad
    assert n_waves > 0


def test_mirror_arrays_equal_packed_snapshot():
    """At every wave of a config-1 run, the mirror's residency, device_free,
    prefix entries (group, tokens, model), loc, clock and done level equal
    pack_states of the executor's snapshot."""
    runs, arrs = G.load("c1")
    r = runs[0]
    inst, cfg = G.c1_setup(r["variant"])
    checks = []

    class Spy(MirrorScorer):
        def score_wave(self, frontier, state, cost_model, dag=None):
            ws = super().score_wave(frontier, state, cost_model, dag)
            got = self.mirror.download()
            packed = self.mirror.dbank.packed
            want = pack.pack_states(packed, [(0, state)], kappa_cap=self.kappa_cap).arrays
            D = packed.scalars["n_devices"]
            for k in ("residency", "dev_free", "kappa_n", "scen_clock", "scen_done_level"):
                assert np.array_equal(np.asarray(got[k]), np.asarray(want[k])), k
            n = len(self.mirror.stage_ids)
            assert np.array_equal(got["loc"][:n], np.asarray(want["loc"])[:n])
            gk = got["kappa"].reshape(D, self.kappa_cap, 4)
            wk = np.asarray(want["kappa"]).reshape(D, self.kappa_cap, 4)
            for d in range(D):
                m = int(want["kappa_n"][d])
                assert np.array_equal(gk[d, :m, :3], wk[d, :m, :3]), d
            checks.append(1)
            return ws

    scorer = Spy(check_ready=True)
    _, problems, _ = G.replay(r, arrs, inst, cfg, scorer, mirror=scorer)
    assert not problems, problems[:3]
    assert len(checks) == len(r["waves"])


def test_executor_on_gpu_frontier_matches_golden_records():
    """The executor taking every wave's frontier from the GPU ready set
    (gpu_frontier) reproduces the captured config-1 and config-3 runs."""
    bad = []
    for name in ("c1", "c3"):
        runs, arrs = G.load(name)
        for r in runs:
            if name == "c1":
                inst, cfg = G.c1_setup(r["variant"])
            else:
                inst, cfg = G.c3_setup(r["ratio"], r["batch"], r["shape"])
            scorer = MirrorScorer(gpu_frontier=True)
            _, problems, _ = G.replay(r, arrs, inst, cfg, scorer, mirror=scorer)
            if problems:
                bad.append((name, problems[:3]))
    assert not bad, bad


def test_mirror_reports_prefix_overflow_and_bad_events():
    import ctypes as C

    from paper_2605_07238_b200 import mirror as M
    from paper_2605_07238_b200.runtime import DeviceBank

    runs, arrs = G.load("c1")
    inst, cfg = G.c1_setup(runs[0]["variant"])
    dbank = DeviceBank(pack.pack_bank([inst], cfg.models, cfg.topology), cfg.weights)
    m = M.DeviceMirror(dbank, 0, kappa_cap=1)
    groups = [g for g, i in sorted(dbank.packed.group_index.items(), key=lambda kv: kv[1])]
    # two stages of different groups completing on device 0 overflow kappa_cap = 1
    sids = [s for s in m.stage_ids if inst.dag.stages[s].keep_cache
            and inst.dag.stages[s].shared_prefix_group is not None]
    by_group = {}
    for s in sids:
        by_group.setdefault(inst.dag.stages[s].shared_prefix_group, s)
    two = list(by_group.values())[:2]
    assert len(two) == 2 and groups
    for sid in two:
        m.pending.append((M.EV_COMMIT, m._g(sid), -1, 1, 0.0, 0, 0))
        m.pending.append((M.EV_START, m._g(sid), 0, 0, 1.0, 0, 0))
        m.pending.append((M.EV_COMPLETE, m._g(sid), 0, 0, 1.0, 0, 0))
    with pytest.raises(ValueError):  # FATE_ETOOBIG -> status < 0
        m.ready()
    m.close()
    m = M.DeviceMirror(dbank, 0, kappa_cap=4)
    m.pending.append((M.EV_START, m._g(two[0]), 999, 0, 1.0, 0, 0))  # device out of range
    with pytest.raises(ValueError):
        m.ready()
    m.close()


@pytest.mark.parametrize("name", ["c1", "c3", "c2"])
@pytest.mark.parametrize("with_mirror", [True, False])
def test_executor_issue_durations_on_gpu(name, with_mirror):
    """the reference executor prices every issued task
    with the GPU (durations.GpuCostModel via compat.install(durations=True)),
    from the device mirror of its live state or from a packed upload; every
    wave and RunRecord still equals the captured reference run."""
    from paper_2605_07238_b200.planner import GpuScorer

    runs, arrs = G.load(name)
    if name == "c2":
        runs = runs[::12]
    bad = []
    for r in runs:
        if name == "c1":
            inst, cfg = G.c1_setup(r["variant"])
        elif name == "c2":
            inst, cfg = G.c2_setup(r["key"])
        else:
            inst, cfg = G.c3_setup(r["ratio"], r["batch"], r["shape"])
        scorer = MirrorScorer() if with_mirror else GpuScorer()
        _, problems, _ = G.replay(r, arrs, inst, cfg, scorer,
                                  mirror=scorer if with_mirror else None, durations=True)
        if problems:
            bad.append(problems[:3])
    assert not bad, bad


def test_gpu_realized_duration_equals_reference_on_shards():
    """fate_realized against the reference CostModel.realized_duration on
    multi-shard assignments (partial query sets, every eligible device) over
    the canonical config-5 scenario states."""
    import wfsched.costs as RC

    from paper_2605_07238_b200 import durations, scenarios
    from paper_2605_07238_b200.planner import GpuScorer

    cfg = scenarios.config_c5()
    durations.set_source(GpuScorer())
    try:
        for i in range(3):
            inst = scenarios.c5_instance(i, cfg)
            st = scenarios.build_scenario(inst, cfg, i)
            ref = RC.CostModel(cfg.models, cfg.topology, cfg.weights)
            gpu = durations.GpuCostModel(cfg.models, cfg.topology, cfg.weights)
            qids = tuple(q.query_id for q in inst.queries)
            for sid in sorted(inst.dag.stages)[::37]:
                stage = inst.dag.stages[sid]
                devs = sorted(stage.eligible_devices)
                shards = [(devs[0], qids[:5]), (devs[-1], qids[5:11]), (devs[3], qids[11:])]
                want = ref.realized_duration(stage, shards, st, inst.dag)
                got = gpu.realized_duration(stage, shards, st, inst.dag)
                assert [(t.switch_s.hex(), t.transfer_s.hex(), t.compute_s.hex()) for t in got] == \
                    [(t.switch_s.hex(), t.transfer_s.hex(), t.compute_s.hex()) for t in want], sid
                with pytest.raises(ValueError):
                    gpu.realized_duration(stage, [(devs[0], qids[:3]), (devs[1], qids[2:4])], st)
    finally:
        durations.set_source(None)
