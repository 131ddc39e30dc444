"""GPU path vs golden vectors captured from the REFERENCE (end to end).

For configs 1-3 the reference executor runs the GPU FATE policy (a subclass of
the reference FatePolicy) with the GPU scorer;
every wave's Psi / S / completion must equal the reference's bits and the final
RunRecord (makespan, p95, counters, per-query completions) must be identical.
Config 2 additionally reproduces table1's FATE row (normalised makespan/P95 vs
RoundRobin, mechanism rates) from the replayed FATE records and the golden
baseline records.  Configs 4/5: sampled Psi/S/tail/completion on the canonical
scenario states.
"""

from __future__ import annotations

import pytest

from paper_2605_07238_b200.planner import GpuScorer

import golden_replay as G
import golden_checks as GC

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scorer():
    return GpuScorer()


def test_c1_all_variants(scorer):
    runs, arrs = G.load("c1")
    bad = {}
    for r in runs:
        inst, cfg = G.c1_setup(r["variant"])
        _, problems, _ = G.replay(r, arrs, inst, cfg, scorer)
        if problems:
            bad[r["variant"]["tag"]] = problems[:3]
    assert not bad, bad


def test_c1_known_answer(scorer):
    GC.check_c1_known_answer(scorer)


def test_c3_prefix_suite_and_table(scorer):
    runs, arrs = G.load("c3")
    bad = []
    records = {}
    for r in runs:
        inst, cfg = G.c3_setup(r["ratio"], r["batch"], r["shape"])
        rec, problems, _ = G.replay(r, arrs, inst, cfg, scorer)
        records[(r["ratio"], r["batch"], r["shape"])] = rec
        if problems:
            bad.append(((r["ratio"], r["batch"], r["shape"]), problems[:3]))
    assert not bad, bad
    assert GC.check_c3_table(records) == GC.C3_TABLE_FATE


def test_c2_suite_and_table1(scorer):
    runs, arrs = G.load("c2")
    bad = []
    records = []
    for r in runs:
        inst, cfg = G.c2_setup(r["key"])
        rec, problems, _ = G.replay(r, arrs, inst, cfg, scorer)
        records.append(rec)
        if problems:
            bad.append((r["key"], problems[:3]))
    assert not bad, bad[:5]
    GC.check_c2_table1(records)


def test_c45_sampled(scorer):
    GC.check_c45_sampled(gpu=True)


def test_c5_assignments_budget0(scorer):
    assert GC.check_c5_assign(gpu=True) == 16


def test_c5_full_frontiers_64_instances_bench_batch():
    """SURVEY §8(d) gate: all candidates of 64 config-5 instances (spread over
    the bench's 4096) bit-identical in the bench's own batch, plus identical
    budget-0 assignments (reference solve and native solve)."""
    assert GC.check_c5_full(gpu=True) == 89312


def test_c4_frontier_assignments_all_scenarios():
    """SURVEY §8(d) gate: all frontier candidates of the 8 canonical config-4
    scenarios (the bench's frontier batch) and their budget-0 assignments."""
    assert GC.check_c4_assign(gpu=True) > 80000


def test_c1_from_reference_instance_json(scorer):
    """The config-1 instance as the reference CLI writes it to disk
    (tests/golden/instances/c1.json), read back by the reference's own
    reader, replays the golden default run."""
    import os

    from wfsched.model import instance_from_json

    runs, arrs = G.load("c1")
    r = next(x for x in runs if x["variant"]["tag"] == "default")
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "instances",
                        "c1.json")
    with open(path) as fh:
        inst = instance_from_json(fh.read())
    _, cfg = G.c1_setup(r["variant"])
    _, problems, n_psi = G.replay(r, arrs, inst, cfg, scorer)
    assert not problems, problems[:3]
    assert n_psi > 0


def test_compat_install_gpu_scorer_in_unmodified_reference():
    """compat.install() with the GPU scorer: the reference's own factory
    (wfsched.harness.make_policy, as run_manifest calls it) returns the GPU
    policy, and the reference executor reproduces the captured config-1 and
    config-3 runs exactly."""
    import wfsched.executor as RE
    import wfsched.harness as RH

    from paper_2605_07238_b200 import compat
    from paper_2605_07238_b200.planner import FateGpuPolicy

    bad = []
    compat.install(scorer=GpuScorer())
    try:
        for name in ("c1", "c3"):
            runs, _ = G.load(name)
            for r in runs:
                if name == "c1":
                    inst, cfg = G.c1_setup(r["variant"])
                else:
                    inst, cfg = G.c3_setup(r["ratio"], r["batch"], r["shape"])
                pol = RH.make_policy("fate")
                assert isinstance(pol, FateGpuPolicy)
                rec = RE.run(pol, inst, cfg)
                bad += G.record_mismatches(rec, r["record"])[:2]
    finally:
        compat.uninstall()
    assert not bad, bad
