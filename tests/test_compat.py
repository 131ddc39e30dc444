"""compat.install() wires the drop-in into the unchanged reference package.

Build container only (needs the reference); the scorer is the oracle here, the
GPU on a box that has both.  The reference's own executor/harness path must
produce the same RunRecord as the stock reference.
"""

from __future__ import annotations

from dataclasses import replace

import pytest

from paper_2605_07238_b200 import compat

from oracle_scorer import OracleScorer

pytestmark = pytest.mark.reference


@pytest.mark.parametrize("horizon,policy_factory", [(2, True), (0, True), (3, False)])
def test_reference_executor_with_dropin(reference, horizon, policy_factory):
    from wfsched import executor
    from wfsched.benchgen import lifted_instance
    from wfsched.config import default_config
    import wfsched.policies as P

    cfg = default_config(4)
    inst = lifted_instance("soykb", cfg, seed=12, batch_size=16, scale=0.75, min_groups=18)
    cfg = cfg.with_weights(replace(cfg.weights, horizon=horizon))
    want = executor.run(P.make_policy("fate"), inst, cfg)
    compat.install(scorer=OracleScorer(), policy_factory=policy_factory)
    try:
        pol = P.make_policy("fate")
        assert type(pol).__name__ == ("FateGpuPolicy" if policy_factory else "FatePolicy")
        got = executor.run(pol, inst, cfg)
    finally:
        compat.uninstall()
    assert P.build_problem.__module__ == "wfsched.planner"
    assert got.makespan == want.makespan
    assert got.query_completion == want.query_completion
    assert (got.solver_solves, got.solver_optimal, got.cross_device_parent_edges) == (
        want.solver_solves, want.solver_optimal, want.cross_device_parent_edges)


def test_build_problem_returns_reference_types(reference):
    """The drop-in build_problem returns the caller's own FrontierProblem of
    Candidate tuples, equal to the reference's element for element."""
    import wfsched.planner as RP
    from wfsched.benchgen import lifted_instance
    from wfsched.config import default_config
    from wfsched.costs import CostModel
    from wfsched.model import ready_set
    from wfsched.state import ExecutionState

    from paper_2605_07238_b200 import planner

    cfg = default_config(4)
    inst = lifted_instance("soykb", cfg, seed=11, batch_size=16, scale=1.0, min_groups=50)
    cm = CostModel(cfg.models, cfg.topology, cfg.weights)
    st = ExecutionState.initial(inst, cfg.topology.device_ids)
    front = ready_set(inst.dag, st.completed)
    got = planner.build_problem(front, st, cm, inst.dag, scorer=OracleScorer())
    want = RP.build_problem(front, st, cm, inst.dag)
    assert type(got) is RP.FrontierProblem
    assert all(type(c) is RP.Candidate for c in got.candidates)
    assert got.candidates == want.candidates
    assert [c.psi.hex() for c in got.candidates] == [c.psi.hex() for c in want.candidates]
    assert got.shard_bounds == want.shard_bounds and got.device_ids == want.device_ids


def test_gpu_policy_is_the_reference_policy(reference):
    """FateGpuPolicy subclasses the caller's FatePolicy and emits the caller's
    ScheduledTask; the wave view raises the reference's errors."""
    import wfsched.executor as RE
    import wfsched.policies as P
    from wfsched.benchgen import lifted_instance
    from wfsched.config import default_config
    from wfsched.costs import CostModel
    from wfsched.model import ready_set
    from wfsched.state import ExecutionState

    from paper_2605_07238_b200 import planner

    assert issubclass(planner.FateGpuPolicy, P.FatePolicy)
    cfg = default_config(4)
    inst = lifted_instance("soykb", cfg, seed=11, batch_size=16, scale=1.0, min_groups=50)
    cm = CostModel(cfg.models, cfg.topology, cfg.weights)
    st = ExecutionState.initial(inst, cfg.topology.device_ids)
    front = ready_set(inst.dag, st.completed)
    pol = planner.FateGpuPolicy(scorer=OracleScorer())
    tasks = pol.plan_wave(st, set(front), inst.dag, cm)
    assert tasks and all(type(t) is RE.ScheduledTask for t in tasks)
    want = P.FatePolicy().plan_wave(st, set(front), inst.dag, cm)
    assert [(t.stage_id, t.slot, t.device_id, t.queries) for t in tasks] == \
        [(t.stage_id, t.slot, t.device_id, t.queries) for t in want]
    wave = OracleScorer().score_wave(front, st, cm, inst.dag)
    view = planner.WaveCostModel(cm, wave, st)
    sid = sorted(front)[0]
    stage = inst.dag.stages[sid]
    with pytest.raises(ValueError):
        view.plan_score(stage, stage.shard_bound, sorted(stage.eligible_devices)[0], st, inst.dag)
    for d in sorted(stage.eligible_devices):
        assert view.sched_score(stage, d, st, inst.dag) == cm.sched_score(stage, d, st, inst.dag)
        t_got = view.realized_duration(stage, [(d, tuple(q.query_id for q in inst.queries))], st)
        t_want = cm.realized_duration(stage, [(d, tuple(q.query_id for q in inst.queries))], st)
        assert t_got == t_want
    with pytest.raises(KeyError):  # not scored in this wave: no silent CPU fallback
        view.realized_duration(stage, [(d, ("q0",))], st)


def test_make_policy_keeps_reference_signature(reference):
    import wfsched.harness as H
    import wfsched.policies as P

    compat.install(scorer=OracleScorer())
    try:
        pol = H.make_policy("fate", solver_budget_s=0.5)
        assert type(pol).__name__ == "FateGpuPolicy" and pol.solver_budget_s == 0.5
        halo = P.make_policy("halo", beam=P.BeamConfig(beam_width=2))
        assert type(halo).__name__ == "HaloBeamPolicy"
        with pytest.raises(ValueError):
            P.make_policy("nope")
    finally:
        compat.uninstall()


def test_install_twice_with_other_scorer_raises(reference):
    a, b = OracleScorer(), OracleScorer()
    compat.install(scorer=a)
    try:
        compat.install(scorer=a)  # same arguments: no-op
        with pytest.raises(RuntimeError):
            compat.install(scorer=b)
    finally:
        compat.uninstall()
    compat.install(scorer=b)  # after uninstall: rebinds
    compat.uninstall()
