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
