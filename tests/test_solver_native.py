"""Native frontier solve (csrc/fate_solver.cpp) against the
reference's own solver (``wfsched.planner``, planner.py:101-234): identical
selection, objective bits, optimal flag and node count.  CPU only."""

from __future__ import annotations

import os
import random

import pytest

from paper_2605_07238_b200 import runtime
import wfsched.planner as MF

import golden_checks as GC

pytestmark = pytest.mark.skipif(not os.path.exists(runtime.LIB_PATH), reason="libfate.so not built")


def _native():
    from paper_2605_07238_b200 import solver

    return solver


def _problem(rng, n_stages, n_dev, max_bound=3, sparse=False, ties=False):
    devs = [f"d{i}" for i in range(n_dev)]
    cands, bounds = [], {}
    for s in range(n_stages):
        sid = f"s{s:02d}"
        b = rng.randint(1, max_bound)
        bounds[sid] = b
        elig = [d for d in devs if not sparse or rng.random() < 0.6] or devs[:1]
        for k in range(b):
            for d in elig:
                v = rng.choice([-1.0, 0.5, 2.0]) if ties else round(rng.uniform(-10, 10), 6)
                cands.append(MF.Candidate(sid, k, d, v))
    return MF.FrontierProblem(tuple(cands), bounds, tuple(devs))


def _same(a, b):
    assert a.selected == b.selected
    assert a.objective.hex() == b.objective.hex()
    assert a.optimal == b.optimal
    assert a.nodes_explored == b.nodes_explored


def test_native_matches_reference_solver_on_random_problems():
    S = _native()
    rng = random.Random(11)
    for it in range(300):
        prob = _problem(rng, rng.randint(1, 6), rng.randint(1, 6), sparse=it % 3 == 0,
                        ties=it % 4 == 0)
        for budget in (5.0, 0.0):
            _same(S.solve_frontier(prob, budget_s=budget), MF.solve_frontier(prob, budget_s=budget))


def test_native_empty_and_invalid():
    S = _native()
    with pytest.raises(ValueError):
        S.solve_frontier(MF.FrontierProblem((), {}, ("d0",)))
    # all options negative: optimal empty selection even at zero budget
    prob = MF.FrontierProblem((MF.Candidate("a", 0, "d0", -1.0),), {"a": 1}, ("d0",))
    for budget in (0.0, 1.0):
        _same(S.solve_frontier(prob, budget_s=budget), MF.solve_frontier(prob, budget_s=budget))


def test_native_matches_reference_solver(reference):
    from wfsched import planner as RP
    from wfsched.verification import random_problem

    S = _native()
    rng = random.Random(7)
    for _ in range(200):
        p = random_problem(rng)
        mine = MF.FrontierProblem(tuple(MF.Candidate(*c) for c in p.candidates),
                                  dict(p.shard_bounds), tuple(p.device_ids))
        for budget in (5.0, 0.0):
            a = RP.solve_frontier(p, budget_s=budget)
            b = S.solve_frontier(mine, budget_s=budget)
            assert (a.selected, a.objective.hex(), a.optimal, a.nodes_explored) == (
                b.selected, b.objective.hex(), b.optimal, b.nodes_explored)


def test_native_c5_assignment_goldens():
    """Budget-0 assignments of the 16 golden config-5 instances."""
    assert GC.check_c5_assign(gpu=False, native_solver=True) == 16


def test_native_full_search_matches_and_is_faster():
    """Problems the Python search finishes: same optimum, node count, and the
    native solve is faster."""
    S = _native()
    rng = random.Random(3)
    for ns, nd in ((12, 10), (14, 12)):
        prob = _problem(rng, ns, nd, max_bound=2)
        a = S.solve_frontier(prob, budget_s=60.0)
        b = MF.solve_frontier(prob, budget_s=60.0)
        assert a.optimal and b.optimal
        _same(a, b)
        assert a.wall_time < b.wall_time


def test_native_zero_budget_on_config4_sized_frontier():
    """Config-4 sized frontier (100 stages, 2 slots, 64 devices): the option
    enumeration the reference spends ~2 s on per wave, then
    the zero-budget greedy -- identical to the Python restatement."""
    S = _native()
    rng = random.Random(5)
    prob = _problem(rng, 100, 64, max_bound=2)
    a = S.solve_frontier(prob, budget_s=0.0)
    b = MF.solve_frontier(prob, budget_s=0.0)
    _same(a, b)
    assert not a.optimal
    assert a.wall_time < b.wall_time


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_native_solver_replays_full_fate_runs(name):
    """Every captured reference run of configs 1 and 3 (all solves finished
    optimally there) replayed with the native solve: every wave and the final
    RunRecord bit-identical."""
    import golden_replay as G
    from oracle_scorer import OracleScorer

    runs, arrs = G.load(name)
    bad = []
    for r in runs:
        if name == "c1":
            inst, cfg = G.c1_setup(r["variant"])
        else:
            inst, cfg = G.c3_setup(r["ratio"], r["batch"], r["shape"])
        _, problems, _ = G.replay(r, arrs, inst, cfg, OracleScorer(), solver="native")
        if problems:
            bad.append(problems[:3])
    assert not bad, bad


def test_native_option_cap():
    S = _native()
    rng = random.Random(9)
    prob = _problem(rng, 4, 6, max_bound=3)
    with pytest.raises(ValueError):
        S.solve_frontier(prob, budget_s=0.0, max_options=5)
