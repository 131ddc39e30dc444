"""CPU oracle pinned against golden vectors captured from the reference.

Also validates the host side of the drop-in (the GPU policy subclassing the
reference FatePolicy, the packer, the native solver) by replaying every
captured reference run through the reference executor with the oracle as the
scorer: every wave's Psi / S / completion and the final
RunRecord must match the reference bit for bit.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle

import golden_checks as GC
import golden_replay as G
from oracle_scorer import OracleScorer


def test_pysum_matches_cpython():
    rng = np.random.default_rng(3)
    for n in (0, 1, 2, 3, 17, 1000):
        for scale in (1.0, 1e-8, 1e12):
            x = rng.standard_normal(n) * scale
            x[::7] *= 1e16
            assert oracle.pysum(x) == sum(x.tolist())
    assert oracle.pysum([-0.0]) == sum([-0.0]) and str(sum([-0.0])) == "0.0"
    assert oracle.pysum([1e308, 1e308, -1e308]) == sum([1e308, 1e308, -1e308])


def test_c1_known_answer_vectors():
    GC.check_c1_known_answer(OracleScorer())


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_replay_c1_c3(name):
    runs, arrs = G.load(name)
    bad = []
    records = {}
    for r in runs:
        if name == "c1":
            inst, cfg = G.c1_setup(r["variant"])
        else:
            inst, cfg = G.c3_setup(r["ratio"], r["batch"], r["shape"])
        rec, problems, _ = G.replay(r, arrs, inst, cfg, OracleScorer())
        if name == "c3":
            records[(r["ratio"], r["batch"], r["shape"])] = rec
        if problems:
            bad.append(problems[:3])
    assert not bad, bad
    if name == "c3":
        assert GC.check_c3_table(records) == GC.C3_TABLE_FATE


def test_replay_c2_and_table1():
    runs, arrs = G.load("c2")
    records, bad = [], []
    scorer = OracleScorer()
    for r in runs:
        inst, cfg = G.c2_setup(r["key"])
        rec, problems, _ = G.replay(r, arrs, inst, cfg, scorer)
        records.append(rec)
        if problems:
            bad.append((r["key"], problems[:3]))
    assert not bad, bad[:5]
    GC.check_c2_table1(records)


@pytest.mark.skipif(not os.path.exists(os.path.join(G.GOLDEN, "c45_sampled.json")),
                    reason="c45 golden not generated")
def test_c45_sampled():
    assert GC.check_c45_sampled(gpu=False) > 2000


def test_c5_assignments_budget0():
    assert GC.check_c5_assign(gpu=False) == 16


def test_c5_full_frontiers_oracle():
    """The oracle on all frontier candidates of the 64 golden config-5
    instances (native generator, one instance at a time) and the budget-0
    assignments of both solvers on its matrix."""
    assert GC.check_c5_full(gpu=False) == 89312


@pytest.mark.skipif(not os.path.exists(os.path.join(G.GOLDEN, "c4_assign.json")),
                    reason="c4 golden not generated yet")
def test_c4_frontier_oracle_two_scenarios():
    assert GC.check_c4_assign(gpu=False, scenarios_=(0, 5)) > 15000
