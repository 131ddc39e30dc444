"""Oracle vs the reference scorer itself (build container only).

Runs the reference ``CostModel`` (``wfsched/costs.py``) on the very same
objects the packer consumes and requires the C oracle to reproduce every Psi,
S, tail and completion bit.  Skipped where the reference is absent (GPU box);
there the committed golden vectors (test_oracle_golden.py) pin the oracle.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

import oracle
from paper_2605_07238_b200.wf.weights import AblationFlags

from cases import ALL_ABLATIONS, bits, c5_case, edge_case, small_case, token_case

pytestmark = pytest.mark.reference


def reference_scores(ref, case):
    from wfsched.costs import CostModel

    cm = CostModel(case.cfg.models, case.cfg.topology, case.weights)
    bank = case.bank
    n_dev = bank.scalars["n_devices"]
    psi = np.full(case.work.n_psi, np.nan)
    extra = {k: np.full(case.work.n_items * n_dev, np.nan) for k in ("sched", "tail", "completion")}
    scen_objs = case.scen_objs
    for w in range(case.work.n_items):
        s = int(case.work.scen[w])
        g = int(case.work.stage[w])
        ii, st = scen_objs[s]
        inst = case.instances[ii]
        sid = bank.stage_ids[ii][g - int(bank.inst_stage_off[ii])]
        stage = inst.dag.stages[sid]
        qids = tuple(q.query_id for q in inst.queries)
        for k in range(int(case.work.bounds[w])):
            for d, dev in enumerate(bank.device_ids):
                if dev in stage.eligible_devices:
                    psi[int(case.work.psi_off[w]) + k * n_dev + d] = cm.plan_score(stage, k, dev, st, inst.dag)
        for d, dev in enumerate(bank.device_ids):
            if dev not in stage.eligible_devices:
                continue
            r = w * n_dev + d
            extra["sched"][r] = cm.sched_score(stage, dev, st, inst.dag)
            extra["tail"][r] = cm.tail_value(stage, dev, st, inst.dag)
            t = cm.realized_duration(stage, [(dev, qids)], st, inst.dag)[0]
            extra["completion"][r] = max(0.0, st.device_free.get(dev, 0.0) - st.clock) + t.total_s
    return psi, extra


def _check(ref, case):
    got = oracle.score(case.bank, case.wrec, case.states, case.work)
    psi, extra = reference_scores(ref, case)
    assert np.array_equal(bits(got["psi"]), bits(psi)), case
    for k in extra:
        assert np.array_equal(bits(got[k]), bits(extra[k])), (case, k)


def _with_objs(builder, *a, **kw):
    # rebuild keeping the (instance, state) objects for the reference side
    import cases as C

    orig = C.Case.__init__

    def init(self, name, instances, cfg, weights, scen_states, items):
        orig(self, name, instances, cfg, weights, scen_states, items)
        self.scen_objs = list(scen_states)

    C.Case.__init__ = init
    try:
        return builder(*a, **kw)
    finally:
        C.Case.__init__ = orig


@pytest.mark.parametrize("horizon", [0, 1, 2, 3, 4, 6])
def test_edge_case_all_branches(reference, horizon):
    _check(reference, _with_objs(edge_case, horizon=horizon))


@pytest.mark.parametrize("flag", ALL_ABLATIONS)
def test_edge_case_ablations(reference, flag):
    _check(reference, _with_objs(edge_case, horizon=3,
                                 ablation=AblationFlags.from_names([flag])))


def test_edge_case_no_overrides(reference):
    _check(reference, _with_objs(edge_case, horizon=4, overrides=False))


def test_lifted_scenarios(reference):
    _check(reference, _with_objs(small_case))


def test_prefix_suite_scenarios(reference):
    _check(reference, _with_objs(small_case, prefix=True))


def test_c5_frontier(reference):
    _check(reference, _with_objs(c5_case, n_inst=2))


def test_partial_hit_token_case(reference):
    _check(reference, _with_objs(token_case, horizon=3))
