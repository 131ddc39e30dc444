"""Native batch generator == packing the Python objects (bit for bit)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2605_07238_b200 import fastgen, pack, runtime, scenarios
from paper_2605_07238_b200.wf import workloads as W
from paper_2605_07238_b200.wf.weights import default_config

pytestmark = pytest.mark.skipif(not os.path.exists(runtime.LIB_PATH), reason="libfate.so not built")


@pytest.mark.parametrize("spec", [
    ("c5", 6, 1000, 20, 25, 0.12, 16),
    ("c4-like", 2, 1, 12, 30, 0.03, 16),
    ("tiny", 5, 77, 3, 2, 0.9, 5),
])
def test_fastgen_equals_object_path(spec):
    _, n, seed0, depth, width, density, batch = spec
    cfg = scenarios.config_c5() if spec[0] == "c5" else scenarios.config_c4_catalog()
    fb = fastgen.synth_batch(cfg, n, seed0, 0, depth, width, density, batch)
    insts = [W.make_instance(W.synth_generate(W.SuiteSpec(kind="synthetic", depth=depth, width=width,
                                                          density=density, seed=seed0 + i,
                                                          batch_size=batch), cfg),
                             batch, seed0 + i) for i in range(n)]
    bank = pack.pack_bank(insts, cfg.models, cfg.topology)
    states = pack.pack_states(bank, [(i, scenarios.build_scenario(inst, cfg, i))
                                     for i, inst in enumerate(insts)], kappa_cap=fb.states.kappa_cap)
    a, b = fb.bank.arrays, bank.arrays
    for k in ("st_inst", "st_model", "st_prompt", "st_out", "st_flags", "st_shard", "st_level",
              "st_elig", "par_ptr", "par_idx", "ch_ptr", "ch_idx", "q_prompt", "q_group",
              "dev_speed", "beta", "model_prefill", "model_decode", "model_switch"):
        assert np.array_equal(a[k], b[k]), k
    for k in ("role_cplx", "role_prefill", "role_decode", "role_comm"):
        assert np.array_equal(a[k][a["st_role"]], b[k][b["st_role"]]), k
    # groups: the fast path numbers pg:<alias> by model id; compare by name
    inv_a = {v: k for k, v in fb.bank.group_index.items()}
    inv_b = {v: k for k, v in bank.group_index.items()}
    ga = [inv_a.get(int(x)) for x in a["st_group"]]
    gb = [inv_b.get(int(x)) for x in b["st_group"]]
    assert ga == gb
    sa, sb = fb.states.arrays, states.arrays
    for k in ("scen_inst", "scen_clock", "scen_loc_off", "loc", "residency", "dev_free", "kappa_n"):
        assert np.array_equal(sa[k], sb[k]), k
    ka = sa["kappa"].reshape(-1, fb.states.kappa_cap, 4).copy()
    kb = sb["kappa"].reshape(-1, states.kappa_cap, 4).copy()
    n_live = sa["kappa_n"]
    for r in range(ka.shape[0]):
        ea = [(inv_a[int(e[0])], int(e[1]), int(e[2])) for e in ka[r, : n_live[r]]]
        eb = [(inv_b[int(e[0])], int(e[1]), int(e[2])) for e in kb[r, : n_live[r]]]
        assert ea == eb, r
    # frontier = ready_set of the scenario
    sc, g = fb.frontier_items()
    for i, inst in enumerate(insts):
        st = scenarios.build_scenario(inst, cfg, i)
        want = [bank.global_index(i, s) for s in scenarios.scenario_frontier(inst, st)]
        assert sorted(g[sc == i].tolist()) == want


def test_c4_builder_equals_object_path():
    """bench.build_c4 (native generator, 8 scenario states of one 10k-stage
    instance) == packing the mirror objects of scenarios.c4_instance."""
    import bench

    cfg, bank, states, work = bench.build_c4("frontier", n_scen=2)
    inst = scenarios.c4_instance(cfg)
    ref = pack.pack_bank([inst], cfg.models, cfg.topology)
    for k in ("st_model", "st_prompt", "st_out", "st_flags", "st_shard", "st_level", "par_ptr",
              "par_idx", "ch_ptr", "ch_idx", "q_prompt"):
        assert np.array_equal(bank.arrays[k], ref.arrays[k]), k
    rs = pack.pack_states(ref, [(0, scenarios.build_scenario(inst, cfg, s)) for s in range(2)],
                          kappa_cap=states.kappa_cap)
    for k in ("scen_clock", "loc", "residency", "dev_free", "kappa_n"):
        assert np.array_equal(states.arrays[k], rs.arrays[k]), k
    front = [ref.global_index(0, sid) for s in range(2)
             for sid in scenarios.scenario_frontier(inst, scenarios.build_scenario(inst, cfg, s))]
    assert work.stage.tolist() == front
