"""CPU tests of the host side: C-ABI library exports, native window builder,
packer invariants, solver vs exhaustive enumeration (no GPU needed)."""

from __future__ import annotations

import ctypes
import itertools
import os
import random
import re

import numpy as np
import pytest

from paper_2605_07238_b200 import pack, runtime, scenarios
from wfsched.planner import Candidate, FrontierProblem, check_constraints, solve_frontier

from cases import c5_case, edge_case, small_case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    text = open(os.path.join(ROOT, "include", "fate.h")).read()
    return re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(fate_\w+)\s*\(", text, re.M)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(runtime.LIB_PATH):
        pytest.skip("libfate.so not built")
    lib = ctypes.CDLL(runtime.LIB_PATH)
    names = _declared_functions()
    assert {"fate_score", "fate_prepare", "fate_windows_build_host"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n
    assert runtime.load_library().fate_abi_version() == 3


def _py_windows(bank, levels):
    a = bank.arrays
    ptr = [0]
    idx = []
    lvl = a["st_level"]
    ch_ptr, ch_idx = a["ch_ptr"], a["ch_idx"]
    for v in range(bank.n_stages):
        seen, front, found = set(), [v], []
        while front:  # full descendant walk, like the reference
            nxt = []
            for u in front:
                for c in ch_idx[ch_ptr[u]:ch_ptr[u + 1]]:
                    if c not in seen:
                        seen.add(int(c))
                        nxt.append(int(c))
            front = nxt
        for l in range(1, levels + 1):
            bucket = sorted(x for x in seen if lvl[x] - lvl[v] == l)
            idx += bucket
            ptr.append(len(idx))
    return np.asarray(ptr), np.asarray(idx)


@pytest.mark.parametrize("levels", [0, 1, 2, 3, 5])
def test_native_windows_equal_full_descendant_walk(levels):
    if not os.path.exists(runtime.LIB_PATH):
        pytest.skip("libfate.so not built")
    for case in (edge_case(), small_case(), c5_case(n_inst=2)):
        bank = case.bank
        bank.windows.clear()
        ptr, idx = runtime.build_windows(bank, levels)
        want_ptr, want_idx = _py_windows(bank, levels)
        assert np.array_equal(ptr, want_ptr)
        assert np.array_equal(idx[: ptr[-1]], want_idx)


def test_pack_roundtrip_state():
    case = edge_case()
    bank = case.bank
    st = case.states
    D = bank.scalars["n_devices"]
    # residency / free / kappa round trip for scenario 0
    import cases as C

    c = C.edge_case()
    assert np.array_equal(c.states.arrays["residency"], st.arrays["residency"])
    assert st.kappa_cap >= 1
    assert st.arrays["residency"].size == st.n_scenarios * D


def test_bounds_follow_planner_rule():
    case = edge_case(horizon=2)
    for w in range(case.work.n_items):
        g = int(case.work.stage[w])
        R = int(case.bank.arrays["st_shard"][g])
        n = bin(int(case.bank.arrays["st_elig"][g])).count("1")
        assert case.work.bounds[w] == min(R, n)


def _random_problem(rng, n_stages, n_dev):
    devs = [f"d{i}" for i in range(n_dev)]
    cands, bounds = [], {}
    for s in range(n_stages):
        sid = f"s{s:02d}"
        b = rng.choice([1, 2])
        bounds[sid] = b
        for k in range(b):
            for d in devs:
                cands.append(Candidate(sid, k, d, round(rng.uniform(-10, 10), 4)))
    return FrontierProblem(tuple(cands), bounds, tuple(devs))


def _enumerate(problem):
    """Exhaustive optimum (same objective and tie-break as the reference's
    verification.enumerate_optimum, verification.py:36-71)."""
    by = {}
    for c in problem.candidates:
        by.setdefault(c.stage_id, {}).setdefault(c.slot, {})[c.device_id] = c.psi
    stages = sorted(by)
    per = []
    for sid in stages:
        opts = [((), 0.0)]
        devs = sorted(problem.device_ids)
        for n in range(1, len(by[sid]) + 1):
            for combo in itertools.permutations(devs, n):
                if all(d in by[sid][k] for k, d in enumerate(combo)):
                    val = 0.0
                    for k, d in enumerate(combo):
                        val += by[sid][k][d]
                    opts.append((tuple((sid, k, d) for k, d in enumerate(combo)), val))
        per.append(opts)
    best = (0.0, ())
    for choice in itertools.product(*per):
        used = [d for t, _ in choice for (_, _, d) in t]
        if len(used) != len(set(used)):
            continue
        val = 0.0
        for _, v in choice:
            val += v
        sel = tuple(sorted(x for t, _ in choice for x in t))
        if val > best[0] + 1e-12:
            best = (val, sel)
    return best


def test_solver_matches_exhaustive_search():
    rng = random.Random(7)
    for _ in range(60):
        prob = _random_problem(rng, rng.randint(1, 4), rng.randint(1, 3))
        sol = solve_frontier(prob, budget_s=5.0)
        assert sol.optimal
        assert not check_constraints(prob, sol.selected)
        opt, _ = _enumerate(prob)
        assert abs(sol.objective - opt) <= 1e-9


def test_solver_timeout_falls_back_to_greedy():
    rng = random.Random(1)
    prob = _random_problem(rng, 6, 4)
    sol = solve_frontier(prob, budget_s=0.0)
    assert not check_constraints(prob, sol.selected)


def test_scenario_generator_is_deterministic():
    cfg = scenarios.config_c5()
    inst = scenarios.c5_instance(3, cfg)
    a = scenarios.build_scenario(inst, cfg, 3)
    b = scenarios.build_scenario(inst, cfg, 3)
    assert a.clock == b.clock and a.residency == b.residency
    assert a.parent_loc == b.parent_loc and a.device_free == b.device_free
    front = scenarios.scenario_frontier(inst, a)
    assert len(front) == 25


def test_pipeline_rejects_bad_arguments_before_touching_cuda():
    """fate_pipeline_create validates its sizes first (status < 0, no CUDA call)."""
    if not os.path.exists(runtime.LIB_PATH):
        pytest.skip("libfate.so not built")
    L = runtime.load_library()
    h = ctypes.c_void_p()
    assert L.fate_pipeline_create(0, 0, 1, ctypes.byref(h)) == -1
    assert L.fate_pipeline_create(0, 4, 0, ctypes.byref(h)) == -1
    assert b"chunk" in L.fate_last_error()
    assert L.fate_pipeline_destroy(None) == 0


def test_host_batch_wire_format_round_trip():
    """The scenario records follow fate.h's FATE_SCEN_REC_BYTES layout."""
    case = c5_case(n_inst=3)
    D = case.bank.scalars["n_devices"]
    hb = pack.host_batch(case.states, case.work, D)
    a, S, cap = case.states.arrays, case.states.n_scenarios, case.states.kappa_cap
    rb = pack.scen_rec_bytes(D, cap)
    assert rb % 16 == 0 and hb.rec.size == S * rb
    rec = hb.rec.reshape(S, rb)
    assert np.array_equal(rec[:, 0:8].copy().view("<f8").ravel(), a["scen_clock"])
    assert np.array_equal(rec[:, 8:16].copy().view("<i8").ravel(), a["scen_loc_off"])
    assert np.array_equal(rec[:, 16:20].copy().view("<i4").ravel(), a["scen_inst"])
    assert np.array_equal(rec[:, 20:24].copy().view("<i4").ravel(), a["scen_done_level"])
    o = 32
    assert np.array_equal(rec[:, o:o + 4 * D].copy().view("<i4").ravel(), a["residency"])
    o += 4 * D
    assert np.array_equal(rec[:, o:o + 4 * D].copy().view("<i4").ravel(), a["kappa_n"])
    o += 4 * D
    assert np.array_equal(rec[:, o:o + 8 * D].copy().view("<f8").ravel(), a["dev_free"])
    o += 8 * D
    assert np.array_equal(rec[:, o:].copy().view("<i4").ravel(), np.ravel(a["kappa"]))
    assert hb.items.itemsize == 16
    assert np.array_equal(hb.items["stage"], case.work.stage)
    assert np.array_equal(hb.items["psi_off"], case.work.psi_off)


def test_ptx_contraction_check_allows_only_tagged_exact_fmas():
    from paper_2605_07238_b200 import build

    tagged = ("// begin inline asm\n{\n\t// fate-fma01\n\tfma.rn.f64 %fd1, %fd2, f, %fd1;\n}\n"
              "// end inline asm\n")
    plain = "\tfma.rn.f64 %fd3, %fd4, %fd5, %fd6;\n"
    untagged_asm = "// begin inline asm\n\tfma.rn.f64 %fd1, %fd2, %fd3, %fd1;\n// end inline asm\n"
    assert build.ptx_contraction_free("add.rn.f64 %fd1, %fd2, %fd3;\n" + tagged)
    assert not build.ptx_contraction_free(tagged + plain)
    assert not build.ptx_contraction_free(untagged_asm)
    built = os.path.join(ROOT, "paper_2605_07238_b200", "fate_kernels.ptx")
    if os.path.exists(built):  # by-product of build(); the build itself also checks
        with open(built) as fh:
            assert build.ptx_contraction_free(fh.read())


def test_bank_flags_declare_query_groups_exactly():
    """FATE_BANK_NO_QGROUPS (the lean kernel) is set iff no query of the bank
    has a prefix group -- by the object packer and by the native generator."""
    from cases import token_case, wide_case
    from paper_2605_07238_b200 import fastgen

    c5 = c5_case(n_inst=2)
    assert c5.bank.scalars["flags"] & pack.BANK_NO_QGROUPS
    assert not np.any(c5.bank.arrays["q_group"] != -1)
    assert token_case().bank.scalars["flags"] & pack.BANK_NO_QGROUPS
    for case in (edge_case(), wide_case(33, 16, 3, False, 3)):
        assert np.any(case.bank.arrays["q_group"] != -1)
        assert not case.bank.scalars["flags"] & pack.BANK_NO_QGROUPS
    fb = fastgen.synth_batch(scenarios.config_c5(), 2, 1000, 0, 20, 25, 0.12)
    assert fb.bank.scalars["flags"] & pack.BANK_NO_QGROUPS


def test_c_abi_from_plain_c(tmp_path):
    """examples/solve_frontier.c links libfate.so from C (no Python) and its
    native solve equals the reference's solve_frontier on the same problem (selection, objective, node count)."""
    import shutil
    import subprocess

    from wfsched.planner import Candidate as Cd

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib_dir = os.path.join(ROOT, "paper_2605_07238_b200")
    exe = str(tmp_path / "solve_frontier")
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "solve_frontier.c"), "-L", lib_dir, "-lfate",
                    f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    line = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.strip()
    fields = dict(kv.split("=", 1) for kv in line.split())
    cands = [Cd("s0", 0, "d0", 5.0), Cd("s0", 0, "d1", 3.0), Cd("s0", 1, "d0", 0.5),
             Cd("s0", 1, "d1", 0.25), Cd("s1", 0, "d0", 4.0), Cd("s1", 0, "d1", 6.0),
             Cd("s2", 0, "d2", -1.0)]
    want = solve_frontier(FrontierProblem(candidates=tuple(cands),
                                          shard_bounds={"s0": 2, "s1": 1, "s2": 1},
                                          device_ids=("d0", "d1", "d2")), budget_s=0.25)
    got = tuple(tuple(int(x) for x in t.split(":")) for t in fields["sel"].split(","))
    assert got == tuple((int(s[1:]), k, int(d[1:])) for s, k, d in want.selected)
    assert float(fields["objective"]) == want.objective
    assert int(fields["optimal"]) == int(want.optimal)
    assert int(fields["nodes"]) == want.nodes_explored
    assert int(fields["abi"]) == runtime.load_library().fate_abi_version()


def test_production_library_has_one_kernel_generation():
    """Without -DFATE_AB the library carries the v6 scoring kernel only (no
    v5 A/B generation) and no environment knobs."""
    import shutil
    import subprocess

    if not os.path.exists(runtime.LIB_PATH) or shutil.which("cuobjdump") is None:
        pytest.skip("libfate.so or cuobjdump missing")
    from paper_2605_07238_b200 import build

    if build.ab_build():
        pytest.skip("experiment build")
    names = subprocess.run(["cuobjdump", "-symbols", runtime.LIB_PATH], capture_output=True,
                           text=True).stdout
    assert "fate_score_v6_kernel" in names
    assert "fate_score_v5_kernel" not in names
    with open(runtime.LIB_PATH, "rb") as fh:
        blob = fh.read()
    for knob in (b"FATE_SCORE_KERNEL", b"FATE_MINB", b"FATE_V6_OPCAP", b"FATE_V6_FETCH",
                 b"FATE_PIPE_TRACE", b"FATE_V6_DYNLAYOUT"):
        assert knob not in blob, knob


def _capture_waves(inst, cfg):
    """(frontier, snapshot state, cost model) of every wave of one reference
    FATE run (the reference's own build_problem, wrapped)."""
    import wfsched.executor as RE
    import wfsched.policies as RP

    seen = []
    real = RP.build_problem

    def spy(frontier, state, cost_model, dag):
        seen.append((set(frontier), state, cost_model))
        return real(frontier, state, cost_model, dag)

    RP.build_problem = spy
    try:
        RE.run(RP.make_policy("fate"), inst, cfg)
    finally:
        RP.build_problem = real
    return seen


@pytest.mark.parametrize("which", ["c1", "c3"])
def test_wave_packer_equals_pack_states(which):
    """WaveRunner's single-scenario packer (pack.pack_state_into, written into
    the pinned staging block) gives the same fate_state arrays as
    pack.pack_states on every wave of a reference run."""
    import golden_replay as GR

    inst, cfg = GR.c1_setup({}) if which == "c1" else GR.c3_setup(0.5, 16, 1)
    waves = _capture_waves(inst, cfg)
    assert waves
    bank = pack.pack_bank([inst], cfg.models, cfg.topology)
    D = bank.scalars["n_devices"]
    n = len(bank.stage_ids[0])
    for frontier, st, _ in waves:
        ref = pack.pack_states(bank, [(0, st)])
        cap = ref.kappa_cap + 2
        v = {"scen_inst": np.zeros(1, np.int32), "scen_clock": np.zeros(1), "scen_loc_off":
             np.zeros(1, np.int64), "scen_done_level": np.zeros(1, np.int32),
             "residency": np.zeros(D, np.int32), "dev_free": np.zeros(D),
             "kappa_n": np.zeros(D, np.int32), "kappa": np.zeros(D * cap * 4, np.int32),
             "loc": np.zeros(n, np.int32)}
        pack.pack_state_into(bank, 0, st, v, cap)
        for k in ("scen_inst", "scen_clock", "scen_loc_off", "scen_done_level", "residency",
                  "dev_free", "kappa_n", "loc"):
            assert np.array_equal(v[k], ref.arrays[k]), k
        got = v["kappa"].reshape(D, cap, 4)[:, : ref.kappa_cap]
        assert np.array_equal(got, ref.arrays["kappa"].reshape(D, ref.kappa_cap, 4))
        assert not v["kappa"].reshape(D, cap, 4)[:, ref.kappa_cap:].any()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_c4_rank_shares_partition_the_sweep(world):
    """bench.c4_plan / build_c4: the ranks' (scenario, stage)
    work items are disjoint and together are exactly the single-process
    sweep, in the same per-rank order (scenario-major, ascending stage)."""
    import bench

    _, _, _, full = bench.build_c4("sweep", n_scen=2)
    want = set(zip(full.scen.tolist(), full.stage.tolist()))
    got = []
    for r in range(world):
        p = bench.c4_plan(r, world, n_scen=2)
        _, _, _, w = bench.build_c4("sweep", n_scen=p["count"], first_scen=p["first"],
                                    stage_rank=p["stage_rank"], stage_world=p["stage_world"])
        items = list(zip(w.scen.tolist(), w.stage.tolist()))
        assert items == sorted(items)
        assert all(g % world == r for _, g in items)
        got += items
    assert len(got) == len(set(got)) == len(want)
    assert set(got) == want
