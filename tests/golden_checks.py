"""Golden checks shared by the oracle (CPU) and GPU test suites."""

from __future__ import annotations

import json
import math
import os

import numpy as np

from paper_2605_07238_b200 import pack, scenarios

import golden_replay as G

# table1_overall FATE row of the reference's default manifest
# (SURVEY.md App. C.4 / BASELINE.md §2): norm_makespan, norm_p95, xdev, cache, cont
C2_TABLE1_FATE = ("0.820", "0.820", "0.874", "0.416", "0.573")

# known-answer Psi of config 1 (captured from the reference)
C1_WAVE0 = {
    "alignment_to_reference": ("-0x1.9485d66e363ecp+1", "-0x1.7b6837f7be122p+3"),
    "alignment_to_reference+17": ("-0x1.0062cd54b208fp+2", "-0x1.5e98ea4731170p+3"),
    "alignment_to_reference+27": ("-0x1.1a7c17a89331cp+1", "-0x1.5cf80dc33721ep+3"),
    "alignment_to_reference+4": ("0x1.d623d0bfa0940p-1", "-0x1.defa765343740p+3"),
    "alignment_to_reference+4+13": ("-0x1.1531769a91107p+2", "-0x1.6f1e7d9988d2ap+3"),
    "alignment_to_reference+4+13+29": ("-0x1.4e58e64b23141p+2", "-0x1.7337110e453d2p+3"),
    "alignment_to_reference+4+28": ("-0x1.1dc96030c23fbp+2", "-0x1.6110a137f38c6p+3"),
    "alignment_to_reference+8": ("-0x1.ac2ee84ad794bp+3", "-0x1.d2b0bbf50e348p+3"),
    "alignment_to_reference+8+30": ("-0x1.82893faf42786p+3", "-0x1.d8d5992428d44p+3"),
}
C1_WAVE1 = {
    "alignment_to_reference+4+13": (
        ("-0x1.5c4f3343fa2adp+5", "-0x1.947dc37a3db3cp+3", "-0x1.09aae6c8f7554p+3",
         "-0x1.7b585be1a8262p+5"),
        ("-0x1.90b6aa4b9884dp+5", "-0x1.330dcfcc5b8dcp+4", "-0x1.db48c2e770bd0p+3",
         "-0x1.afbfd2e946802p+5")),
    "alignment_to_reference+8": (
        ("-0x1.2cd245b291b82p+5", "-0x1.55a2834d26fa4p+5", "-0x1.32edcc20d562ap+5",
         "-0x1.dbdb6e503fb37p+5"),
        ("-0x1.199b39e279dd4p+5", "-0x1.126b777d0f1f5p+5", "-0x1.df6d80a17b0f7p+4",
         "-0x1.c8a4628027d89p+5")),
}
C1_WAVE10 = {
    "alignment_to_reference+8": (
        ("-0x1.ed0247021d106p+1", "-0x1.52d9a847b2462p+5", "-0x1.6fc6759ab6d01p+4",
         "-0x1.620398a654930p+4"),
        ("-0x1.732314013ec3bp+0", "-0x1.5c7a1d323fee2p+5", "-0x1.d2b0bbf50e348p+3",
         "-0x1.7544827b6fe2ep+4")),
}


class _Recorder:
    def __init__(self, inner):
        self.inner = inner
        self.waves = []

    def score_wave(self, frontier, state, cost_model, dag=None):
        ws = self.inner.score_wave(frontier, state, cost_model, dag)
        self.waves.append(ws)
        return ws


def check_c1_known_answer(scorer) -> None:
    from wfsched.executor import run

    from paper_2605_07238_b200.planner import FateGpuPolicy

    inst, cfg = G.c1_setup({"tag": "default", "horizon": 2})
    rec = _Recorder(scorer)
    record = run(FateGpuPolicy(scorer=rec), inst, cfg)
    assert record.makespan == 607.6001919999999
    assert (record.workflow_tasks, record.cross_device_parent_edges,
            record.prefix_cache_hits_est, record.same_model_continuations) == (50, 54, 21, 34)
    assert (record.solver_solves, record.solver_optimal) == (48, 48)

    def table(ws):
        out = {}
        for c in ws.candidates():
            out.setdefault(c.stage_id, {}).setdefault(c.slot, {})[c.device_id] = c.psi.hex()
        return out

    w0 = table(rec.waves[0])
    assert sorted(w0) == sorted(C1_WAVE0)
    for sid, (s0, s1) in C1_WAVE0.items():
        assert set(w0[sid][0].values()) == {float.fromhex(s0).hex()}, sid
        assert set(w0[sid][1].values()) == {float.fromhex(s1).hex()}, sid
    for wave_i, known in ((1, C1_WAVE1), (10, C1_WAVE10)):
        tab = table(rec.waves[wave_i])
        for sid, slots in known.items():
            for k, vals in enumerate(slots):
                got = [tab[sid][k][f"d{j}"] for j in range(4)]
                assert got == [float.fromhex(v).hex() for v in vals], (wave_i, sid, k)


def _csv6(x: float) -> float:
    return float(f"{x:.6f}")


def _geo(values) -> float:
    acc = 0.0
    for v in values:
        acc += math.log(v)
    return math.exp(acc / len(values))


def check_c2_table1(fate_records) -> None:
    """FATE row of table1_overall (reference harness.py:549-566, metrics.py)
    from replayed FATE records + golden RoundRobin records."""
    with open(os.path.join(G.GOLDEN, "c2_baselines.json")) as fh:
        base = json.load(fh)["records"]
    rr = {(r["workflow_id"], r["batch_size"], r["perturbation"]): r
          for r in base if r["method"] == "roundrobin"}
    norm_ms, norm_p95 = [], []
    tasks = xdev = hits = cont = 0
    for rec in fate_records:
        b = rr[(rec.workflow_id, rec.batch_size, rec.perturbation)]
        norm_ms.append(_csv6(rec.makespan) / _csv6(float.fromhex(b["makespan"])))
        norm_p95.append(_csv6(rec.p95_latency()) / _csv6(float.fromhex(b["p95"])))
        tasks += rec.workflow_tasks
        xdev += rec.cross_device_parent_edges
        hits += rec.prefix_cache_hits_est
        cont += rec.same_model_continuations
    got = (f"{_geo(norm_ms):.3f}", f"{_geo(norm_p95):.3f}", f"{xdev / tasks:.3f}",
           f"{hits / tasks:.3f}", f"{cont / tasks:.3f}")
    assert len(fate_records) == 96
    assert got == C2_TABLE1_FATE, got


# C3 at H=3, batch 16, normalised by halo at ratio 0
# (harness.py:620-626 / _suite_table 711-733)
C3_TABLE_FATE = ("0.936", "0.890", "0.820", "0.705")


def check_c3_table(fate_records) -> tuple:
    """The normalised prefix-reuse table's FATE row, recomputed from the
    GPU-run FATE records and the reference's halo records (golden
    c3_baselines.json, H=3) exactly as ``_suite_table`` does: per ratio the
    geometric mean of the CSV-rounded makespans of the batch-16 instances,
    divided by halo's at ratio 0."""
    with open(os.path.join(G.GOLDEN, "c3_baselines.json")) as fh:
        base = json.load(fh)["records"]
    assert len(fate_records) == 24
    ratios = (0.0, 0.25, 0.5, 1.0)

    def geo_of(recs):
        return _geo([_csv6(float.fromhex(r["makespan"])) if isinstance(r, dict)
                     else _csv6(r.makespan) for r in recs])

    halo0 = geo_of([r for r in base if r["method"] == "halo" and r["ratio"] == 0.0
                    and r["batch"] == 16])
    row = []
    for ratio in ratios:
        recs = [rec for (rr, b, _k), rec in fate_records.items() if rr == ratio and b == 16]
        assert len(recs) == 3
        row.append(f"{geo_of(recs) / halo0:.3f}")
    assert tuple(row) == C3_TABLE_FATE, row
    return tuple(row)


def check_c45_sampled(gpu: bool) -> int:
    with open(os.path.join(G.GOLDEN, "c45_sampled.json")) as fh:
        samples = json.load(fh)["samples"]
    cfg4 = scenarios.config_c4_catalog()
    inst4 = None
    cfg5 = scenarios.config_c5()
    checked = 0
    groups: dict = {}
    for smp in samples:
        groups.setdefault((smp["which"], smp["instance"]), []).append(smp)
    for (which, idx), smps in sorted(groups.items()):
        if which == "c4":
            inst4 = inst4 or scenarios.c4_instance(cfg4)
            inst, cfg = inst4, cfg4
        else:
            inst, cfg = scenarios.c5_instance(idx, cfg5), cfg5
        bank = pack.pack_bank([inst], cfg.models, cfg.topology)
        states, items, wants = [], [], []
        for smp in smps:
            st = scenarios.build_scenario(inst, cfg, smp["scenario"])
            assert st.clock.hex() == smp["clock"]
            if smp.get("frontier") is not None:
                assert scenarios.scenario_frontier(inst, st) == smp["frontier"]
            states.append((0, st))
            for it in smp["items"]:
                items.append((len(states) - 1, bank.global_index(0, it["stage"])))
                wants.append(it)
        pst = pack.pack_states(bank, states)
        work = pack.make_work(bank, items, cfg.weights.ablation.no_shard)
        wrec = pack.weights_record(cfg.weights)
        if gpu:
            from paper_2605_07238_b200 import runtime

            res = runtime.DeviceBank(bank, cfg.weights).score(pst, work, extras=True)
            out = {k: getattr(res, k).cpu().numpy() for k in ("psi", "sched", "tail",
                                                               "completion")}
        else:
            import oracle

            out = oracle.score(bank, wrec, pst, work)
        D = bank.scalars["n_devices"]
        for w, it in enumerate(wants):
            g = int(work.stage[w])
            m = int(bank.arrays["st_elig"][g])
            cols = [d for d in range(D) if m >> d & 1]
            for k, row in enumerate(it["psi"]):
                base = int(work.psi_off[w]) + k * D
                got = out["psi"][base: base + D][cols].view(np.uint64).tolist()
                assert got == row, (which, idx, it["stage"], k)
                checked += len(row)
            for key in ("sched", "tail", "completion"):
                got = out[key][w * D: (w + 1) * D][cols].view(np.uint64).tolist()
                assert got == it[key], (which, idx, it["stage"], key)
    return checked


def check_c5_assign(gpu: bool, native_solver: bool = False) -> int:
    """Config-5 assignments: the host solve (budget 0, deterministic greedy) on
    the GPU/oracle cost matrix selects exactly what the reference's solve
    selects on the reference's own cost matrix (tests/golden/c5_assign.json).
    ``native_solver`` solves with ``fate_solve_frontier`` instead of the
    Python restatement."""
    from wfsched.planner import Candidate, FrontierProblem, solve_frontier

    if native_solver:
        from paper_2605_07238_b200.solver import solve_frontier

    with open(os.path.join(G.GOLDEN, "c5_assign.json")) as fh:
        golden = json.load(fh)
    cfg = scenarios.config_c5()
    n = 0
    for g in golden["instances"]:
        i = g["instance"]
        inst = scenarios.c5_instance(i, cfg)
        st = scenarios.build_scenario(inst, cfg, i)
        bank = pack.pack_bank([inst], cfg.models, cfg.topology)
        sids = scenarios.scenario_frontier(inst, st)
        pst = pack.pack_states(bank, [(0, st)])
        work = pack.make_work(bank, [(0, bank.global_index(0, s)) for s in sids], False)
        if gpu:
            from paper_2605_07238_b200 import runtime

            psi = runtime.DeviceBank(bank, cfg.weights).score(pst, work, extras=False).psi
            psi = psi.cpu().numpy()
        else:
            import oracle

            psi = oracle.score(bank, pack.weights_record(cfg.weights), pst, work)["psi"]
        cands = tuple(Candidate(*c) for c in pack.candidates_from_psi(bank, work, psi, 0))
        assert len(cands) == g["n_candidates"]
        prob = FrontierProblem(cands, {s: int(b) for s, b in zip(sids, work.bounds)},
                               tuple(cfg.topology.device_ids))
        sol = solve_frontier(prob, budget_s=golden["budget_s"])
        assert [list(x) for x in sol.selected] == g["selected"], i
        assert sol.objective.hex() == g["objective"], i
        n += 1
    return n


# ---------------------------------------------------------------------------
# round 2: SURVEY §8(d) parity gates at full size (make_golden.py --r2)
# ---------------------------------------------------------------------------


def _f64(bits_list):
    return np.asarray(bits_list, dtype=np.uint64)


def _solve_both(cands, bounds, device_ids, budget):
    """Budget-0 host solve of a cost matrix with the reference's own
    ``solve_frontier`` and with the native one; both results returned."""
    from wfsched.planner import Candidate, FrontierProblem, solve_frontier

    from paper_2605_07238_b200.solver import solve_frontier as native

    prob = FrontierProblem(tuple(Candidate(*c) for c in cands), bounds, tuple(device_ids))
    return solve_frontier(prob, budget_s=budget), native(prob, budget_s=budget)


def _check_wave(bank, work, out, items, want_psi, want_sched, want_compl, meta, cfg, tag):
    """Psi (candidate order), S and completion ((stage, eligible device)
    order) of the items ``items`` of one scenario, then the budget-0
    assignments of both solvers, against the reference's."""
    D = bank.scalars["n_devices"]
    devs = bank.device_ids
    inst = int(bank.arrays["st_inst"][int(work.stage[items[0]])])
    off0 = int(bank.inst_stage_off[inst])
    sids = bank.stage_ids[inst]
    cands, sched, compl, bounds = [], [], [], {}
    for w in items:
        g = int(work.stage[w])
        sid = sids[g - off0]
        mask = int(bank.arrays["st_elig"][g])
        base = int(work.psi_off[w])
        bounds[sid] = int(work.bounds[w])
        for k in range(bounds[sid]):
            for d in range(D):
                if mask >> d & 1:
                    cands.append((sid, k, devs[d], float(out["psi"][base + k * D + d])))
        for d in range(D):
            if mask >> d & 1:
                sched.append(out["sched"][w * D + d])
                compl.append(out["completion"][w * D + d])
    assert [c[0] for c in cands][:1] and sorted(bounds) == meta["frontier"], tag
    assert len(cands) == meta["n_cand"], tag
    got = np.asarray([c[3] for c in cands], dtype=np.float64).view(np.uint64)
    assert np.array_equal(got, want_psi), tag
    assert np.array_equal(np.asarray(sched, dtype=np.float64).view(np.uint64), want_sched), tag
    assert np.array_equal(np.asarray(compl, dtype=np.float64).view(np.uint64), want_compl), tag
    ref, nat = _solve_both(cands, bounds, cfg.topology.device_ids, 0.0)
    for sol in (ref, nat):
        assert [list(x) for x in sol.selected] == meta["selected"], tag
        assert sol.objective.hex() == meta["objective"], tag
        assert sol.optimal == meta["optimal"], tag
    return len(cands)


def _score(bank, weights, states, work, gpu):
    if gpu:
        from paper_2605_07238_b200 import runtime

        res = runtime.DeviceBank(bank, weights).score(states, work, extras=True)
        return {k: getattr(res, k).cpu().numpy() for k in ("psi", "sched", "completion")}
    import oracle

    return oracle.score(bank, pack.weights_record(weights), states, work)


def _load_r2(name):
    with open(os.path.join(G.GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)
    arr = np.load(os.path.join(G.GOLDEN, f"{name}.npz"))
    return meta, {k: arr[k] for k in arr.files}


def check_c5_full(gpu: bool) -> int:
    """Every frontier candidate of 64 config-5 instances (i = 0, 64, ...,
    4032) and their budget-0 assignments.  On the GPU the batch is the bench's
    own (bench.build_c5: all 4096 instances, one launch); on the CPU (oracle)
    each instance is generated alone by the same native generator."""
    import bench
    from paper_2605_07238_b200 import fastgen

    meta, arr = _load_r2("c5_full")
    cfg = scenarios.config_c5()
    if gpu:
        cfg, bank, states, work = bench.build_c5(bench.shard_plan(0, 1), "frontier")
        out = _score(bank, cfg.weights, states, work, True)
        scen = np.asarray(work.scen)
    pc = sc = 0
    n = 0
    for m in meta["instances"]:
        i = m["instance"]
        if not gpu:
            fb = fastgen.synth_batch(cfg, 1, 1000 + i, i, *bench.C5_SHAPE.values())
            sc_i, g_i = fb.frontier_items()
            bank, states = fb.bank, fb.states
            work = pack.make_work(bank, zip(sc_i.tolist(), g_i.tolist()), False)
            out = _score(bank, cfg.weights, states, work, False)
            items = list(range(work.n_items))
        else:
            items = np.flatnonzero(scen == i).tolist()
        n += _check_wave(bank, work, out, items, arr["psi"][pc: pc + m["n_cand"]],
                         arr["sched"][sc: sc + m["n_pairs"]],
                         arr["completion"][sc: sc + m["n_pairs"]], m, cfg, ("c5", i))
        pc += m["n_cand"]
        sc += m["n_pairs"]
    return n


def check_c4_assign(gpu: bool, scenarios_: tuple | None = None) -> int:
    """Every frontier candidate of the 8 canonical config-4 scenarios (the
    bench's frontier-mode batch, bench.build_c4) and their budget-0
    assignments."""
    import bench

    meta, arr = _load_r2("c4_assign")
    cfg, bank, states, work = bench.build_c4("frontier")
    out = _score(bank, cfg.weights, states, work, gpu)
    scen = np.asarray(work.scen)
    pc = sc = 0
    n = 0
    for m in meta["scenarios"]:
        s = m["scenario"]
        if scenarios_ is None or s in scenarios_:
            assert states.arrays["scen_clock"][s].hex() == m["clock"]
            items = np.flatnonzero(scen == s).tolist()
            n += _check_wave(bank, work, out, items, arr["psi"][pc: pc + m["n_cand"]],
                             arr["sched"][sc: sc + m["n_pairs"]],
                             arr["completion"][sc: sc + m["n_pairs"]], m, cfg, ("c4", s))
        pc += m["n_cand"]
        sc += m["n_pairs"]
    return n
