"""Generate golden vectors by running the REFERENCE scheduler (build container).

    python tests/golden/make_golden.py [--quick]

Imports the reference package from /root/reference/pkg/src (read-only) and
records, for every planning wave of every captured run, the reference's own
outputs on the hot path:
  * Psi of every candidate, in FrontierProblem order
    (wfsched.planner.build_problem -> CostModel.plan_score);
  * S(v,d) = CostModel.sched_score and the work-conserving completion time
    wait + realized_duration(full batch).total_s (policies.py:91-95) for every
    (frontier stage, eligible device);
  * the final RunRecord (makespan/p95 as float.hex, counters, solver counts).
Runs captured: config 1 (default, five ablations, H in {0,1,3,4},
perturbations), config 3 (24 prefix-suite instances, H=3), config 2 (all 96
FATE main cells at H=4 plus the RunRecords of all 576 main cells for the
normalised table).  Configs 4/5: sampled Psi/S/tail/completion on the
canonical scenario states (paper_2605_07238_b200/scenarios.py, applied to
reference objects).

Outputs: tests/golden/<name>.json (metadata) + <name>.npz (fp64 bit patterns as
uint64).  The GPU box never runs this file; it only reads its outputs.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import wfsched.benchgen as RB  # noqa: E402
import wfsched.harness as RH  # noqa: E402
import wfsched.planner as RP  # noqa: E402
import wfsched.policies as RPol  # noqa: E402
from wfsched import executor as RE  # noqa: E402
from wfsched import state as RS  # noqa: E402
from wfsched.config import AblationFlags, default_config  # noqa: E402

from paper_2605_07238_b200 import scenarios as SC  # noqa: E402


def u64(x: float) -> int:
    return int(np.float64(x).view(np.uint64))


def record_dict(rec) -> dict:
    return {
        "method": rec.method, "workflow_id": rec.workflow_id, "family": rec.family,
        "batch_size": rec.batch_size, "seed": rec.seed, "makespan": rec.makespan.hex(),
        "p95": rec.p95_latency().hex(), "workflow_tasks": rec.workflow_tasks,
        "cross_device_parent_edges": rec.cross_device_parent_edges,
        "prefix_cache_hits_est": rec.prefix_cache_hits_est,
        "same_model_continuations": rec.same_model_continuations,
        "solver_solves": rec.solver_solves, "solver_optimal": rec.solver_optimal,
        "ablation": rec.ablation, "perturbation": rec.perturbation, "h_value": rec.h_value,
        "query_completion": {k: v.hex() for k, v in rec.query_completion.items()},
    }


class Capture:
    """Wraps FatePolicy.plan_wave and records the reference scorer outputs."""

    def __init__(self):
        self.waves = []
        self.psi, self.sched, self.compl = [], [], []

    def __enter__(self):
        self._orig = RPol.FatePolicy.plan_wave
        cap = self

        def plan_wave(policy, state, frontier, dag, cost_model):
            sids = sorted(frontier)
            n_c = 0
            if cost_model.weights.horizon != 0:
                prob = RP.build_problem(set(frontier), state, cost_model, dag)
                cap.psi.extend(u64(c.psi) for c in prob.candidates)
                n_c = len(prob.candidates)
            qids = tuple(q.query_id for q in state.instance.queries)
            n_p = 0
            for sid in sids:
                stage = dag.stages[sid]
                for dev in sorted(stage.eligible_devices):
                    cap.sched.append(u64(cost_model.sched_score(stage, dev, state, dag)))
                    t = cost_model.realized_duration(stage, [(dev, qids)], state, dag)[0]
                    wait = max(0.0, state.device_free.get(dev, 0.0) - state.clock)
                    cap.compl.append(u64(wait + t.total_s))
                    n_p += 1
            cap.waves.append({"frontier": sids, "n_cand": n_c, "n_pairs": n_p})
            return cap._orig(policy, state, frontier, dag, cost_model)

        RPol.FatePolicy.plan_wave = plan_wave
        return self

    def __exit__(self, *exc):
        RPol.FatePolicy.plan_wave = self._orig


def run_captured(instance, config):
    with Capture() as cap:
        rec = RE.run(RPol.make_policy("fate"), instance, config)
    return rec, cap


def save(name: str, runs: list, psi, sched, compl) -> None:
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump({"runs": runs}, fh, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                        psi=np.asarray(psi, dtype=np.uint64),
                        sched=np.asarray(sched, dtype=np.uint64),
                        completion=np.asarray(compl, dtype=np.uint64))
    print(f"{name}: {len(runs)} runs, {len(psi)} psi, {len(sched)} pairs")


# ---------------------------------------------------------------------------
# config 1
# ---------------------------------------------------------------------------

C1_VARIANTS = (
    {"tag": "default", "horizon": 2},
    {"tag": "h0", "horizon": 0},
    {"tag": "h1", "horizon": 1},
    {"tag": "h3", "horizon": 3},
    {"tag": "h4", "horizon": 4},
    *({"tag": f"abl_{f}", "horizon": 2, "ablation": [f]} for f in
      ("no_future_planning", "no_locality", "no_same_model", "no_prefix", "no_shard")),
    {"tag": "switch_x2", "horizon": 2, "switch_x": 2.0},
    {"tag": "transfer_x0.5", "horizon": 2, "transfer_x": 0.5},
    {"tag": "prefix_x2", "horizon": 2, "prefix_x": 2.0},
    {"tag": "state_scale1.5", "horizon": 4, "state_scale": 1.5},
)


def weights_for(base, variant: dict):
    kw = {k: v for k, v in variant.items() if k not in ("tag", "ablation")}
    if "ablation" in variant:
        kw["ablation"] = AblationFlags.from_names(variant["ablation"])
    return replace(base, **kw)


def gen_c1():
    cfg = default_config(4)
    inst = RB.lifted_instance("soykb", cfg, seed=11, batch_size=16, scale=1.0, min_groups=50)
    runs, psi, sched, compl = [], [], [], []
    for var in C1_VARIANTS:
        conf = cfg.with_weights(weights_for(cfg.weights, var))
        rec, cap = run_captured(inst, conf)
        runs.append({"variant": var, "record": record_dict(rec), "waves": cap.waves})
        psi += cap.psi
        sched += cap.sched
        compl += cap.compl
    save("c1", runs, psi, sched, compl)


# ---------------------------------------------------------------------------
# config 3
# ---------------------------------------------------------------------------


def gen_c3():
    cfg = default_config(4)
    conf = cfg.with_weights(replace(cfg.weights, horizon=3))
    runs, psi, sched, compl = [], [], [], []
    for ratio in (0.0, 0.25, 0.5, 1.0):
        for batch in (16, 32):
            suite = RB.build_prefix_suite(RB.SuiteSpec(kind="prefix_reuse", repeat_ratio=ratio,
                                                       batch_size=batch, seed=20260423), cfg)
            for k, inst in enumerate(suite):
                rec, cap = run_captured(inst, conf)
                runs.append({"ratio": ratio, "batch": batch, "shape": k,
                             "record": record_dict(rec), "waves": cap.waves})
                psi += cap.psi
                sched += cap.sched
                compl += cap.compl
    save("c3", runs, psi, sched, compl)


# ---------------------------------------------------------------------------
# config 2
# ---------------------------------------------------------------------------

_REG = {}
_CFG = None


def _c2_cell(args):
    key, method = args
    inst = _REG[key]
    if method == "fate":
        rec, cap = run_captured(inst, _CFG)
        return key, method, record_dict(rec), cap.waves, cap.psi, cap.sched, cap.compl
    rec = RE.run(RPol.make_policy(method), inst, _CFG)
    return key, method, record_dict(rec), None, [], [], []


def gen_c2(parallel: int):
    global _REG, _CFG
    man = RH.default_manifest()
    _CFG = default_config(man.num_devices)
    _REG = RH.materialize_workloads(man, _CFG)
    main_keys = sorted(k for k, inst in _REG.items()
                       if inst.dag.family not in ("prefix_reuse", "conflict"))
    cells = [(k, m) for k in main_keys for m in man.methods]
    with mp.get_context("fork").Pool(parallel) as pool:
        out = pool.map(_c2_cell, cells, chunksize=1)
    runs, psi, sched, compl, others = [], [], [], [], []
    for key, method, rec, waves, p, s, c in out:
        if method == "fate":
            inst = _REG[key]
            src = "synthetic" if inst.dag.family == "synthetic" else "lifted"
            runs.append({"key": key, "source": src, "record": rec, "waves": waves})
            psi += p
            sched += s
            compl += c
        else:
            others.append(rec)
    save("c2", runs, psi, sched, compl)
    with open(os.path.join(HERE, "c2_baselines.json"), "w") as fh:
        json.dump({"records": others, "manifest_seed": man.seeds[0]}, fh, indent=0,
                  sort_keys=True)


# ---------------------------------------------------------------------------
# configs 4 / 5 (sampled, on canonical scenario states)
# ---------------------------------------------------------------------------


def reference_kit():
    return SC.StateKit(RS.ExecutionState.initial, RS.PrefixEntry,
                       RS.ExecutionState._merge_entry, RE.partition_shards)


def _score_items(args):
    """(instance-builder key, scenario seed, [stage ids]) -> reference outputs."""
    which, idx, s, sids = args
    if which == "c4":
        cfg = SC.config_c4_catalog()
        inst = SC.c4_instance(cfg)
    else:
        cfg = SC.config_c5()
        inst = SC.c5_instance(idx, cfg)
    # rebuild the instance with the REFERENCE generator and check it matches
    if which == "c4":
        rdag = RB.synth_generate(RB.SuiteSpec(kind="synthetic", depth=100, width=100,
                                              density=0.03, seed=1, batch_size=16), cfg)
        rinst = RB.make_instance(rdag, 16, 1)
    else:
        rdag = RB.synth_generate(RB.SuiteSpec(kind="synthetic", depth=20, width=25, density=0.12,
                                              seed=1000 + idx, batch_size=16), cfg)
        rinst = RB.make_instance(rdag, 16, 1000 + idx)
    assert sorted(rinst.dag.edges) == sorted(inst.dag.edges)
    st = SC.build_scenario(rinst, cfg, s, kit=reference_kit())
    from wfsched.costs import CostModel

    cm = CostModel(cfg.models, cfg.topology, cfg.weights)
    qids = tuple(q.query_id for q in rinst.queries)
    out = []
    for sid in sids:
        stage = rinst.dag.stages[sid]
        bound = min(stage.shard_bound, len(stage.eligible_devices))
        devs = sorted(stage.eligible_devices)
        psi = [[u64(cm.plan_score(stage, k, d, st, rinst.dag)) for d in devs] for k in range(bound)]
        sched = [u64(cm.sched_score(stage, d, st, rinst.dag)) for d in devs]
        tail = [u64(cm.tail_value(stage, d, st, rinst.dag)) for d in devs]
        compl = []
        for d in devs:
            t = cm.realized_duration(stage, [(d, qids)], st, rinst.dag)[0]
            compl.append(u64(max(0.0, st.device_free.get(d, 0.0) - st.clock) + t.total_s))
        out.append({"stage": sid, "psi": psi, "sched": sched, "tail": tail, "completion": compl})
    frontier = sorted(RE.ready_set(rinst.dag, st.completed)) if hasattr(RE, "ready_set") else None
    return {"which": which, "instance": idx, "scenario": s, "items": out,
            "frontier": frontier, "clock": st.clock.hex()}


def gen_sampled(parallel: int, quick: bool):
    import random

    from wfsched.model import ready_set

    tasks = []
    # C4: 8 scenarios x (2 frontier stages + 2 sweep stages incl. completed ones)
    cfg4 = SC.config_c4_catalog()
    inst4 = SC.c4_instance(cfg4)
    all4 = sorted(inst4.dag.stages)
    for s in range(8 if not quick else 2):
        st = SC.build_scenario(inst4, cfg4, s)
        front = sorted(ready_set(inst4.dag, st.completed))
        rng = random.Random(77 + s)
        picks = rng.sample(front, 2) + rng.sample(all4, 2)
        for sid in picks:
            tasks.append(("c4", 0, s, [sid]))
    # C5: 8 instances, full frontier; plus 4 sweep stages each
    cfg5 = SC.config_c5()
    for i in range(8 if not quick else 2):
        inst = SC.c5_instance(i, cfg5)
        st = SC.build_scenario(inst, cfg5, i)
        front = sorted(ready_set(inst.dag, st.completed))
        rng = random.Random(500 + i)
        sweep = rng.sample(sorted(inst.dag.stages), 4)
        tasks.append(("c5", i, i, front + sorted(set(sweep) - set(front))))
    with mp.get_context("fork").Pool(parallel) as pool:
        results = pool.map(_score_items, tasks, chunksize=1)
    with open(os.path.join(HERE, "c45_sampled.json"), "w") as fh:
        json.dump({"samples": results}, fh, indent=0, sort_keys=True)
    n = sum(len(k) * len(k[0]) for r in results for it in r["items"] for k in [it["psi"]])
    print(f"c45_sampled: {len(results)} samples, {n} psi")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="c1,c2,c3,c45")
    ap.add_argument("--parallel", type=int, default=os.cpu_count() or 4)
    a = ap.parse_args()
    todo = a.only.split(",")
    if "c1" in todo:
        gen_c1()
    if "c3" in todo:
        gen_c3()
    if "c2" in todo:
        gen_c2(a.parallel)
    if "c45" in todo:
        gen_sampled(a.parallel, a.quick)


if __name__ == "__main__" and "--c5-assign" not in sys.argv and "--r2" not in sys.argv:
    main()


# ---------------------------------------------------------------------------
# config 5 assignments (host solve on the reference's own cost matrix)
# ---------------------------------------------------------------------------


def _c5_assign(i):
    from wfsched.costs import CostModel
    from wfsched.model import ready_set

    cfg = SC.config_c5()
    rdag = RB.synth_generate(RB.SuiteSpec(kind="synthetic", depth=20, width=25, density=0.12,
                                          seed=1000 + i, batch_size=16), cfg)
    rinst = RB.make_instance(rdag, 16, 1000 + i)
    st = SC.build_scenario(rinst, cfg, i, kit=reference_kit())
    cm = CostModel(cfg.models, cfg.topology, cfg.weights)
    front = set(ready_set(rinst.dag, st.completed))
    prob = RP.build_problem(front, st, cm, rinst.dag)
    sol = RP.solve_frontier(prob, budget_s=0.0)
    return {"instance": i, "selected": [list(x) for x in sol.selected],
            "objective": sol.objective.hex(), "n_candidates": len(prob.candidates)}


def gen_c5_assign(parallel: int, n: int = 16):
    with mp.get_context("fork").Pool(parallel) as pool:
        res = pool.map(_c5_assign, list(range(n)), chunksize=1)
    with open(os.path.join(HERE, "c5_assign.json"), "w") as fh:
        json.dump({"budget_s": 0.0, "instances": res}, fh, indent=0, sort_keys=True)
    print(f"c5_assign: {len(res)} instances")


if __name__ == "__main__" and "--c5-assign" in sys.argv:
    gen_c5_assign(os.cpu_count() or 4)


# ---------------------------------------------------------------------------
# round 2: SURVEY §8(d) parity gates at full size
# ---------------------------------------------------------------------------
# * c5_full: every frontier candidate of 64 config-5 instances spread over the
#   bench's 4096 (i = 0, 64, ..., 4032): Psi in FrontierProblem order, S and
#   completion per (sorted stage, sorted eligible device), and the budget-0
#   assignment of the reference's own solve (planner.py:150-234);
# * c4_assign: the same for the frontier of all 8 canonical config-4 scenarios
#   (frontier mode, ~11.3k Psi each), scored in stage chunks across processes;
# * c3_base: halo / kvflow / roundrobin RunRecords of the 24 prefix-suite
#   instances at H=3, so the normalised C3 table can be recomputed from
#   GPU-run FATE records.

C5_FULL = tuple(range(0, 4096, 64))


def _ref_c5(i):
    cfg = SC.config_c5()
    rdag = RB.synth_generate(RB.SuiteSpec(kind="synthetic", depth=20, width=25, density=0.12,
                                          seed=1000 + i, batch_size=16), cfg)
    return cfg, RB.make_instance(rdag, 16, 1000 + i)


def _ref_c4():
    cfg = SC.config_c4_catalog()
    rdag = RB.synth_generate(RB.SuiteSpec(kind="synthetic", depth=100, width=100,
                                          density=0.03, seed=1, batch_size=16), cfg)
    return cfg, RB.make_instance(rdag, 16, 1)


def _pairs(cm, st, dag, sids):
    """S and completion per (sorted stage, sorted eligible device)."""
    qids = tuple(q.query_id for q in st.instance.queries)
    sched, compl = [], []
    for sid in sids:
        stage = dag.stages[sid]
        for d in sorted(stage.eligible_devices):
            sched.append(u64(cm.sched_score(stage, d, st, dag)))
            t = cm.realized_duration(stage, [(d, qids)], st, dag)[0]
            compl.append(u64(max(0.0, st.device_free.get(d, 0.0) - st.clock) + t.total_s))
    return sched, compl


def _c5_full_one(i):
    from wfsched.costs import CostModel
    from wfsched.model import ready_set

    cfg, rinst = _ref_c5(i)
    st = SC.build_scenario(rinst, cfg, i, kit=reference_kit())
    cm = CostModel(cfg.models, cfg.topology, cfg.weights)
    sids = sorted(ready_set(rinst.dag, st.completed))
    prob = RP.build_problem(set(sids), st, cm, rinst.dag)
    sol = RP.solve_frontier(prob, budget_s=0.0)
    sched, compl = _pairs(cm, st, rinst.dag, sids)
    return ({"instance": i, "frontier": sids, "n_cand": len(prob.candidates),
             "n_pairs": len(sched), "selected": [list(x) for x in sol.selected],
             "objective": sol.objective.hex(), "optimal": sol.optimal},
            [u64(c.psi) for c in prob.candidates], sched, compl)


def gen_c5_full(parallel: int):
    with mp.get_context("fork").Pool(parallel) as pool:
        res = pool.map(_c5_full_one, list(C5_FULL), chunksize=1)
    meta = [r[0] for r in res]
    psi = [x for r in res for x in r[1]]
    sched = [x for r in res for x in r[2]]
    compl = [x for r in res for x in r[3]]
    with open(os.path.join(HERE, "c5_full.json"), "w") as fh:
        json.dump({"budget_s": 0.0, "instances": meta}, fh, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "c5_full.npz"), psi=np.asarray(psi, np.uint64),
                        sched=np.asarray(sched, np.uint64), completion=np.asarray(compl, np.uint64))
    print(f"c5_full: {len(meta)} instances, {len(psi)} psi, {len(sched)} pairs")


_C4 = {}


def _c4_chunk(args):
    """Reference Psi / S / completion of a slice of one scenario's frontier."""
    from wfsched.costs import CostModel

    s, sids = args
    if "inst" not in _C4:
        _C4["cfg"], _C4["inst"] = _ref_c4()
    cfg, rinst = _C4["cfg"], _C4["inst"]
    st = SC.build_scenario(rinst, cfg, s, kit=reference_kit())
    cm = CostModel(cfg.models, cfg.topology, cfg.weights)
    dag = rinst.dag
    psi = []
    for sid in sids:  # build_problem's loop order (planner.py:83-97)
        stage = dag.stages[sid]
        bound = 1 if cfg.weights.ablation.no_shard else min(stage.shard_bound,
                                                            len(stage.eligible_devices))
        for k in range(bound):
            for d in sorted(stage.eligible_devices):
                psi.append(cm.plan_score(stage, k, d, st, dag))
    sched, compl = _pairs(cm, st, dag, sids)
    return s, sids, psi, sched, compl


def gen_c4_assign(parallel: int, n_scen: int = 8, chunk: int = 4):
    from wfsched.costs import CostModel
    from wfsched.model import ready_set

    cfg, rinst = _ref_c4()
    tasks, fronts = [], {}
    for s in range(n_scen):
        st = SC.build_scenario(rinst, cfg, s, kit=reference_kit())
        fronts[s] = sorted(ready_set(rinst.dag, st.completed))
        tasks += [(s, fronts[s][j: j + chunk]) for j in range(0, len(fronts[s]), chunk)]
    with mp.get_context("fork").Pool(parallel) as pool:
        out = pool.map(_c4_chunk, tasks, chunksize=1)
    meta, psi_all, sched_all, compl_all = [], [], [], []
    for s in range(n_scen):
        parts = [o for o in out if o[0] == s]
        psi = [x for o in parts for x in o[2]]
        st = SC.build_scenario(rinst, cfg, s, kit=reference_kit())
        cm = CostModel(cfg.models, cfg.topology, cfg.weights)
        # the reference's own FrontierProblem from the reference's Psi values
        cands, it = [], iter(psi)
        bounds = {}
        for sid in fronts[s]:
            stage = rinst.dag.stages[sid]
            bounds[sid] = min(stage.shard_bound, len(stage.eligible_devices))
            for k in range(bounds[sid]):
                for d in sorted(stage.eligible_devices):
                    cands.append(RP.Candidate(sid, k, d, next(it)))
        prob = RP.FrontierProblem(tuple(cands), bounds, cfg.topology.device_ids)
        sol = RP.solve_frontier(prob, budget_s=0.0)
        meta.append({"scenario": s, "frontier": fronts[s], "n_cand": len(cands),
                     "n_pairs": sum(len(o[3]) for o in parts), "clock": st.clock.hex(),
                     "selected": [list(x) for x in sol.selected],
                     "objective": sol.objective.hex(), "optimal": sol.optimal})
        psi_all += [u64(x) for x in psi]
        sched_all += [x for o in parts for x in o[3]]
        compl_all += [x for o in parts for x in o[4]]
        del cm
    with open(os.path.join(HERE, "c4_assign.json"), "w") as fh:
        json.dump({"budget_s": 0.0, "scenarios": meta}, fh, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "c4_assign.npz"), psi=np.asarray(psi_all, np.uint64),
                        sched=np.asarray(sched_all, np.uint64),
                        completion=np.asarray(compl_all, np.uint64))
    print(f"c4_assign: {len(meta)} scenarios, {len(psi_all)} psi")


def _c3_base_cell(args):
    ratio, batch, k, method = args
    cfg = default_config(4)
    conf = cfg.with_weights(replace(cfg.weights, horizon=3))
    suite = RB.build_prefix_suite(RB.SuiteSpec(kind="prefix_reuse", repeat_ratio=ratio,
                                               batch_size=batch, seed=20260423), cfg)
    rec = RE.run(RPol.make_policy(method), suite[k], conf)
    d = record_dict(rec)
    d.update({"ratio": ratio, "batch": batch, "shape": k})
    return d


def gen_c3_base(parallel: int):
    cells = [(r, b, k, m) for r in (0.0, 0.25, 0.5, 1.0) for b in (16, 32) for k in range(3)
             for m in ("halo", "kvflow", "roundrobin")]
    with mp.get_context("fork").Pool(parallel) as pool:
        recs = pool.map(_c3_base_cell, cells, chunksize=1)
    with open(os.path.join(HERE, "c3_baselines.json"), "w") as fh:
        json.dump({"horizon": 3, "records": recs}, fh, indent=0, sort_keys=True)
    print(f"c3_baselines: {len(recs)} records")


if __name__ == "__main__" and "--r2" in sys.argv:
    _which = sys.argv[sys.argv.index("--r2") + 1].split(",")
    _par = os.cpu_count() or 4
    if "c3base" in _which:
        gen_c3_base(_par)
    if "c5full" in _which:
        gen_c5_full(_par)
    if "c4assign" in _which:
        gen_c4_assign(_par)
