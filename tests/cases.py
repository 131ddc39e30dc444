"""Shared test cases: (bank, weights, states, work).  Instances come from the
package's generator mirror (wf/workloads, bit-identical to the reference's,
tests/test_reference_mirror.py); execution states are the reference's own
``wfsched.state.ExecutionState``."""

from __future__ import annotations

import random
from dataclasses import replace

import numpy as np

from paper_2605_07238_b200 import pack, scenarios
from paper_2605_07238_b200.wf import workloads as W
from paper_2605_07238_b200.wf.dagmodel import (
    DeviceSpec, DeviceTopology, Query, Stage, WorkflowDag, WorkflowInstance, annotate_topology,
)
from wfsched.state import ExecutionState, PrefixEntry
from paper_2605_07238_b200.wf.weights import AblationFlags, ScoreWeights, default_config


class Case:
    def __init__(self, name, instances, cfg, weights, scen_states, items):
        self.name = name
        self.instances = instances
        self.cfg = cfg
        self.weights = weights
        self.bank = pack.pack_bank(instances, cfg.models, cfg.topology)
        self.states = pack.pack_states(self.bank, scen_states)
        self.work = pack.make_work(self.bank, items, weights.ablation.no_shard)
        self.wrec = pack.weights_record(weights)

    def __repr__(self):
        return f"Case({self.name}, items={self.work.n_items}, psi={self.work.n_psi})"


def bits(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    out = a.view(np.uint64).copy()
    out[np.isnan(a)] = np.uint64(0x7FF8000000000000)
    return out


def c4_case(scen=(0,), sweep_stride: int | None = None, frontier: bool = True):
    cfg = scenarios.config_c4_catalog()
    inst = scenarios.c4_instance(cfg)
    states, items = [], []
    bank_tmp = pack.pack_bank([inst], cfg.models, cfg.topology)
    for j, s in enumerate(scen):
        st = scenarios.build_scenario(inst, cfg, s)
        states.append((0, st))
        if frontier:
            items += [(j, bank_tmp.global_index(0, sid)) for sid in scenarios.scenario_frontier(inst, st)]
        if sweep_stride:
            items += [(j, g) for g in range(0, bank_tmp.n_stages, sweep_stride)]
    return Case(f"c4{tuple(scen)}", [inst], cfg, cfg.weights, states, items)


def c5_case(n_inst: int = 4, first: int = 0, sweep: bool = False):
    cfg = scenarios.config_c5()
    insts = [scenarios.c5_instance(first + i, cfg) for i in range(n_inst)]
    bank_tmp = pack.pack_bank(insts, cfg.models, cfg.topology)
    states, items = [], []
    for j, inst in enumerate(insts):
        st = scenarios.build_scenario(inst, cfg, first + j)
        states.append((j, st))
        if sweep:
            items += [(j, bank_tmp.global_index(j, sid)) for sid in sorted(inst.dag.stages)]
        else:
            items += [(j, bank_tmp.global_index(j, sid))
                      for sid in scenarios.scenario_frontier(inst, st)]
    return Case(f"c5x{n_inst}", insts, cfg, cfg.weights, states, items)


def small_case(weights=None, num_devices=4, family="soykb", seed=11, scen_seeds=(0, 1, 2),
               prefix=False):
    """Lifted or prefix-suite instance + several scenario states, all stages."""
    cfg = default_config(num_devices)
    weights = weights or replace(cfg.weights, horizon=3)
    if prefix:
        insts = W.build_prefix_suite(W.SuiteSpec(kind="prefix_reuse", repeat_ratio=0.5,
                                                 batch_size=16, seed=20260423), cfg)
    else:
        insts = [W.lifted_instance(family, cfg, seed=seed, batch_size=16, scale=1.0,
                                   min_groups=50)]
    bank_tmp = pack.pack_bank(insts, cfg.models, cfg.topology)
    states, items = [], []
    for ii, inst in enumerate(insts):
        for s in scen_seeds:
            st = scenarios.build_scenario(inst, cfg, s)
            states.append((ii, st))
            j = len(states) - 1
            items += [(j, bank_tmp.global_index(ii, sid)) for sid in sorted(inst.dag.stages)]
    return Case(f"small-{family}-{prefix}", insts, cfg, weights, states, items)


def edge_case(seed: int = 7, horizon: int = 4, ablation=None, overrides=True):
    """Hand-built DAG exercising the rarely-taken branches: transfer
    overrides, per-device speeds, base_cost_override, restricted and empty
    eligibility, shard bounds > 2, stages without model / role / group, query
    prefix groups, prefix entries under foreign or empty-string models, sticky
    entries, busy and idle devices."""
    rng = random.Random(seed)
    cfg = default_config(6)
    devs = [DeviceSpec(id=f"d{i}", speed_factor=[1.0, 1.25, 0.8, 1.0, 2.0, 0.5][i])
            for i in range(6)]
    over = {}
    if overrides:
        for a in range(6):
            for b in range(6):
                if a != b and rng.random() < 0.4:
                    over[(f"d{a}", f"d{b}")] = rng.choice([0.5, 1.5, 3.0, 0.0])
    topo = DeviceTopology(devices=tuple(devs), default_transfer_coeff=2.0, transfer_overrides=over)
    models = cfg.models
    aliases = sorted(models)
    roles = list(cfg.roles.values())
    ids = [f"e{i:02d}" for i in range(18)]
    levels = [ids[0:3], ids[3:7], ids[7:11], ids[11:15], ids[15:18]]
    edges = set()
    for li in range(1, len(levels)):
        for v in levels[li]:
            ups = [u for u in levels[li - 1] if rng.random() < 0.6] or [levels[li - 1][0]]
            edges.update((u, v) for u in ups)
            if li >= 2 and rng.random() < 0.3:
                edges.add((rng.choice(levels[li - 2]), v))
    stages = {}
    for i, sid in enumerate(ids):
        role = None if i % 7 == 3 else roles[i % len(roles)]
        model = None if i % 9 == 4 else aliases[i % 3]
        if i % 5 == 2:
            elig = frozenset(f"d{j}" for j in range(6) if (i + j) % 3)
        else:
            elig = frozenset(f"d{j}" for j in range(6))
        if i == 16:
            elig = frozenset()  # _mean_base falls back to all devices in topology order
        shard = 1 if (role is not None and not role.shard_eligible) else [1, 2, 3, 4][i % 4]
        group = None if i % 4 == 1 else ("pg:shared" if i % 3 else f"pg:{model}")
        ov = {"d1": 3.5, "d4": 0.25} if i % 6 == 5 else None
        stages[sid] = Stage(id=sid, model=model, eligible_devices=elig, shard_bound=shard,
                            role=role, prompt_token_proxy=rng.choice([0, 128, 512, 1024]),
                            output_token_proxy=rng.choice([0, 128, 384, 640]),
                            shared_prefix_group=group, keep_cache=bool(i % 2),
                            cache_reuse=bool(i % 3), base_cost_override=ov)
    dag = annotate_topology(WorkflowDag("edge", "edge", stages, frozenset(edges)))
    queries = tuple(Query(f"q{i:03d}", 100 + rng.randrange(900),
                          None if i % 3 == 0 else f"qg{i % 4}") for i in range(13))
    inst = WorkflowInstance(dag=dag, queries=queries, batch_size=13,
                            prefix_groups={"qg1": 300, "qg2": 2000})
    weights = replace(ScoreWeights(), horizon=horizon, switch_x=1.5, transfer_x=0.75,
                      prefix_x=2.0, state_scale=1.25, locality_scale=0.5, prefix_scale=1.5,
                      ablation=ablation or AblationFlags())
    states = []
    for s in range(4):
        st = ExecutionState.initial(inst, topo.device_ids)
        st.clock = 100.0 * s
        r2 = random.Random(1000 + s)
        for sid in sorted(ids)[: 3 + 4 * s]:
            d1, d2 = r2.sample([f"d{j}" for j in range(6)], 2)
            qids = tuple(q.query_id for q in queries)
            if r2.random() < 0.5:
                st.parent_loc[sid] = ((d1, qids[:7]), (d2, qids[7:]))
            else:
                st.parent_loc[sid] = ((d1, qids),)
            st.completed.add(sid)
        for j in range(6):
            d = f"d{j}"
            st.residency[d] = r2.choice([None] + aliases)
            st.device_free[d] = st.clock + r2.choice([-5.0, 0.0, 1e-13, 3.0, 12.5])
            store = st.prefix_store[d]
            for g in r2.sample(["pg:shared", "pg:qwen-7b", "qg1", "qg2", "qg3", "other"], 3):
                store[g] = PrefixEntry(g, r2.choice([50, 400, 5000]),
                                       r2.choice(aliases + [""]), sticky=r2.random() < 0.5)
        states.append((0, st))
    bank_tmp = pack.pack_bank([inst], models, topo)
    items = [(j, bank_tmp.global_index(0, sid)) for j in range(len(states)) for sid in ids]

    class _Cfg:
        pass

    c = _Cfg()
    c.models, c.topology = models, topo
    return Case(f"edge-h{horizon}", [inst], c, weights, states, items)


def token_case(seed: int = 3, horizon: int = 3):
    """Uniform speeds, no query prefix groups, one big prefix group whose
    keep_cache stages have five distinct prompts, and prefix entries whose
    token counts are those prompts, other counts, or under other models: every
    kind of class the kernel's partial-hit tables (tok_vals/tok_sums) see --
    tabulated, beyond the three tabulated values, untabulated counts, full
    hits, misses -- next to shard bounds 1-3."""
    rng = random.Random(seed)
    cfg = default_config(6)
    topo = cfg.topology
    models = cfg.models
    aliases = sorted(models)
    roles = list(cfg.roles.values())
    ids = [f"t{i:02d}" for i in range(24)]
    levels = [ids[0:6], ids[6:12], ids[12:18], ids[18:24]]
    edges = set()
    for li in range(1, len(levels)):
        for v in levels[li]:
            ups = [u for u in levels[li - 1] if rng.random() < 0.5] or [levels[li - 1][0]]
            edges.update((u, v) for u in ups)
    prompts = [100, 200, 300, 400, 500]
    stages = {}
    for i, sid in enumerate(ids):
        role = roles[i % len(roles)]
        shard = 1 if not role.shard_eligible else [1, 2, 3][i % 3]
        stages[sid] = Stage(id=sid, model=aliases[i % 2], eligible_devices=frozenset(topo.device_ids),
                            shard_bound=shard, role=role,
                            prompt_token_proxy=prompts[i % 5] + (0 if i % 7 else 100),
                            output_token_proxy=rng.choice([128, 384]),
                            shared_prefix_group="pg" if i % 6 else "other",
                            keep_cache=bool(i % 2 == 0 or i % 5 == 3), cache_reuse=True)
    dag = annotate_topology(WorkflowDag("tok", "tok", stages, frozenset(edges)))
    queries = tuple(Query(f"q{i:03d}", 100 + rng.randrange(700), None) for i in range(16))
    inst = WorkflowInstance(dag=dag, queries=queries, batch_size=16, prefix_groups={})
    weights = replace(cfg.weights, horizon=horizon)
    states = []
    for s in range(5):
        st = ExecutionState.initial(inst, topo.device_ids)
        st.clock = 50.0 * s
        r2 = random.Random(500 + s)
        for sid in sorted(ids)[: 4 * s]:
            st.parent_loc[sid] = ((r2.choice(topo.device_ids), tuple(q.query_id for q in queries)),)
            st.completed.add(sid)
        for d in topo.device_ids:
            st.residency[d] = r2.choice(aliases)
            st.device_free[d] = st.clock + r2.choice([-5.0, 0.0, 4.0])
            store = st.prefix_store[d]
            tok = r2.choice([100, 200, 300, 400, 500, 600, 250, 1000])
            store["pg"] = PrefixEntry("pg", tok, r2.choice(aliases), sticky=r2.random() < 0.5)
            if r2.random() < 0.5:
                store["other"] = PrefixEntry("other", r2.choice([100, 300]), r2.choice(aliases))
        states.append((0, st))
    bank_tmp = pack.pack_bank([inst], models, topo)
    items = [(j, bank_tmp.global_index(0, sid)) for j in range(len(states)) for sid in ids]
    return Case(f"tok-h{horizon}", [inst], cfg, weights, states, items)


ALL_ABLATIONS = ("no_future_planning", "no_locality", "no_same_model", "no_prefix", "no_shard")


def wide_case(n_dev: int, n_queries: int, kappa: int, overrides: bool, horizon: int = 4,
              seed: int = 11, n_stages: int = 30, uniform_speed: bool = False,
              n_scen: int = 3, qgroups: bool = True):
    """Random layered DAG at the ABI's size limits: up to 64 devices (one or
    two device slots per lane, the 32/33 boundary), query batches past the
    static 16-query layout up to MAX_QUERIES, up to MAX_KAPPA prefix entries
    per device, eight models (displacement masks), transfer overrides on or
    off, shard bounds 1-4, restricted and empty eligibility."""
    rng = random.Random(seed)
    cat = scenarios.config_c4_catalog()
    models = cat.models
    aliases = sorted(models)
    roles = list(cat.roles.values())
    devs = [DeviceSpec(id=f"w{i:02d}", speed_factor=1.0 if uniform_speed else
                       rng.choice([0.5, 0.8, 1.0, 1.25, 2.0])) for i in range(n_dev)]
    dev_ids = [d.id for d in devs]
    over = {}
    if overrides:
        for a in dev_ids:
            for b in rng.sample(dev_ids, min(3, n_dev)):
                if a != b:
                    over[(a, b)] = rng.choice([0.5, 1.5, 3.0, 0.0])
    topo = DeviceTopology(devices=tuple(devs), default_transfer_coeff=2.0,
                          transfer_overrides=over)
    ids = [f"s{i:03d}" for i in range(n_stages)]
    width = 5
    levels = [ids[i:i + width] for i in range(0, n_stages, width)]
    edges = set()
    for li in range(1, len(levels)):
        for v in levels[li]:
            ups = [u for u in levels[li - 1] if rng.random() < 0.5] or [levels[li - 1][0]]
            edges.update((u, v) for u in ups)
            if li >= 2 and rng.random() < 0.4:
                edges.add((rng.choice(levels[li - 2]), v))
    groups = ["pg0", "pg1", "pg2", None]
    stages = {}
    for i, sid in enumerate(ids):
        role = None if i % 11 == 5 else roles[i % len(roles)]
        if i % 7 == 3:
            elig = frozenset(rng.sample(dev_ids, max(1, n_dev // 2)))
        else:
            elig = frozenset(dev_ids)
        if i == n_stages - 2:
            elig = frozenset()
        shard = 1 if (role is not None and not role.shard_eligible) else 1 + i % 4
        stages[sid] = Stage(id=sid, model=None if i % 13 == 6 else aliases[i % len(aliases)],
                            eligible_devices=elig, shard_bound=shard, role=role,
                            prompt_token_proxy=rng.choice([0, 256, 512, 768, 1024]),
                            output_token_proxy=rng.choice([0, 128, 384, 640]),
                            shared_prefix_group=groups[i % 4], keep_cache=bool(i % 2),
                            cache_reuse=bool(i % 3))
    dag = annotate_topology(WorkflowDag("wide", "wide", stages, frozenset(edges)))
    qg_names = ["qa", "qb", "pg1", None] if qgroups else [None]
    queries = tuple(Query(f"q{i:03d}", 50 + rng.randrange(950), qg_names[i % len(qg_names)])
                    for i in range(n_queries))
    inst = WorkflowInstance(dag=dag, queries=queries, batch_size=n_queries,
                            prefix_groups={"qa": 100, "qb": 700})
    weights = replace(ScoreWeights(), horizon=horizon, switch_x=1.25, transfer_x=0.5,
                      prefix_x=1.5, state_scale=0.75, locality_scale=1.5)
    kgroups = ["pg0", "pg1", "pg2", "qa", "qb"] + [f"x{k}" for k in range(max(0, kappa - 5))]
    states = []
    for s in range(n_scen):
        st = ExecutionState.initial(inst, topo.device_ids)
        st.clock = 10.0 + 40.0 * s
        r2 = random.Random(seed * 100 + s)
        for sid in sorted(ids)[: width * (s + 1)]:
            d1, d2 = r2.sample(dev_ids, 2) if n_dev > 1 else (dev_ids[0], dev_ids[0])
            qids = tuple(q.query_id for q in queries)
            if n_dev > 1 and r2.random() < 0.3 and len(qids) > 1:
                h = len(qids) // 2
                st.parent_loc[sid] = ((d1, qids[:h]), (d2, qids[h:]))
            else:
                st.parent_loc[sid] = ((d1, qids),)
            st.completed.add(sid)
        for d in dev_ids:
            st.residency[d] = r2.choice([None] + aliases)
            st.device_free[d] = st.clock + r2.choice([-5.0, 0.0, 1e-13, 3.0, 12.5])
            store = st.prefix_store[d]
            for g in r2.sample(kgroups, r2.randint(0, kappa)) if d != dev_ids[0] else kgroups[:kappa]:
                store[g] = PrefixEntry(g, r2.choice([30, 256, 400, 5000]),
                                       r2.choice(aliases + [""]), sticky=r2.random() < 0.5)
        states.append((0, st))
    bank_tmp = pack.pack_bank([inst], models, topo)
    items = [(j, bank_tmp.global_index(0, sid)) for j in range(len(states)) for sid in ids]

    class _Cfg:
        pass

    c = _Cfg()
    c.models, c.topology = models, topo
    return Case(f"wide-d{n_dev}-b{n_queries}-k{kappa}-o{int(overrides)}-h{horizon}", [inst], c,
                weights, states, items)
