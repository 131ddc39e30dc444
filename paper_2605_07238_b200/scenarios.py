"""Canonical configs 1-5 and the deterministic scenario-state generator.

Config definitions follow ``BASELINE.json``'s ``configs`` and SURVEY.md §8(d):

* C1  ``lifted_instance("soykb", default_config(4), seed=11, batch_size=16,
  scale=1.0, min_groups=50)``, horizon 2, full FATE run;
* C2  the reference default manifest (``harness.py:182-200``), horizon 4;
* C3  ``build_prefix_suite`` at ratios {0, .25, .5, 1} x batch {16, 32}, horizon 3;
* C4  ``synth_generate(depth=100, width=100, density=0.03, seed=1)`` on 64
  devices with 8 model types, horizon 4, scenario states s = 0..S-1;
* C5  4096 x ``synth_generate(depth=20, width=25, density=0.12, seed=1000+i)``
  on 32 devices, horizon 3, one scenario per instance (s = i).

The scenario generator builds a *real* execution state (so the reference
``CostModel`` consumes it directly): stages below a hashed level ``L`` are
completed on hashed devices (2-way sharded when hashed so), their prefix
entries seeded exactly as the reference's ``_seed_prefixes`` would
(``state.py:236-261``), then each device gets a hashed resident model (with the
reference eviction rule, ``state.py:224-234``) and a hashed free time.  It is
written against a small "kit" of state primitives (by default the caller's
``wfsched``: the states are real reference ``ExecutionState`` objects).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

from .wf.dagmodel import ModelProfile, ready_set
from .wf.weights import ScoreWeights, default_config
from .wf.workloads import SuiteSpec, make_instance, stable_hash64, synth_generate


@dataclass(frozen=True)
class StateKit:
    """State primitives: the reference's or the mirror's."""

    initial: object          # ExecutionState.initial
    prefix_entry: object     # PrefixEntry constructor
    merge_entry: object      # _merge_entry(store, entry)
    partition_shards: object  # executor.partition_shards


def reference_kit() -> StateKit:
    """The caller's ``wfsched`` state primitives (``state.py:26-272``,
    ``executor.py:86-108``)."""
    from wfsched.executor import partition_shards
    from wfsched.state import ExecutionState, PrefixEntry

    return StateKit(ExecutionState.initial, PrefixEntry, ExecutionState._merge_entry,
                    partition_shards)


# ---------------------------------------------------------------------------
# configs
# ---------------------------------------------------------------------------


def config_c4_catalog():
    """``default_config(64)`` + models m0-7b..m4-7b; every role may use all 8
    aliases (sorted)."""
    cfg = default_config(64)
    models = dict(cfg.models)
    for i in range(5):
        alias = f"m{i}-7b"
        models[alias] = ModelProfile(alias, memory_gb=15.0, prefill_coeff=0.7 + 0.05 * i,
                                     decode_coeff=0.001 + 0.0001 * i, switch_penalty=10.0 + i)
    everyone = tuple(sorted(models))
    return replace(cfg, models=models, role_models={k: everyone for k in cfg.role_models},
                   weights=replace(ScoreWeights(), horizon=4))


def c4_instance(cfg=None):
    cfg = cfg or config_c4_catalog()
    dag = synth_generate(SuiteSpec(kind="synthetic", depth=100, width=100, density=0.03,
                                   seed=1, batch_size=16), cfg)
    return make_instance(dag, 16, 1)


def config_c5():
    cfg = default_config(32)
    return cfg.with_weights(replace(cfg.weights, horizon=3))


def c5_spec(i: int) -> SuiteSpec:
    return SuiteSpec(kind="synthetic", depth=20, width=25, density=0.12, seed=1000 + i,
                     batch_size=16)


def c5_instance(i: int, cfg=None):
    cfg = cfg or config_c5()
    return make_instance(synth_generate(c5_spec(i), cfg), 16, 1000 + i)


# ---------------------------------------------------------------------------
# scenario states
# ---------------------------------------------------------------------------


def build_scenario(instance, cfg, s: int, kit: StateKit | None = None):
    """Deterministic mid-run state for scenario seed ``s``."""
    kit = kit or reference_kit()
    dag = instance.dag
    devs = sorted(cfg.topology.device_ids)
    n_dev = len(devs)
    models = sorted(cfg.models)
    wid = dag.workflow_id
    st = kit.initial(instance, cfg.topology.device_ids)
    top = dag.annotations.max_level
    cut = 1 + stable_hash64(wid, "L", s) % max(top, 1)
    st.clock = 1000.0 * cut
    qids = tuple(q.query_id for q in instance.queries)
    qmap = {q.query_id: q for q in instance.queries}
    levels = dag.annotations.level
    for sid in sorted(dag.stages):
        if levels[sid] >= cut:
            continue
        stage = dag.stages[sid]
        h = stable_hash64(wid, "loc", sid, s)
        first = devs[h % n_dev]
        if stage.shard_bound == 2 and (h >> 8) & 1:
            shards = kit.partition_shards(stage, [first, devs[(h % n_dev + 1) % n_dev]], qids)
        else:
            shards = [(first, qids)]
        st.parent_loc[sid] = tuple(sorted(shards))
        st.completed.add(sid)
        model = stage.model or ""
        for dev, shard_q in shards:
            store = st.prefix_store[dev]
            if stage.keep_cache and stage.shared_prefix_group is not None:
                kit.merge_entry(store, kit.prefix_entry(
                    group=stage.shared_prefix_group, tokens=stage.prompt_token_proxy,
                    model=model, sticky=True))
            for qid in shard_q:
                q = qmap[qid]
                if q.prefix_group is None:
                    continue
                kit.merge_entry(store, kit.prefix_entry(
                    group=q.prefix_group, tokens=int(instance.prefix_groups.get(
                        q.prefix_group, q.prompt_tokens)),
                    model=model, sticky=stage.keep_cache))
    for dev in devs:
        h = stable_hash64(wid, "dev", dev, s)
        model = models[h % len(models)]
        st._evict_on_switch(dev, model)
        st.residency[dev] = model
        st.device_free[dev] = st.clock + 12.5 * ((h >> 8) % 4) if (h >> 16) & 1 else st.clock - 5.0
    return st


def scenario_frontier(instance, state) -> list:
    return sorted(ready_set(instance.dag, state.completed))
