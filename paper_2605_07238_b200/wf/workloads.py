"""Workload generators for configs 1-5 (host side, deterministic).

Restates the reference generators (``pkg/src/wfsched/benchgen.py`` and
``hashutil.py``) so the canonical instances can be rebuilt on a GPU box where
the reference package is absent.  Every function is a pure function of its
arguments and produces the same DAGs, queries and ids as the reference
(checked against the reference in ``tests/test_workloads.py`` when it is
importable).  Structure differs from the reference: graph bookkeeping uses
indexed adjacency and heaps instead of repeated edge scans.
"""

from __future__ import annotations

import heapq
import json
import math
import random
import re
from dataclasses import dataclass, replace

from .dagmodel import (
    Query, Stage, WorkflowDag, WorkflowInstance, annotate_topology, validate_dag,
)
from .weights import DEFAULT_SEED

# ---------------------------------------------------------------------------
# Stable hashing (reference hashutil.py:15-29): FNV-1a 64 over "a|b|c" UTF-8
# ---------------------------------------------------------------------------

_FNV_BASIS = 0xCBF29CE484222325
_FNV_MUL = 0x100000001B3
_U64 = (1 << 64) - 1


def stable_hash64(*parts) -> int:
    h = _FNV_BASIS
    for byte in "|".join(map(str, parts)).encode("utf-8"):
        h = ((h ^ byte) * _FNV_MUL) & _U64
    return h


def stable_choice(options, *parts):
    if not options:
        raise ValueError("stable_choice requires a nonempty option list")
    return options[stable_hash64(*parts) % len(options)]


def stable_hash64_many(keys) -> list:
    """FNV-1a of many strings at once (numpy, grouped by byte length)."""
    import numpy as np

    enc = [k.encode("utf-8") for k in keys]
    out = np.zeros(len(enc), dtype=np.uint64)
    by_len: dict = {}
    for i, b in enumerate(enc):
        by_len.setdefault(len(b), []).append(i)
    mul = np.uint64(_FNV_MUL)
    for n, rows in by_len.items():
        rows_a = np.asarray(rows, dtype=np.int64)
        mat = np.frombuffer(b"".join(enc[i] for i in rows), dtype=np.uint8).reshape(len(rows), n)
        h = np.full(len(rows), _FNV_BASIS, dtype=np.uint64)
        with np.errstate(over="ignore"):
            for col in range(n):
                h = (h ^ mat[:, col].astype(np.uint64)) * mul
        out[rows_a] = h
    return [int(x) for x in out]


# ---------------------------------------------------------------------------
# Specs
# ---------------------------------------------------------------------------

EARLY_ROLES = ("prompt_prep", "retrieval", "routing", "decomposition")
MERGE_ROLES = ("merge", "aggregation")
LATE_ROLES = ("summarization", "validation", "verification", "final_synthesis")


class BenchgenError(ValueError):
    pass


@dataclass(frozen=True)
class RawTaskDag:
    tasks: tuple
    source_file: str = "<inline>"


@dataclass(frozen=True)
class LiftParams:
    max_stages: int = 64
    min_groups: int = 12
    seed: int = DEFAULT_SEED
    family: str = "unknown"
    prefix_collapse: bool = True

    def __post_init__(self) -> None:
        if self.max_stages < 1:
            raise ValueError("max_stages must be >= 1")


@dataclass(frozen=True)
class SuiteSpec:
    kind: str
    repeat_ratio: float = 0.0
    prefix_length: int = 2000
    chain_length: int = 12
    width: int = 3
    depth: int = 4
    density: float = 0.5
    group_size: int = 4
    batch_size: int = 16
    seed: int = DEFAULT_SEED

    def __post_init__(self) -> None:
        if not 0.0 <= self.repeat_ratio <= 1.0:
            raise ValueError("repeat_ratio must lie in [0, 1]")


# ---------------------------------------------------------------------------
# Raw workflow documents (reference benchgen.py:83-157, 403-513)
# ---------------------------------------------------------------------------


def import_workflow_json(document: str, source_file: str = "<inline>") -> RawTaskDag:
    try:
        doc = json.loads(document)
    except json.JSONDecodeError as exc:
        raise BenchgenError(f"{source_file}: malformed JSON at line {exc.lineno}, "
                            f"column {exc.colno}: {exc.msg}") from exc
    if not isinstance(doc, dict):
        raise BenchgenError(f"{source_file}: top-level JSON value must be an object")
    box = doc["workflow"] if isinstance(doc.get("workflow"), dict) else doc
    listing = next((box[k] for k in ("tasks", "jobs", "nodes") if isinstance(box.get(k), list)),
                   None)
    if listing is None:
        raise BenchgenError(f"{source_file}: no tasks/jobs/nodes list found")
    tasks = []
    seen: set = set()
    for pos, item in enumerate(listing):
        if not isinstance(item, dict):
            raise BenchgenError(f"{source_file}: task #{pos} is not an object")
        name = item.get("name") or item.get("id")
        if not name:
            raise BenchgenError(f"{source_file}: task #{pos} has no name")
        ups = item.get("parents") or item.get("parentNames") or []
        if not isinstance(ups, list):
            raise BenchgenError(f"{source_file}: task {name}: parents must be a list")
        if name in seen:
            raise BenchgenError(f"{source_file}: duplicate task name {name}")
        seen.add(name)
        tasks.append((str(name), tuple(str(p) for p in ups)))
    for name, ups in tasks:
        for p in ups:
            if p not in seen:
                raise BenchgenError(f"{source_file}: task {name} references unknown parent {p}")
    return RawTaskDag(tasks=tuple(tasks), source_file=source_file)


# (phase, base count, wiring to the previous phase) per family -- benchgen.py:403-479
FAMILY_PHASES = {
    "1000genome": [("individuals", 20, "root"), ("individuals_merge", 5, "fan"),
                   ("sifting", 2, "root"), ("mutation_overlap", 6, "fan"),
                   ("frequency", 6, "pair")],
    "blast": [("split_fasta", 1, "root"), ("blast_a", 10, "fan"), ("blast_b", 10, "root"),
              ("cat_blast", 1, "funnel"), ("cat", 1, "pair")],
    "bwa": [("fastq_reduce", 1, "root"), ("bwa_align_a", 12, "fan"),
            ("bwa_align_b", 12, "root"), ("cat_bwa", 2, "fan"), ("bwa_index", 1, "funnel")],
    "cycles": [("baseline_cycles", 8, "root"), ("cycles_a", 8, "pair"),
               ("fertilizer_increase", 8, "pair"), ("cycles_fi", 8, "pair"),
               ("summary", 2, "fan")],
    "montage": [("mproject", 10, "root"), ("mdifffit", 14, "fan"), ("mconcatfit", 1, "funnel"),
                ("mbgmodel", 1, "pair"), ("mbackground", 10, "fan"), ("mimgtbl", 1, "funnel"),
                ("madd", 1, "pair"), ("mshrink", 2, "fan"), ("mjpeg", 1, "funnel")],
    "nextflow": [("fastqc", 6, "root"), ("trimgalore", 6, "pair"), ("star_align", 6, "pair"),
                 ("markduplicates", 6, "pair"), ("multiqc", 1, "funnel")],
    "rnaseq": [("prep_genome", 1, "root"), ("hisat2_align", 8, "fan"),
               ("stringtie", 8, "pair"), ("ballgown", 1, "funnel")],
    "seismology": [("sg1iterdecon", 18, "root"), ("wrapper_siftstfbypixels", 1, "funnel"),
                   ("siftmerge", 1, "pair")],
    "soykb": [("alignment_to_reference", 10, "root"), ("sort_sam", 10, "pair"),
              ("dedup", 10, "pair"), ("add_replace", 10, "pair"),
              ("realign_target_creator", 2, "fan"), ("indel_realign", 2, "pair"),
              ("haplotype_caller", 6, "fan"), ("genotype_gvcfs", 1, "funnel"),
              ("combine_variants", 1, "pair")],
    "srasearch": [("prefetch", 12, "root"), ("fasterq_dump", 12, "pair"),
                  ("bowtie2_build", 1, "root"), ("bowtie2_align", 12, "fan"),
                  ("samtools_merge", 2, "fan")],
}
FAMILY_NAMES = tuple(sorted(FAMILY_PHASES))


def synth_raw_family(family: str, seed: int, scale: float = 1.0) -> str:
    if family not in FAMILY_PHASES:
        raise BenchgenError(f"unknown family {family!r}; known: {FAMILY_NAMES}")
    rng = random.Random(stable_hash64(family, seed) & 0x7FFFFFFF)
    tasks = []
    prev: list = []
    for phase, base, wiring in FAMILY_PHASES[family]:
        count = max(1, round(base * scale * (0.8 + 0.4 * rng.random())))
        names = [f"{phase}_{i + 1:05d}" for i in range(count)]
        for i, name in enumerate(names):
            if wiring == "root" or not prev:
                ups = []
            elif wiring == "fan":
                ups = list(prev)
            elif wiring == "pair":
                ups = [prev[i % len(prev)]]
            elif wiring == "funnel":
                ups = list(prev) if i == 0 else [prev[i % len(prev)]]
            else:
                raise BenchgenError(f"unknown wiring {wiring!r}")
            tasks.append({"name": name, "parents": ups})
        prev = names
    return json.dumps({"name": family, "workflow": {"tasks": tasks}}, indent=2, sort_keys=True)


# ---------------------------------------------------------------------------
# Lifting (reference benchgen.py:131-239)
# ---------------------------------------------------------------------------

_INDEX_SUFFIX = re.compile(r"([_\-.]\d+)+$")


def normalize_task_name(name: str) -> str:
    return _INDEX_SUFFIX.sub("", name.lower())


def _raw_is_acyclic(raw: RawTaskDag) -> bool:
    names = [n for n, _ in raw.tasks]
    waiting = {n: len(ups) for n, ups in raw.tasks}
    down: dict = {n: [] for n in names}
    for n, ups in raw.tasks:
        for p in ups:
            down[p].append(n)
    stack = [n for n in names if waiting[n] == 0]
    visited = 0
    while stack:
        n = stack.pop()
        visited += 1
        for c in down[n]:
            waiting[c] -= 1
            if waiting[c] == 0:
                stack.append(c)
    return visited == len(names)


def _longest_levels(groups, edges) -> dict:
    ups: dict = {g: [] for g in groups}
    for src, dst in edges:
        ups[dst].append(src)
    memo: dict = {}
    for root in sorted(groups):
        if root in memo:
            continue
        stack = [root]
        while stack:
            g = stack[-1]
            todo = [p for p in ups[g] if p not in memo]
            if todo:
                stack.extend(todo)
                continue
            stack.pop()
            memo[g] = max((memo[p] + 1 for p in ups[g]), default=0)
    return memo


def lift_dag(raw: RawTaskDag, params: LiftParams) -> WorkflowDag:
    """Collapse tasks into name-prefix groups, split to ``min_groups``, then
    drop deepest groups down to ``max_stages`` splicing their edges."""
    if not _raw_is_acyclic(raw):
        raise BenchgenError(f"{raw.source_file}: raw task graph is cyclic")
    group_of: dict = {}
    members: dict = {}
    for name, _ in raw.tasks:
        g = normalize_task_name(name) if params.prefix_collapse else name.lower()
        group_of[name] = g
        members.setdefault(g, []).append(name)
    for g in members:
        members[g].sort()

    splits = 0
    while len(members) < params.min_groups:
        g = min(members, key=lambda k: (-len(members[k]), k))
        names = members[g]
        if len(names) < 2:
            break
        splits += 1
        cut = math.ceil(len(names) / 2)
        fresh = f"{g}+{splits}"
        members[g], members[fresh] = names[:cut], names[cut:]
        for n in members[fresh]:
            group_of[n] = fresh

    edges = {(group_of[p], group_of[name]) for name, ups in raw.tasks for p in ups
             if group_of[p] != group_of[name]}

    levels = _longest_levels(set(members), edges)
    while len(members) > params.max_stages:
        victim = min(members, key=lambda g: (-levels[g], g))
        ins = {s for (s, d) in edges if d == victim}
        outs = {d for (s, d) in edges if s == victim}
        edges = {(s, d) for (s, d) in edges if s != victim and d != victim}
        edges |= {(s, d) for s in ins for d in outs if s != d}
        del members[victim], levels[victim]

    dag = WorkflowDag(
        workflow_id=f"{params.family}-{raw.source_file}", family=params.family,
        stages={g: Stage(id=g) for g in sorted(members)}, edges=frozenset(edges),
    )
    return annotate_topology(dag)


# ---------------------------------------------------------------------------
# Roles, models, devices (reference benchgen.py:247-340)
# ---------------------------------------------------------------------------


def assign_roles(dag: WorkflowDag, config, seed: int = DEFAULT_SEED) -> WorkflowDag:
    if dag.annotations is None:
        dag = annotate_topology(dag)
    ann = dag.annotations
    top = ann.max_level
    staged = {}
    for sid in sorted(dag.stages):
        lvl, fan_in, fan_out = ann.level[sid], ann.indegree[sid], ann.outdegree[sid]
        here_w = ann.level_width.get(lvl, 1)
        prev_w = ann.level_width.get(lvl - 1, 1)
        if fan_in == 0 or (lvl <= 1 and here_w >= 3):
            bucket = EARLY_ROLES
        elif lvl < top and fan_out >= 3:
            bucket = ("worker",)
        elif fan_in >= 3 or (fan_in >= 2 and 2 * fan_in >= prev_w):
            bucket = MERGE_ROLES
        elif fan_out == 0 or lvl == top:
            bucket = LATE_ROLES
        else:
            bucket = ("worker",)
        role = config.roles[stable_choice(list(bucket), sid, seed)]
        staged[sid] = replace(
            dag.stages[sid], role=role, shard_bound=2 if role.shard_eligible else 1,
            prompt_token_proxy=role.max_token_proxy // 4,
            output_token_proxy=role.output_size_proxy,
            keep_cache=role.default_keep_cache, cache_reuse=role.default_cache_reuse,
        )
    return annotate_topology(replace(dag, stages=staged))


def assign_models(dag: WorkflowDag, seed: int, config, pinned_alias: str | None = None):
    staged = {}
    for sid in sorted(dag.stages):
        st = dag.stages[sid]
        if st.role is None:
            raise BenchgenError(f"stage {sid}: assign_roles must run before assign_models")
        if pinned_alias is not None:
            alias = pinned_alias
        else:
            cands = config.role_models.get(st.role.kind, ())
            if not cands:
                raise BenchgenError(f"role {st.role.kind}: empty model candidate set")
            alias = stable_choice(list(cands), dag.workflow_id, sid, seed)
        staged[sid] = replace(st, model=alias,
                              shared_prefix_group=f"pg:{alias}" if st.cache_reuse else None)
    return annotate_topology(replace(dag, stages=staged))


def assign_devices(dag: WorkflowDag, device_ids) -> WorkflowDag:
    everyone = frozenset(device_ids)
    staged = {sid: replace(st, eligible_devices=everyone) for sid, st in dag.stages.items()}
    return annotate_topology(replace(dag, stages=staged))


def finalize_dag(dag: WorkflowDag, config, seed: int, pinned_alias: str | None = None):
    dag = assign_roles(dag, config, seed=seed)
    dag = assign_models(dag, seed, config, pinned_alias=pinned_alias)
    dag = assign_devices(dag, config.topology.device_ids)
    report = validate_dag(dag, config.topology)
    if not report.ok:
        raise BenchgenError(f"generated dag invalid: {report.violations[:3]}")
    return dag


def make_queries(workflow_id: str, batch_size: int, seed: int, min_tokens: int = 200,
                 span: int = 600) -> tuple:
    return tuple(
        Query(f"q{i:03d}", min_tokens + stable_hash64(workflow_id, "query", i, seed) % span)
        for i in range(batch_size)
    )


def make_instance(dag: WorkflowDag, batch_size: int, seed: int) -> WorkflowInstance:
    return WorkflowInstance(dag=dag, queries=make_queries(dag.workflow_id, batch_size, seed),
                            batch_size=batch_size)


# ---------------------------------------------------------------------------
# Synthetic layered DAGs (reference benchgen.py:369-393)
# ---------------------------------------------------------------------------


def synth_layers(spec: SuiteSpec):
    """Layer names and edge set of the layered random DAG (the RNG-consuming
    part of ``synth_generate``)."""
    rng = random.Random(spec.seed)
    layers = [[f"s{d * spec.width + i:02d}" for i in range(spec.width)]
              for d in range(spec.depth)]
    edges = set()
    for d in range(1, spec.depth):
        above = layers[d - 1]
        for v in layers[d]:
            ups = [u for u in above if rng.random() < spec.density]
            if not ups:
                ups = [above[rng.randrange(len(above))]]
            edges.update((u, v) for u in ups)
    return layers, edges


def synth_generate(spec: SuiteSpec, config) -> WorkflowDag:
    if spec.kind != "synthetic":
        raise BenchgenError(f"synth_generate got suite kind {spec.kind!r}")
    layers, edges = synth_layers(spec)
    dag = WorkflowDag(
        workflow_id=f"synthetic-d{spec.depth}w{spec.width}-s{spec.seed}", family="synthetic",
        stages={sid: Stage(id=sid) for layer in layers for sid in layer},
        edges=frozenset(edges),
    )
    return finalize_dag(annotate_topology(dag), config, seed=spec.seed)


def lifted_instance(family: str, config, seed: int, batch_size: int = 16, scale: float = 1.0,
                    max_stages: int = 64, min_groups: int = 12) -> WorkflowInstance:
    raw = import_workflow_json(synth_raw_family(family, seed, scale=scale),
                               source_file=f"{family}-{seed}")
    dag = lift_dag(raw, LiftParams(max_stages=max_stages, min_groups=min_groups, seed=seed,
                                   family=family))
    dag = replace(dag, workflow_id=f"{family}-s{seed}")
    dag = finalize_dag(annotate_topology(dag), config, seed=seed)
    return make_instance(dag, batch_size, seed)


# ---------------------------------------------------------------------------
# Controlled suites (reference benchgen.py:542-655)
# ---------------------------------------------------------------------------


def grouped_queries(workflow_id: str, spec: SuiteSpec):
    n_grouped = math.floor(spec.repeat_ratio * spec.batch_size)
    queries = []
    groups: dict = {}
    for i in range(spec.batch_size):
        tokens = spec.prefix_length + 100 + stable_hash64(workflow_id, "tail", i, spec.seed) % 100
        gid = None
        if i < n_grouped:
            gid = f"qg{i // spec.group_size:02d}"
            groups[gid] = spec.prefix_length
        queries.append(Query(f"q{i:03d}", tokens, gid))
    return tuple(queries), groups


_PREFIX_SHAPES = (("chain", 4, 1, 1.0), ("funnelweb", 3, 2, 1.0), ("wide", 3, 3, 0.7))


def build_prefix_suite(spec: SuiteSpec, config) -> list:
    if spec.kind != "prefix_reuse":
        raise BenchgenError(f"build_prefix_suite got suite kind {spec.kind!r}")
    out = []
    for shape, depth, width, density in _PREFIX_SHAPES:
        shape_seed = spec.seed + stable_hash64("prefix", shape) % 1000
        dag = synth_generate(replace(spec, kind="synthetic", depth=depth, width=width,
                                     density=density, seed=shape_seed), config)
        dag = annotate_topology(replace(dag, stages={
            sid: replace(st, keep_cache=True, cache_reuse=True) for sid, st in dag.stages.items()
        }))
        dag = assign_models(dag, spec.seed, config)
        dag = assign_devices(dag, config.topology.device_ids)
        tag = f"{int(round(spec.repeat_ratio * 100)):03d}"
        dag = replace(dag, workflow_id=f"prefix-{shape}-r{tag}-b{spec.batch_size}",
                      family="prefix_reuse")
        queries, groups = grouped_queries(dag.workflow_id, spec)
        out.append(WorkflowInstance(dag=dag, queries=queries, batch_size=spec.batch_size,
                                    prefix_groups=groups))
    return out


CONFLICT_RATIOS = (0.0, 0.25, 0.5, 1.0)
_CONFLICT_MODELS = ("qwen-7b", "deepseek-7b", "llama-8b")


def build_conflict_suite(spec: SuiteSpec, config) -> list:
    if spec.kind != "conflict":
        raise BenchgenError(f"build_conflict_suite got suite kind {spec.kind!r}")
    worker = config.roles["worker"]
    everyone = frozenset(config.topology.device_ids)
    out = []
    for ratio in CONFLICT_RATIOS:
        wid = f"conflict-{int(round(ratio * 100)):03d}-b{spec.batch_size}"
        stages = {}
        for i in range(spec.chain_length):
            sid = f"c{i:02d}"
            stages[sid] = Stage(
                id=sid, model=_CONFLICT_MODELS[i % 3], eligible_devices=everyone, shard_bound=1,
                role=worker, prompt_token_proxy=spec.prefix_length,
                output_token_proxy=worker.output_size_proxy,
                shared_prefix_group="conflict-chain", keep_cache=True, cache_reuse=True,
            )
        edges = frozenset((f"c{i - 1:02d}", f"c{i:02d}") for i in range(1, spec.chain_length))
        dag = annotate_topology(WorkflowDag(workflow_id=wid, family="conflict", stages=stages,
                                            edges=edges))
        queries, groups = grouped_queries(wid, replace(spec, repeat_ratio=ratio,
                                                       prefix_length=400))
        out.append(WorkflowInstance(dag=dag, queries=queries, batch_size=spec.batch_size,
                                    prefix_groups=groups))
    return out
