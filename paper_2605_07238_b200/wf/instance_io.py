"""Instance / DAG JSON interchange (``wfsched.dag@1``, ``wfsched.instance@1``).

Restates the reference's serialisers (``pkg/src/wfsched/model.py:322-422``)
over the mirror's types so that instance files written by the reference CLI
(``wfsched.cli`` ``generate``, ``cli.py:82``) or listed in a harness manifest
(``harness.py:246``) load here unchanged, and files written here load in the
reference: same schema strings, same key set, ``sort_keys`` + ``indent=2``
text, stages sorted by id, edges as sorted ``[src, dst]`` pairs,
``base_cost_override`` emitted only when set, annotations recomputed on load.
The round trip is byte-identical to the reference's text for the same
instance (tests/test_instance_io.py).
"""

from __future__ import annotations

import json

from .dagmodel import Query, Stage, StageRole, WorkflowDag, WorkflowInstance, annotate_topology

DAG_SCHEMA = "wfsched.dag@1"
INSTANCE_SCHEMA = "wfsched.instance@1"

_ROLE_FIELDS = ("kind", "complexity", "prefill_scale", "decode_scale", "max_token_proxy",
                "output_size_proxy", "comm_weight", "default_keep_cache",
                "default_cache_reuse", "shard_eligible")


def _role_doc(role: StageRole) -> dict:
    return {name: getattr(role, name) for name in _ROLE_FIELDS}


def _stage_doc(stage: Stage) -> dict:
    doc = {
        "id": stage.id,
        "model": stage.model,
        "eligible_devices": sorted(stage.eligible_devices),
        "shard_bound": stage.shard_bound,
        "role": None if stage.role is None else _role_doc(stage.role),
        "prompt_token_proxy": stage.prompt_token_proxy,
        "output_token_proxy": stage.output_token_proxy,
        "shared_prefix_group": stage.shared_prefix_group,
        "keep_cache": stage.keep_cache,
        "cache_reuse": stage.cache_reuse,
    }
    if stage.base_cost_override is not None:
        doc["base_cost_override"] = {k: stage.base_cost_override[k]
                                     for k in sorted(stage.base_cost_override)}
    return doc


def _stage_of(doc: dict) -> Stage:
    role_doc = doc.get("role")
    return Stage(
        id=doc["id"],
        model=doc.get("model"),
        eligible_devices=frozenset(doc.get("eligible_devices", ())),
        shard_bound=int(doc.get("shard_bound", 1)),
        role=StageRole(**role_doc) if role_doc else None,
        prompt_token_proxy=int(doc.get("prompt_token_proxy", 0)),
        output_token_proxy=int(doc.get("output_token_proxy", 0)),
        shared_prefix_group=doc.get("shared_prefix_group"),
        keep_cache=bool(doc.get("keep_cache", False)),
        cache_reuse=bool(doc.get("cache_reuse", False)),
        base_cost_override=doc.get("base_cost_override"),
    )


def _dag_doc(dag: WorkflowDag) -> dict:
    return {
        "schema": DAG_SCHEMA,
        "workflow_id": dag.workflow_id,
        "family": dag.family,
        "stages": [_stage_doc(dag.stages[sid]) for sid in sorted(dag.stages)],
        "edges": [list(e) for e in sorted(dag.edges)],
    }


def _dag_of(doc: dict) -> WorkflowDag:
    if doc.get("schema") != DAG_SCHEMA:
        raise ValueError(f"unsupported dag schema {doc.get('schema')!r}")
    stages = {}
    for sdoc in doc["stages"]:
        st = _stage_of(sdoc)
        stages[st.id] = st
    edges = frozenset((src, dst) for src, dst in doc["edges"])
    return annotate_topology(WorkflowDag(workflow_id=doc["workflow_id"], family=doc["family"],
                                         stages=stages, edges=edges))


def dag_to_json(dag: WorkflowDag) -> str:
    return json.dumps(_dag_doc(dag), indent=2, sort_keys=True)


def dag_from_json(text: str) -> WorkflowDag:
    return _dag_of(json.loads(text))


def instance_to_json(instance: WorkflowInstance) -> str:
    doc = {
        "schema": INSTANCE_SCHEMA,
        "dag": _dag_doc(instance.dag),
        "queries": [list(q) for q in instance.queries],
        "batch_size": instance.batch_size,
        "prefix_groups": {k: instance.prefix_groups[k] for k in sorted(instance.prefix_groups)},
    }
    return json.dumps(doc, indent=2, sort_keys=True)


def instance_from_json(text: str) -> WorkflowInstance:
    doc = json.loads(text)
    if doc.get("schema") != INSTANCE_SCHEMA:
        raise ValueError(f"unsupported instance schema {doc.get('schema')!r}")
    return WorkflowInstance(
        dag=_dag_of(doc["dag"]),
        queries=tuple(Query(q[0], int(q[1]), q[2]) for q in doc["queries"]),
        batch_size=int(doc["batch_size"]),
        prefix_groups={k: int(v) for k, v in doc.get("prefix_groups", {}).items()},
    )
