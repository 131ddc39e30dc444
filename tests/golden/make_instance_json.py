"""Instance JSON fixtures written by the REFERENCE serialiser (build container).

    python tests/golden/make_instance_json.py

Runs the reference's ``instance_to_json`` (pkg/src/wfsched/model.py:400-409)
on three instances and stores the text under tests/golden/instances/:
  * c1.json      -- config 1 (lifted soykb, 4 devices, min_groups=50);
  * prefix.json  -- one config-3 prefix-suite instance (prefix groups set);
  * override.json -- a hand-built 3-stage DAG with a role-less stage and a
                     ``base_cost_override`` (the optional key the writer
                     emits only when set, model.py:355-356).
tests/test_instance_io.py loads them with the mirror's reader and checks the
byte-identical round trip and the packed arrays.
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import wfsched.benchgen as RB  # noqa: E402
from wfsched import model as RM  # noqa: E402
from wfsched.config import default_config  # noqa: E402


def override_instance():
    role = RM.StageRole(kind="worker", complexity=1.5, comm_weight=0.5)
    devs = frozenset(("gpu0", "gpu1"))
    stages = {
        "a": RM.Stage(id="a", model="llama-8b", eligible_devices=devs, role=role,
                      prompt_token_proxy=300, output_token_proxy=200,
                      shared_prefix_group="g0", cache_reuse=True),
        "b": RM.Stage(id="b", model="llama-8b", eligible_devices=devs, shard_bound=2,
                      role=role, prompt_token_proxy=512, output_token_proxy=128,
                      base_cost_override={"gpu1": 3.25, "gpu0": 2.5}),
        "c": RM.Stage(id="c", model=None, eligible_devices=frozenset(("gpu1",)),
                      prompt_token_proxy=64, output_token_proxy=32, keep_cache=True),
    }
    dag = RM.annotate_topology(RM.WorkflowDag(workflow_id="override", family="handmade",
                                              stages=stages,
                                              edges=frozenset({("a", "b"), ("a", "c")})))
    queries = (RM.Query("q0", 210, "g0"), RM.Query("q1", 450, None))
    return RM.WorkflowInstance(dag=dag, queries=queries, batch_size=2,
                               prefix_groups={"g0": 2})


def main():
    out = os.path.join(HERE, "instances")
    os.makedirs(out, exist_ok=True)
    cfg = default_config(4)
    c1 = RB.lifted_instance("soykb", cfg, seed=11, batch_size=16, scale=1.0, min_groups=50)
    suite = RB.build_prefix_suite(RB.SuiteSpec(kind="prefix_reuse", repeat_ratio=0.5,
                                               batch_size=16, seed=20260423), cfg)
    for name, inst in (("c1", c1), ("prefix", suite[0]), ("override", override_instance())):
        with open(os.path.join(out, f"{name}.json"), "w") as fh:
            fh.write(RM.instance_to_json(inst))
        print(name, len(inst.dag.stages), "stages")


if __name__ == "__main__":
    main()
