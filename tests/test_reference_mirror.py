"""Host-side mirrors and the drop-in policy against the live reference.

* generators: every config-1..5 instance built by the package's generator
  mirror (wf/workloads, used by the native-generator tests and the C4/C5
  canonical configs) equals the reference's (stages, roles, models, edges,
  annotations, queries, groups);
* policy: FateGpuPolicy (a subclass of the reference FatePolicy whose scores
  come from a scorer -- here the oracle) run by the reference executor
  reproduces the reference FatePolicy's RunRecords on instances outside the
  golden set (conflict suite, other lifted families).
"""

from __future__ import annotations

import random
from dataclasses import replace

import pytest

from paper_2605_07238_b200 import scenarios
from paper_2605_07238_b200.planner import FateGpuPolicy
from paper_2605_07238_b200.wf import workloads as MB
from paper_2605_07238_b200.wf import weights as MC

from oracle_scorer import OracleScorer

pytestmark = pytest.mark.reference


def _stage_sig(s):
    r = s.role
    role = None if r is None else (r.kind, r.complexity, r.prefill_scale, r.decode_scale,
                                   r.max_token_proxy, r.output_size_proxy, r.comm_weight,
                                   r.default_keep_cache, r.default_cache_reuse, r.shard_eligible)
    return (s.id, s.model, tuple(sorted(s.eligible_devices)), s.shard_bound, role,
            s.prompt_token_proxy, s.output_token_proxy, s.shared_prefix_group, s.keep_cache,
            s.cache_reuse, s.base_cost_override)


def sig(inst):
    d, a = inst.dag, inst.dag.annotations
    return (d.workflow_id, d.family, tuple(_stage_sig(d.stages[k]) for k in sorted(d.stages)),
            tuple(sorted(d.edges)), tuple(sorted(a.level.items())),
            tuple(sorted(a.indegree.items())), tuple(sorted(a.outdegree.items())),
            tuple(sorted(a.reverse_depth.items())), tuple(sorted(a.level_width.items())),
            tuple(tuple(q) for q in inst.queries), inst.batch_size,
            tuple(sorted(inst.prefix_groups.items())))


def test_generators_match_reference(reference):
    import wfsched.benchgen as RB
    import wfsched.config as RC

    rc, mc = RC.default_config(4), MC.default_config(4)
    for fam in MB.FAMILY_NAMES:
        for seed in (11, 14):
            a = RB.lifted_instance(fam, rc, seed=seed, batch_size=32, scale=0.75 + 0.25 * (seed % 3),
                                   min_groups=14 + 4 * (seed % 4))
            b = MB.lifted_instance(fam, mc, seed=seed, batch_size=32, scale=0.75 + 0.25 * (seed % 3),
                                   min_groups=14 + 4 * (seed % 4))
            assert sig(a) == sig(b), (fam, seed)
    for r in (0.0, 0.5, 1.0):
        A = RB.build_prefix_suite(RB.SuiteSpec(kind="prefix_reuse", repeat_ratio=r), rc)
        B = MB.build_prefix_suite(MB.SuiteSpec(kind="prefix_reuse", repeat_ratio=r), mc)
        assert [sig(x) for x in A] == [sig(x) for x in B]
    A = RB.build_conflict_suite(RB.SuiteSpec(kind="conflict"), rc)
    B = MB.build_conflict_suite(MB.SuiteSpec(kind="conflict"), mc)
    assert [sig(x) for x in A] == [sig(x) for x in B]
    cfg5 = scenarios.config_c5()
    for i in (0, 1, 4095):
        a = RB.make_instance(RB.synth_generate(RB.SuiteSpec(
            kind="synthetic", depth=20, width=25, density=0.12, seed=1000 + i), cfg5), 16, 1000 + i)
        assert sig(a) == sig(scenarios.c5_instance(i, cfg5))
    for text in ("hello", "x|y|3", "ü"):
        assert MB.stable_hash64(text, 7) == __import__("wfsched.hashutil").hashutil.stable_hash64(text, 7)
    keys = [f"s{i}|{i * 7}" for i in range(300)]
    assert MB.stable_hash64_many(keys) == [MB.stable_hash64(k) for k in keys]


def test_instance_json_matches_reference_serialiser(reference):
    """Mirror writer == reference writer, text for text; each reader accepts
    the other's output (model.py:322-422)."""
    import wfsched.benchgen as RB
    import wfsched.model as RM

    from paper_2605_07238_b200.wf import instance_io as IO

    cfg5 = scenarios.config_c5()
    pairs = [(RB.make_instance(RB.synth_generate(RB.SuiteSpec(
        kind="synthetic", depth=20, width=25, density=0.12, seed=1000 + i), cfg5), 16, 1000 + i),
        scenarios.c5_instance(i, cfg5)) for i in (0, 7)]
    rc, mc = __import__("wfsched.config").config.default_config(4), MC.default_config(4)
    pairs += list(zip(RB.build_prefix_suite(RB.SuiteSpec(kind="prefix_reuse", repeat_ratio=0.25), rc),
                      MB.build_prefix_suite(MB.SuiteSpec(kind="prefix_reuse", repeat_ratio=0.25), mc)))
    for ref_inst, mir_inst in pairs:
        text = RM.instance_to_json(ref_inst)
        assert IO.instance_to_json(mir_inst) == text
        assert IO.instance_to_json(IO.instance_from_json(text)) == text
        assert RM.instance_to_json(RM.instance_from_json(IO.instance_to_json(mir_inst))) == text


def test_executor_matches_reference_on_unseen_runs(reference):
    import wfsched.benchgen as RB
    import wfsched.config as RC
    from wfsched import executor as RE
    from wfsched.policies import make_policy

    rc = RC.default_config(4)
    pairs = [(inst, 4) for inst in RB.build_conflict_suite(RB.SuiteSpec(kind="conflict"), rc)]
    pairs.append((RB.lifted_instance("montage", rc, seed=21, batch_size=24), 3))
    pairs.append((RB.lifted_instance("cycles", RC.default_config(6), seed=5, batch_size=8), 2))
    for inst_r, h in pairs:
        n_dev = len(inst_r.dag.stages[sorted(inst_r.dag.stages)[0]].eligible_devices)
        rcfg = RC.default_config(n_dev)
        rcfg = rcfg.with_weights(replace(rcfg.weights, horizon=h))
        want = RE.run(make_policy("fate"), inst_r, rcfg)
        got = RE.run(FateGpuPolicy(scorer=OracleScorer()), inst_r, rcfg)
        assert got.makespan == want.makespan
        assert got.query_completion == want.query_completion
        assert (got.workflow_tasks, got.cross_device_parent_edges, got.prefix_cache_hits_est,
                got.same_model_continuations, got.solver_solves) == (
            want.workflow_tasks, want.cross_device_parent_edges, want.prefix_cache_hits_est,
            want.same_model_continuations, want.solver_solves)
