"""Replay captured reference runs through the REFERENCE executor
(``wfsched.executor.run``) with the GPU policy plugged in, checking every wave
against the golden vectors.

Golden files (tests/golden/*.json + *.npz) come from the reference itself
(tests/golden/make_golden.py).  Instances and configs are rebuilt with the
reference's own generators; ``wfsched`` is importable from ``baseline/_ref``
(the reference install, which travels to the GPU box) or from
/root/reference in the build container (tests/conftest.py).
"""

from __future__ import annotations

import json
import os
from dataclasses import replace

import numpy as np
import wfsched.benchgen as W
import wfsched.executor as RE
from wfsched.config import AblationFlags, default_config

from paper_2605_07238_b200 import compat
from paper_2605_07238_b200.planner import FateGpuPolicy, WaveScores

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)
    arr = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    runs = meta["runs"]
    pc = sc = 0
    for r in runs:
        for wv in r["waves"]:
            wv["psi_at"] = pc
            wv["pair_at"] = sc
            pc += wv["n_cand"]
            sc += wv["n_pairs"]
    return runs, {k: arr[k] for k in arr.files}


def _f64(bits_u64) -> np.ndarray:
    return np.asarray(bits_u64, dtype=np.uint64).view(np.float64)


# ---------------------------------------------------------------------------
# instance + config rebuild
# ---------------------------------------------------------------------------


def c1_setup(variant: dict):
    cfg = default_config(4)
    inst = W.lifted_instance("soykb", cfg, seed=11, batch_size=16, scale=1.0, min_groups=50)
    kw = {k: v for k, v in variant.items() if k not in ("tag", "ablation")}
    if "ablation" in variant:
        kw["ablation"] = AblationFlags.from_names(variant["ablation"])
    return inst, cfg.with_weights(replace(cfg.weights, **kw))


def c3_setup(ratio: float, batch: int, shape: int):
    cfg = default_config(4)
    suite = W.build_prefix_suite(W.SuiteSpec(kind="prefix_reuse", repeat_ratio=ratio,
                                             batch_size=batch, seed=20260423), cfg)
    return suite[shape], cfg.with_weights(replace(cfg.weights, horizon=3))


_C2_SYNTH = {**{s: (5, 4, 0.5) for s in (101, 102, 103, 104)},
             **{s: (7, 3, 0.7) for s in (105, 106, 107, 108)}}


def c2_setup(key: str):
    """Rebuild a default-manifest main instance (reference harness.py:182-284)."""
    cfg = default_config(4)
    wid, btag = key.rsplit("@b", 1)
    batch = int(btag)
    seed = int(wid.rsplit("-s", 1)[1])
    if wid.startswith("synthetic-"):
        depth, width, density = _C2_SYNTH[seed]
        dag = W.synth_generate(W.SuiteSpec(kind="synthetic", depth=depth, width=width,
                                           density=density, seed=seed, batch_size=batch), cfg)
        inst = W.make_instance(dag, batch, seed)
    else:
        family = wid.rsplit("-s", 1)[0]
        inst = W.lifted_instance(family, cfg, seed=seed, batch_size=batch,
                                 scale=0.75 + 0.25 * (seed % 3), max_stages=64,
                                 min_groups=14 + 4 * (seed % 4))
    assert inst.dag.workflow_id == wid
    return inst, cfg


# ---------------------------------------------------------------------------
# checking scorer
# ---------------------------------------------------------------------------


class CheckingScorer:
    """Delegates to a scorer and compares each wave with the golden one."""

    def __init__(self, inner, run_meta: dict, arrays: dict):
        self.inner = inner
        self.waves = run_meta["waves"]
        self.arrays = arrays
        self.i = 0
        self.mismatches: list = []
        self.n_psi = 0

    def score_wave(self, frontier, state, cost_model, dag=None) -> WaveScores:
        ws = self.inner.score_wave(frontier, state, cost_model, dag)
        if self.i >= len(self.waves):
            self.mismatches.append(f"extra wave {self.i}")
            self.i += 1
            return ws
        g = self.waves[self.i]
        if ws.stage_ids != g["frontier"]:
            self.mismatches.append(f"wave {self.i}: frontier {ws.stage_ids} != {g['frontier']}")
        else:
            if g["n_cand"]:
                got = np.asarray([c.psi for c in ws.candidates()], dtype=np.float64)
                want = _f64(self.arrays["psi"][g["psi_at"]: g["psi_at"] + g["n_cand"]])
                self.n_psi += len(want)
                if got.shape != want.shape or not np.array_equal(got.view(np.uint64),
                                                                 want.view(np.uint64)):
                    self.mismatches.append(f"wave {self.i}: psi differs")
            mask = [[(m >> j) & 1 for j in range(len(ws.device_ids))] for m in ws.elig]
            sel = np.asarray(mask, dtype=bool)
            for key, arr in (("sched", ws.sched), ("completion", ws.completion)):
                got = np.ascontiguousarray(arr[sel])
                want = _f64(self.arrays[key][g["pair_at"]: g["pair_at"] + g["n_pairs"]])
                if got.shape != want.shape or not np.array_equal(got.view(np.uint64),
                                                                 want.view(np.uint64)):
                    self.mismatches.append(f"wave {self.i}: {key} differs")
        self.i += 1
        return ws


def record_mismatches(rec, want: dict) -> list:
    out = []
    got = {
        "makespan": rec.makespan.hex(), "p95": rec.p95_latency().hex(),
        "workflow_tasks": rec.workflow_tasks,
        "cross_device_parent_edges": rec.cross_device_parent_edges,
        "prefix_cache_hits_est": rec.prefix_cache_hits_est,
        "same_model_continuations": rec.same_model_continuations,
        "solver_solves": rec.solver_solves, "solver_optimal": rec.solver_optimal,
        "ablation": rec.ablation, "perturbation": rec.perturbation, "h_value": rec.h_value,
        "query_completion": {k: v.hex() for k, v in rec.query_completion.items()},
        "workflow_id": rec.workflow_id, "batch_size": rec.batch_size,
    }
    for k, v in got.items():
        if want.get(k) != v:
            out.append(f"record {k}: {v} != {want.get(k)}")
    return out


def replay(run_meta: dict, arrays: dict, instance, config, scorer, seed: int = 0,
           solver: str = "reference", mirror=None, durations: bool = False):
    """One FATE run of the reference executor with the GPU policy; ``mirror``
    (a MirrorScorer) is attached to the executor's live state and
    ``durations`` prices the executor's issued tasks on the GPU, both through
    ``compat.install``."""
    chk = CheckingScorer(scorer, run_meta, arrays)
    policy = FateGpuPolicy(scorer=chk, solver=solver)
    hooked = mirror is not None or durations
    if hooked:
        compat.install(scorer=None if mirror is not None else scorer, mirror=mirror,
                       policy_factory=False, durations=durations)
    try:
        rec = RE.run(policy, instance, config, seed=seed)
    finally:
        if hooked:
            compat.uninstall()
    problems = list(chk.mismatches)
    if chk.i != len(run_meta["waves"]):
        problems.append(f"{chk.i} waves != golden {len(run_meta['waves'])}")
    problems += record_mismatches(rec, run_meta["record"])
    return rec, problems, chk.n_psi
