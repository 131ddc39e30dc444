"""Drop-in GPU cost matrix for the reference scheduler, and the FATE policy
that consumes it.

This module sits *behind* the caller's own ``wfsched`` (the reference
package): every type it returns is the caller's type and every decision
that is not scoring is the caller's code.

* :func:`build_problem` -- same signature and result as
  ``wfsched.planner.build_problem(frontier, state, cost_model, dag)``
  (``pkg/src/wfsched/planner.py:75-98``): a ``wfsched.planner.FrontierProblem``
  of ``wfsched.planner.Candidate`` (sorted stage, slot < bound, sorted eligible
  device), Psi bit-identical, negative scores retained -- computed by the
  sm_100a kernel in one launch per wave.
* :class:`WaveCostModel` -- a read-only view of ``wfsched.costs.CostModel``
  answering ``plan_score`` / ``sched_score`` / ``tail_value`` and the
  full-batch ``realized_duration`` (``costs.py:210-247, 281-352, 383-416``)
  from one GPU-scored wave.
* :class:`FateGpuPolicy` -- a subclass of the caller's
  ``wfsched.policies.FatePolicy`` (``policies.py:44-193``, ``name = "fate"``).
  It scores the wave on the GPU and hands the caller's own methods the view:
  the horizon-0 greedy (``_greedy_wave``, reads S), the work-conserving fill
  (``_extend_work_conserving``, reads ``realized_duration``), ``_materialize`` /
  ``_align_shards`` and the solve (``wfsched.planner.solve_frontier``, or the
  native restatement ``solver="native"``) all run unchanged, host-side.

No CPU fallback: without CUDA or ``libfate.so`` these raise
:class:`~paper_2605_07238_b200.runtime.FateUnavailable`.
"""

from __future__ import annotations

import importlib
import time
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import pack
from .runtime import DeviceBank, WaveRunner, WaveStaging


def _wf(name: str):
    """A module of the caller's ``wfsched`` (the package this is a drop-in for)."""
    try:
        return importlib.import_module(f"wfsched.{name}")
    except ImportError as exc:  # pragma: no cover - depends on the caller
        raise ImportError("paper_2605_07238_b200.planner plugs into the reference scheduler "
                          "package 'wfsched'; make it importable") from exc


_PLANNER = _wf("planner")
_POLICIES = _wf("policies")
_COSTS = _wf("costs")


@dataclass
class WaveScores:
    """Host copies of one wave's GPU outputs."""

    stage_ids: list      # sorted frontier
    bounds: list
    device_ids: list     # sorted device ids
    elig: list           # per stage: eligible-device bitmask
    psi: np.ndarray      # [n_psi] dense slot-major rows
    psi_off: np.ndarray
    sched: np.ndarray    # [F, D]
    completion: np.ndarray
    tail: np.ndarray
    timing: np.ndarray | None = None  # [F, D, 3] switch, transfer, compute

    def candidates(self):
        """``wfsched.planner.Candidate`` tuples in ``build_problem`` order."""
        Candidate = _PLANNER.Candidate
        out = []
        D = len(self.device_ids)
        for i, sid in enumerate(self.stage_ids):
            m = self.elig[i]
            base = int(self.psi_off[i])
            for k in range(self.bounds[i]):
                row = self.psi[base + k * D: base + (k + 1) * D]
                out.extend(Candidate(sid, k, self.device_ids[d], float(row[d]))
                           for d in range(D) if m >> d & 1)
        return out


class GpuScorer:
    """Caches HBM-resident static banks per (instance, catalog, weights) and
    scores per-wave state snapshots on the GPU."""

    def __init__(self, max_banks: int = 8, device=None):
        self._banks: OrderedDict = OrderedDict()
        self.max_banks = max_banks
        self.device = device
        self.kernel_seconds = 0.0
        self.bank_seconds = 0.0  # packing + uploading banks (once per instance)
        self._staging = None

    def _entry(self, instance, models, topo, weights):
        key = (id(instance), id(models), id(topo), weights)
        hit = self._banks.get(key)
        if hit is not None and hit[0] is instance:
            self._banks.move_to_end(key)
            return hit
        t0 = time.perf_counter()
        packed = pack.pack_bank([instance], models, topo)
        dbank = DeviceBank(packed, weights, device=self.device)
        self.bank_seconds += time.perf_counter() - t0
        hit = [instance, dbank, models, topo, None]  # strong refs: no id() reuse
        self._banks[key] = hit
        while len(self._banks) > self.max_banks:
            self._banks.popitem(last=False)
        return hit

    def bank_for(self, instance, models, topo, weights) -> DeviceBank:
        return self._entry(instance, models, topo, weights)[1]

    def score_wave(self, frontier, state, cost_model, dag=None) -> WaveScores:
        """One launch per wave through the bank's :class:`~.runtime.WaveRunner`
        (one H2D, one kernel, one D2H)."""
        instance = state.instance
        if dag is not None and dag is not instance.dag and dag != instance.dag:
            raise ValueError("dag must be the state's instance dag")
        entry = self._entry(instance, cost_model.models, cost_model.topo, cost_model.weights)
        dbank, runner = entry[1], entry[4]
        if runner is None:
            if self._staging is None:
                self._staging = WaveStaging(dbank.torch, dbank.device)
            runner = entry[4] = WaveRunner(dbank, self._staging)
        sids = sorted(frontier)
        r = runner.run(state, sids)
        el = runner.elig[r["stage"] - runner.g0]
        return WaveScores(stage_ids=sids, bounds=r["bounds"].tolist(),
                          device_ids=dbank.packed.device_ids, elig=el.tolist(), psi=r["psi"],
                          psi_off=r["psi_off"], sched=r["sched"],
                          completion=r["completion"], tail=r["tail"], timing=r["timing"])


def wave_scores(packed, sids, work, res) -> WaveScores:
    """Host copies of a scored wave (one D2H per output)."""
    D = packed.scalars["n_devices"]
    n = len(sids)
    host = {k: getattr(res, k).cpu().numpy() for k in ("psi", "sched", "completion", "tail")}
    timing = res.timing.cpu().numpy()[: n * D * 3].reshape(n, D, 3) if res.timing is not None \
        else None
    return WaveScores(
        stage_ids=sids, bounds=[int(b) for b in work.bounds], device_ids=packed.device_ids,
        elig=[int(packed.arrays["st_elig"][g]) for g in work.stage],
        psi=host["psi"][: work.n_psi], psi_off=work.psi_off,
        sched=host["sched"][: n * D].reshape(n, D),
        completion=host["completion"][: n * D].reshape(n, D),
        tail=host["tail"][: n * D].reshape(n, D), timing=timing)


_DEFAULT_SCORER: GpuScorer | None = None


def default_scorer() -> GpuScorer:
    global _DEFAULT_SCORER
    if _DEFAULT_SCORER is None:
        _DEFAULT_SCORER = GpuScorer()
    return _DEFAULT_SCORER


def build_problem(frontier, state, cost_model, dag, scorer: GpuScorer | None = None):
    """GPU replacement of ``wfsched.planner.build_problem`` (planner.py:75-98)."""
    wave = (scorer or default_scorer()).score_wave(frontier, state, cost_model, dag)
    return problem_of(wave, cost_model)


def problem_of(wave: WaveScores, cost_model):
    """The caller's ``FrontierProblem`` of a scored wave (planner.py:93-98)."""
    return _PLANNER.FrontierProblem(candidates=tuple(wave.candidates()),
                                    shard_bounds=dict(zip(wave.stage_ids, wave.bounds)),
                                    device_ids=cost_model.topo.device_ids)


class WaveCostModel:
    """``wfsched.costs.CostModel`` answering from one GPU-scored wave.

    Everything the FATE policy asks its cost model about a wave -- Psi
    (``plan_score``), S (``sched_score``), the tail (``tail_value``) and the
    full-batch ``realized_duration`` -- comes from the GPU outputs of that
    wave; the catalog attributes (``models``, ``topo``, ``weights``) are the
    wrapped model's.  Contract violations raise the reference's ``ValueError``
    (``costs.py:152-153, 242-243, 391-401``); anything the wave did not score
    raises ``KeyError`` instead of silently computing it on the CPU."""

    def __init__(self, cost_model, wave: WaveScores, state):
        self._cm = cost_model
        self._wave = wave
        self._state = state
        self._row = {sid: i for i, sid in enumerate(wave.stage_ids)}
        self._col = {dev: j for j, dev in enumerate(wave.device_ids)}
        self._queries = tuple(q.query_id for q in state.instance.queries)

    def __getattr__(self, name):
        return getattr(self._cm, name)

    def _cell(self, stage, device_id: str, state):
        if state is not self._state:
            raise KeyError("WaveCostModel answers only for the state its wave was scored on")
        if device_id not in stage.eligible_devices:
            raise ValueError(f"device {device_id} not eligible for stage {stage.id}")
        return self._row[stage.id], self._col[device_id]

    def plan_score(self, stage, slot: int, device_id: str, state, dag) -> float:
        if slot >= stage.shard_bound:
            raise ValueError(f"slot {slot} exceeds shard bound of stage {stage.id}")
        i, j = self._cell(stage, device_id, state)
        w = self._wave
        if slot >= w.bounds[i]:
            raise KeyError(f"slot {slot} of {stage.id} was not scored")
        return float(w.psi[int(w.psi_off[i]) + slot * len(w.device_ids) + j])

    def sched_score(self, stage, device_id: str, state, dag) -> float:
        i, j = self._cell(stage, device_id, state)
        return float(self._wave.sched[i, j])

    def tail_value(self, stage, device_id: str, state, dag) -> float:
        if self._cm.weights.effective_horizon() <= 1:
            return 0.0
        i, j = self._cell(stage, device_id, state)
        return float(self._wave.tail[i, j])

    def realized_duration(self, stage, shard_assignment, state, dag=None):
        """Full-batch single-shard timing from the wave (the work-conserving
        fill's only use, policies.py:91-95)."""
        if len(shard_assignment) != 1 or tuple(shard_assignment[0][1]) != self._queries:
            raise KeyError("the wave holds full-batch single-shard timings only")
        device_id = shard_assignment[0][0]
        i, j = self._cell(stage, device_id, state)
        sw, tr, comp = (float(x) for x in self._wave.timing[i, j])
        return [_COSTS.ShardTiming(device_id=device_id, queries=self._queries, switch_s=sw,
                                   transfer_s=tr, compute_s=comp)]


class FateGpuPolicy(_POLICIES.FatePolicy):
    """The caller's ``FatePolicy`` (policies.py:44-193) with its scorer on the
    GPU; drop-in for ``make_policy("fate")``.

    ``solver``: "reference" = the caller's ``wfsched.planner.solve_frontier``
    (default), "native" = ``fate_solve_frontier`` (same result whenever both
    finish and at a zero budget; finishes more problems inside a budget)."""

    name = "fate"

    def __init__(self, solver_budget_s: float = 0.25, scorer: GpuScorer | None = None,
                 solver: str = "reference"):
        if solver not in ("reference", "native"):
            raise ValueError(f"unknown solver {solver!r}")
        super().__init__(solver_budget_s=solver_budget_s)
        self.scorer = scorer or default_scorer()
        self.score_seconds = 0.0
        self.solver = solver
        if solver == "native":
            from .solver import solve_frontier as native

            self._solve = native
        else:
            self._solve = _PLANNER.solve_frontier

    def plan_wave(self, state, frontier, dag, cost_model) -> list:
        """``FatePolicy.plan_wave`` (policies.py:53-76) on one GPU launch."""
        t0 = time.perf_counter()
        wave = self.scorer.score_wave(frontier, state, cost_model, dag)
        self.score_seconds += time.perf_counter() - t0
        view = WaveCostModel(cost_model, wave, state)
        if cost_model.weights.horizon == 0:
            return self._greedy_wave(state, frontier, dag, view)
        problem = problem_of(wave, cost_model)
        solution = self._solve(problem, budget_s=self.solver_budget_s)
        self.solver_stats.record(solution)
        selected = self._extend_work_conserving(solution.selected, problem, state, dag, view)
        if not selected:
            if state.running_tasks:
                return []
            best = min((c for c in problem.candidates if c.slot == 0),
                       key=lambda c: (-c.psi, c.stage_id, c.device_id))
            selected = ((best.stage_id, 0, best.device_id),)
        return self._materialize(selected, state, dag)
