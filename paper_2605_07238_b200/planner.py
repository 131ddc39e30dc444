"""Drop-in GPU cost matrix and the FATE policy that consumes it.

* :func:`build_problem` -- same signature and result as the reference
  ``wfsched.planner.build_problem(frontier, state, cost_model, dag)``
  (``pkg/src/wfsched/planner.py:75-98``): one ``Candidate`` per
  (sorted stage, slot < bound, sorted eligible device), Psi bit-identical,
  negative scores retained -- computed by the sm_100a kernel.
* :class:`FateGpuPolicy` -- the reference ``FatePolicy`` (``policies.py:44-193``,
  ``name = "fate"``) with its three scorer consumers on the GPU: the cost
  matrix, the horizon-0 greedy S matrix (``policies.py:129-150``) and the
  work-conserving completion matrix (``policies.py:79-127``).  The frontier
  solve stays on the host (:func:`.wf.frontier.solve_frontier`) and is timed
  separately in ``solver_stats``.

No CPU fallback: without CUDA or ``libfate.so`` these raise
:class:`~paper_2605_07238_b200.runtime.FateUnavailable`.
"""

from __future__ import annotations

import time
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import pack
from .runtime import DeviceBank
from .wf.frontier import Candidate, FrontierProblem, SolverStats, solve_frontier
from .wf.simulate import ScheduledTask, partition_shards


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

    def candidates(self):
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

    def bank_for(self, instance, models, topo, weights) -> DeviceBank:
        key = (id(instance), id(models), id(topo), weights)
        hit = self._banks.get(key)
        if hit is not None and hit[0] is instance:
            self._banks.move_to_end(key)
            return hit[1]
        packed = pack.pack_bank([instance], models, topo)
        dbank = DeviceBank(packed, weights, device=self.device)
        self._banks[key] = (instance, dbank, models, topo)  # strong refs: no id() reuse
        while len(self._banks) > self.max_banks:
            self._banks.popitem(last=False)
        return dbank

    def score_wave(self, frontier, state, cost_model, dag=None) -> WaveScores:
        instance = state.instance
        if dag is not None and dag is not instance.dag and dag != instance.dag:
            raise ValueError("dag must be the state's instance dag")
        dbank = self.bank_for(instance, cost_model.models, cost_model.topo, cost_model.weights)
        packed = dbank.packed
        sids = sorted(frontier)
        states = pack.pack_states(packed, [(0, state)])
        work = pack.make_work(packed, [(0, packed.global_index(0, s)) for s in sids],
                              dbank.no_shard)
        res = dbank.score(states, work, extras=True)
        D = packed.scalars["n_devices"]
        n = len(sids)
        host = {k: getattr(res, k).cpu().numpy() for k in ("psi", "sched", "completion", "tail")}
        return WaveScores(
            stage_ids=sids, bounds=[int(b) for b in work.bounds], device_ids=packed.device_ids,
            elig=[int(packed.arrays["st_elig"][g]) for g in work.stage],
            psi=host["psi"][: work.n_psi], psi_off=work.psi_off,
            sched=host["sched"][: n * D].reshape(n, D),
            completion=host["completion"][: n * D].reshape(n, D),
            tail=host["tail"][: n * D].reshape(n, D))


_DEFAULT_SCORER: GpuScorer | None = None


def default_scorer() -> GpuScorer:
    global _DEFAULT_SCORER
    if _DEFAULT_SCORER is None:
        _DEFAULT_SCORER = GpuScorer()
    return _DEFAULT_SCORER


def build_problem(frontier, state, cost_model, dag, scorer: GpuScorer | None = None):
    """GPU replacement of ``wfsched.planner.build_problem`` (planner.py:75-98)."""
    wave = (scorer or default_scorer()).score_wave(frontier, state, cost_model, dag)
    return _problem_of(wave, cost_model)


def _problem_of(wave: WaveScores, cost_model) -> FrontierProblem:
    return FrontierProblem(candidates=tuple(wave.candidates()),
                           shard_bounds=dict(zip(wave.stage_ids, wave.bounds)),
                           device_ids=tuple(cost_model.topo.device_ids))


class FateGpuPolicy:
    """Frontier planning with GPU horizon-aware scores (reference
    policies.py:44-193); drop-in for ``make_policy("fate")``."""

    name = "fate"

    def __init__(self, solver_budget_s: float = 0.25, scorer: GpuScorer | None = None,
                 solver: str = "python"):
        """``solver``: "python" = the restated reference solve (default: its
        wall-clock behaviour matches the reference's), "native" =
        ``fate_solve_frontier`` (same result whenever both finish or at a zero
        budget; finishes more problems within a budget)."""
        if solver not in ("python", "native"):
            raise ValueError(f"unknown solver {solver!r}")
        self.solver_budget_s = solver_budget_s
        self.solver_stats = SolverStats()
        self.scorer = scorer or default_scorer()
        self.score_seconds = 0.0
        self.solver = solver
        if solver == "native":
            from .solver import solve_frontier as native

            self._solve = native
        else:
            self._solve = solve_frontier

    def plan_wave(self, state, frontier, dag, cost_model) -> list:
        t0 = time.perf_counter()
        wave = self.scorer.score_wave(frontier, state, cost_model, dag)
        self.score_seconds += time.perf_counter() - t0
        queries = tuple(q.query_id for q in state.instance.queries)
        if cost_model.weights.horizon == 0:
            return self._greedy_wave(wave, queries)
        problem = _problem_of(wave, cost_model)
        solution = self._solve(problem, budget_s=self.solver_budget_s)
        self.solver_stats.record(solution)
        chosen = self._fill_idle(solution.selected, problem, wave, state)
        if not chosen:
            if state.running_tasks:
                return []
            top = min((c for c in problem.candidates if c.slot == 0),
                      key=lambda c: (-c.psi, c.stage_id, c.device_id))
            chosen = ((top.stage_id, 0, top.device_id),)
        return self._materialize(chosen, state, dag, queries)

    @staticmethod
    def _fill_idle(selected, problem, wave: WaveScores, state):
        """``_extend_work_conserving`` (policies.py:79-127) on the GPU
        completion matrix: wait + realized full-batch duration per (v, d)."""
        row = {sid: i for i, sid in enumerate(wave.stage_ids)}
        col = {dev: j for j, dev in enumerate(wave.device_ids)}
        done = wave.completion
        chosen = list(selected)
        used = {d for _, _, d in chosen}
        taken = {s for s, _, _ in chosen}
        idle = {d for d, free in state.device_free.items()
                if free <= state.clock + 1e-12 and d not in used}
        while idle:
            pool = [c for c in problem.candidates
                    if c.slot == 0 and c.device_id in idle and c.stage_id not in taken]
            if not pool:
                break
            pick = None
            for c in sorted(pool, key=lambda c: (-c.psi, c.stage_id, c.device_id)):
                i = row[c.stage_id]
                m = wave.elig[i]
                elsewhere = min(float(done[i, j]) for j in range(len(wave.device_ids)) if m >> j & 1)
                if float(done[i, col[c.device_id]]) <= elsewhere + 1e-9:
                    pick = c
                    break
            if pick is None:
                break
            chosen.append((pick.stage_id, 0, pick.device_id))
            idle.discard(pick.device_id)
            taken.add(pick.stage_id)
        return tuple(sorted(chosen))

    @staticmethod
    def _greedy_wave(wave: WaveScores, queries) -> list:
        """Horizon 0: myopic placement by the GPU S matrix (policies.py:129-150)."""
        ranked = []
        for i, sid in enumerate(wave.stage_ids):
            m = wave.elig[i]
            for j, dev in enumerate(wave.device_ids):
                if m >> j & 1:
                    ranked.append((-float(wave.sched[i, j]), sid, dev))
        ranked.sort()
        used: set = set()
        placed: dict = {}
        for _, sid, dev in ranked:
            if sid in placed or dev in used:
                continue
            placed[sid] = dev
            used.add(dev)
        return [ScheduledTask(task_id="", stage_id=s, slot=0, device_id=d, queries=queries)
                for s, d in sorted(placed.items())]

    def _materialize(self, chosen, state, dag, queries) -> list:
        by_stage: dict = {}
        for sid, k, dev in chosen:
            by_stage.setdefault(sid, []).append((k, dev))
        tasks = []
        for sid in sorted(by_stage):
            stage = dag.stages[sid]
            devs = [d for _, d in sorted(by_stage[sid])]
            devs = self._align(stage, devs, queries, state)
            tasks.extend(ScheduledTask(task_id="", stage_id=sid, slot=k, device_id=dev,
                                       queries=shard)
                         for k, (dev, shard) in enumerate(partition_shards(stage, devs, queries)))
        return tasks

    @staticmethod
    def _align(stage, devs, queries, state) -> list:
        """Swap a 2-way split when that keeps more cached query prefix local
        (policies.py:174-193)."""
        if len(devs) != 2:
            return devs
        halves = partition_shards(stage, devs, queries)

        def kept(qids, dev) -> int:
            tot = 0
            for qid in qids:
                q = state.query(qid)
                tot += min(state.cached_tokens(dev, q.prefix_group, stage.model), q.prompt_tokens)
            return tot

        same = kept(halves[0][1], devs[0]) + kept(halves[1][1], devs[1])
        swap = kept(halves[0][1], devs[1]) + kept(halves[1][1], devs[0])
        return [devs[1], devs[0]] if swap > same else devs
