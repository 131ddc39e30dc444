"""Cost-matrix containers and the host-side frontier solve.

Mirrors the types and solver of ``wfsched.planner`` (reference
``pkg/src/wfsched/planner.py:22-260``).  The cost matrix itself is produced on
the GPU (:func:`paper_2605_07238_b200.planner.build_problem`); the solve stays
on the host exactly as in the reference (north star) and is timed
separately.  Semantics preserved bit-for-bit: option enumeration order, the
suffix-nonnegativity filter (which uses Python's builtin ``sum``), memoised
search over device masks, tie-break toward the lexicographically smallest
selection, wall-clock budget with greedy fallback flagged ``optimal=False``.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import NamedTuple


class Candidate(NamedTuple):
    stage_id: str
    slot: int
    device_id: str
    psi: float


@dataclass(frozen=True)
class FrontierProblem:
    candidates: tuple
    shard_bounds: dict
    device_ids: tuple

    def __post_init__(self) -> None:
        known = set(self.device_ids)
        seen = set()
        for c in self.candidates:
            bound = self.shard_bounds.get(c.stage_id)
            if bound is None:
                raise ValueError(f"candidate references unknown stage {c.stage_id}")
            if c.device_id not in known:
                raise ValueError(f"candidate references unknown device {c.device_id}")
            if not 0 <= c.slot < bound:
                raise ValueError(f"candidate slot {c.slot} out of range for {c.stage_id}")
            key = (c.stage_id, c.slot, c.device_id)
            if key in seen:
                raise ValueError(f"duplicate candidate {key}")
            seen.add(key)


@dataclass(frozen=True)
class FrontierSolution:
    selected: tuple
    objective: float
    optimal: bool
    wall_time: float
    nodes_explored: int


@dataclass
class SolverStats:
    solves: int = 0
    optimal: int = 0
    wall_times: list = field(default_factory=list)

    def record(self, solution: FrontierSolution) -> None:
        self.solves += 1
        self.optimal += 1 if solution.optimal else 0
        self.wall_times.append(solution.wall_time)


def _options_for_stage(stage_id, slot_map, device_bit):
    """Every slot->device chain (C2/C3-valid) whose every proper suffix sums
    nonnegative; sorted by triples (reference planner.py:101-147)."""
    found = []
    stack = [(0, 0.0, 0, ())]
    # depth-first in the reference's visiting order: a node is recorded before
    # its children, children in sorted (device, psi) order
    order = []
    while stack:
        slot, value, mask, triples = stack.pop()
        order.append((value, mask, triples))
        row = slot_map.get(slot)
        if row is None:
            continue
        kids = []
        for dev, psi in sorted(row):
            bit = 1 << device_bit[dev]
            if mask & bit:
                continue
            kids.append((slot + 1, value + psi, mask | bit, triples + ((stage_id, slot, dev),)))
        stack.extend(reversed(kids))
    for value, mask, triples in order:
        if not triples:
            continue
        psis = [next(p for dv, p in slot_map[k] if dv == dev) for _, k, dev in triples]
        if all(value - sum(psis[:i]) >= 0.0 for i in range(len(psis))):
            found.append((value, mask, triples))
    found.sort(key=lambda o: o[2])
    return found


def _all_options(problem: FrontierProblem, device_bit):
    grouped: dict = {}
    for c in problem.candidates:
        grouped.setdefault(c.stage_id, {}).setdefault(c.slot, []).append((c.device_id, c.psi))
    return [(sid, _options_for_stage(sid, grouped[sid], device_bit)) for sid in sorted(grouped)]


class _Timeout(Exception):
    pass


def solve_frontier(problem: FrontierProblem, budget_s: float = 0.25) -> FrontierSolution:
    """Optimal (stage, slot, device) selection; ties -> smallest sorted triples
    (reference planner.py:150-214)."""
    if not problem.candidates:
        raise ValueError("solve_frontier requires a nonempty problem")
    started = time.perf_counter()
    device_bit = {d: i for i, d in enumerate(sorted(set(problem.device_ids)))}
    per_stage = _all_options(problem, device_bit)
    n = len(per_stage)
    bound = [0.0] * (n + 1)
    for i in range(n - 1, -1, -1):
        top = max((o[0] for o in per_stage[i][1]), default=0.0)
        bound[i] = bound[i + 1] + max(0.0, top)
    memo: dict = {}
    counter = [0]
    deadline = started + budget_s

    def best(i: int, mask: int):
        counter[0] += 1
        if i == n or bound[i] <= 0.0:
            return 0.0, ()
        hit = memo.get((i, mask))
        if hit is not None:
            return hit
        if time.perf_counter() > deadline:
            raise _Timeout
        val, sel = best(i + 1, mask)
        for value, omask, triples in per_stage[i][1]:
            if omask & mask:
                continue
            sub_val, sub_sel = best(i + 1, mask | omask)
            tot = value + sub_val
            cand = triples + sub_sel
            if tot > val or (tot == val and cand < sel):
                val, sel = tot, cand
        memo[(i, mask)] = (val, sel)
        return val, sel

    try:
        objective, selection = best(0, 0)
        optimal = True
    except _Timeout:
        objective, selection = _greedy(per_stage)
        optimal = False
    return FrontierSolution(selected=tuple(sorted(selection)), objective=objective,
                            optimal=optimal, wall_time=time.perf_counter() - started,
                            nodes_explored=counter[0])


def _greedy(per_stage):
    """Deadline fallback (reference planner.py:217-234)."""
    ranked = sorted(per_stage, key=lambda so: (-max((o[0] for o in so[1]), default=0.0), so[0]))
    used = 0
    total = 0.0
    picked: tuple = ()
    for _, opts in ranked:
        ok = [o for o in opts if o[0] > 0 and not o[1] & used]
        if not ok:
            continue
        value, mask, triples = min(ok, key=lambda o: (-o[0], o[2]))
        used |= mask
        total += value
        picked += triples
    return total, tuple(sorted(picked))


def check_constraints(problem: FrontierProblem, selection) -> list:
    """C1-C4 violations of a selection (reference planner.py:237-260)."""
    out = []
    allowed = {(c.stage_id, c.slot, c.device_id) for c in problem.candidates}
    dev_use: dict = {}
    slot_use: dict = {}
    slots: dict = {}
    for sid, k, dev in selection:
        dev_use[dev] = dev_use.get(dev, 0) + 1
        slot_use[(sid, k)] = slot_use.get((sid, k), 0) + 1
        slots.setdefault(sid, set()).add(k)
        if (sid, k, dev) not in allowed:
            out.append(f"C4: {(sid, k, dev)} not an eligible candidate")
    out += [f"C1: device {d} assigned {n} slots" for d, n in sorted(dev_use.items()) if n > 1]
    out += [f"C2: slot {key} assigned {n} devices" for key, n in sorted(slot_use.items()) if n > 1]
    for sid, ks in sorted(slots.items()):
        out += [f"C3: stage {sid} enables slot {k} without slot {k - 1}"
                for k in ks if k > 0 and k - 1 not in ks]
    return out
