"""Native host frontier solve (``fate_solve_frontier``), drop-in for
``wfsched.planner.solve_frontier`` (reference ``pkg/src/wfsched/planner.py:150-214``).

Same signature, the caller's ``wfsched.planner.FrontierSolution`` (selection,
objective bits, ``optimal`` flag, ``nodes_explored``); the option enumeration,
memoised search, tie-break and greedy fallback run in C++
(``csrc/fate_solver.cpp``).  Only ``wall_time`` -- and therefore which
problems finish inside a wall-clock budget -- differs from the Python solver;
``budget_s=0`` reproduces the reference's zero-budget result exactly and a
budget both finish in gives the identical optimal selection.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .runtime import _check, load_library


class _Frontier(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("n_devices", C.c_int32), ("slot_ptr", C.c_void_p),
                ("cand_ptr", C.c_void_p), ("cand_dev", C.c_void_p), ("cand_psi", C.c_void_p)]


class _Selection(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("n", C.c_int32), ("stage", C.c_void_p),
                ("slot", C.c_void_p), ("device", C.c_void_p), ("objective", C.c_double),
                ("optimal", C.c_int32), ("reserved", C.c_int32), ("nodes", C.c_int64),
                ("n_options", C.c_int64), ("wall_s", C.c_double)]


def _lib():
    L = load_library()
    if not getattr(L, "_solver_bound", False):
        L.fate_solve_frontier.restype = C.c_int
        L.fate_solve_frontier.argtypes = [C.POINTER(_Frontier), C.c_double, C.c_int64,
                                          C.POINTER(_Selection)]
        L._solver_bound = True
    return L


def pack_problem(problem):
    """FrontierProblem -> (stage ids, device ids, CSR arrays) in the order the
    reference's ``_stage_options`` visits them."""
    devices = sorted(set(problem.device_ids))
    dev_index = {d: i for i, d in enumerate(devices)}
    by_stage: dict = {}
    for c in problem.candidates:
        by_stage.setdefault(c.stage_id, {}).setdefault(c.slot, []).append(
            (dev_index[c.device_id], c.psi))
    stages = sorted(by_stage)
    slot_ptr = [0]
    cand_ptr = [0]
    cand_dev: list = []
    cand_psi: list = []
    for sid in stages:
        slots = by_stage[sid]
        top = max(slots)
        for k in range(top + 1):
            row = sorted(slots.get(k, ()))
            cand_dev += [d for d, _ in row]
            cand_psi += [p for _, p in row]
            cand_ptr.append(len(cand_dev))
        slot_ptr.append(len(cand_ptr) - 1)
    arrays = (np.asarray(slot_ptr, dtype=np.int32), np.asarray(cand_ptr, dtype=np.int32),
              np.asarray(cand_dev, dtype=np.int32), np.asarray(cand_psi, dtype=np.float64))
    return stages, devices, arrays


def solve_frontier(problem, budget_s: float = 0.25, max_options: int = 0):
    """``wfsched.planner.solve_frontier`` (planner.py:150-214) natively."""
    from wfsched.planner import FrontierSolution

    if not problem.candidates:
        raise ValueError("solve_frontier requires a nonempty problem")
    L = _lib()
    stages, devices, (slot_ptr, cand_ptr, cand_dev, cand_psi) = pack_problem(problem)
    fr = _Frontier(n_stages=len(stages), n_devices=len(devices),
                   slot_ptr=slot_ptr.ctypes.data, cand_ptr=cand_ptr.ctypes.data,
                   cand_dev=cand_dev.ctypes.data, cand_psi=cand_psi.ctypes.data)
    cap = max(len(devices), 1)
    st = np.zeros(cap, dtype=np.int32)
    sl = np.zeros(cap, dtype=np.int32)
    dv = np.zeros(cap, dtype=np.int32)
    out = _Selection(capacity=cap, stage=st.ctypes.data, slot=sl.ctypes.data,
                     device=dv.ctypes.data)
    _check(L.fate_solve_frontier(C.byref(fr), float(budget_s), int(max_options), C.byref(out)),
           "fate_solve_frontier")
    sel = tuple((stages[int(st[k])], int(sl[k]), devices[int(dv[k])]) for k in range(out.n))
    return FrontierSolution(selected=sel, objective=float(out.objective),
                            optimal=bool(out.optimal), wall_time=float(out.wall_s),
                            nodes_explored=int(out.nodes))


class _BatchArgs(C.Structure):
    _fields_ = [("n_problems", C.c_int32), ("n_devices", C.c_int32), ("item_ptr", C.c_void_p),
                ("item_bound", C.c_void_p), ("item_elig", C.c_void_p), ("psi_off", C.c_void_p),
                ("psi", C.c_void_p), ("budget_s", C.c_double), ("max_options", C.c_int64),
                ("n_threads", C.c_int32), ("reserved", C.c_int32)]


class _BatchOut(C.Structure):
    _fields_ = [("n_sel", C.c_void_p), ("sel", C.c_void_p), ("objective", C.c_void_p),
                ("optimal", C.c_void_p), ("wall_s", C.c_double), ("threads", C.c_int32),
                ("reserved", C.c_int32)]


class BatchSolution:
    """Per problem: selected (work item, slot, device) triples, objective,
    optimal flag; plus the batch's wall time and thread count."""

    def __init__(self, n_sel, sel, objective, optimal, wall_s, threads):
        self.n_sel, self.sel, self.objective, self.optimal = n_sel, sel, objective, optimal
        self.wall_s, self.threads = wall_s, threads

    def selected(self, p: int) -> np.ndarray:
        return self.sel[p, : self.n_sel[p]]


def solve_batch(item_ptr, item_bound, item_elig, psi_off, psi, n_devices: int,
                budget_s: float = 0.0, n_threads: int = 0, max_options: int = 0) -> BatchSolution:
    """``fate_solve_batch``: every problem of a scored batch solved on host
    threads (problem p = work items ``item_ptr[p]:item_ptr[p+1]``, in stage
    order; ``psi`` the host copy of the batch's Psi rows)."""
    L = load_library()
    if not getattr(L, "_batch_bound", False):
        L.fate_solve_batch.restype = C.c_int
        L.fate_solve_batch.argtypes = [C.POINTER(_BatchArgs), C.POINTER(_BatchOut)]
        L._batch_bound = True
    item_ptr = np.ascontiguousarray(item_ptr, dtype=np.int32)
    item_bound = np.ascontiguousarray(item_bound, dtype=np.int32)
    item_elig = np.ascontiguousarray(item_elig, dtype=np.uint64)
    psi_off = np.ascontiguousarray(psi_off, dtype=np.int64)
    psi = np.ascontiguousarray(psi, dtype=np.float64)
    n = len(item_ptr) - 1
    n_sel = np.zeros(max(n, 1), dtype=np.int32)
    sel = np.zeros((max(n, 1), n_devices, 3), dtype=np.int32)
    obj = np.zeros(max(n, 1), dtype=np.float64)
    opt = np.zeros(max(n, 1), dtype=np.int32)
    a = _BatchArgs(n_problems=n, n_devices=n_devices, item_ptr=item_ptr.ctypes.data,
                   item_bound=item_bound.ctypes.data, item_elig=item_elig.ctypes.data,
                   psi_off=psi_off.ctypes.data, psi=psi.ctypes.data, budget_s=float(budget_s),
                   max_options=int(max_options), n_threads=int(n_threads))
    o = _BatchOut(n_sel=n_sel.ctypes.data, sel=sel.ctypes.data, objective=obj.ctypes.data,
                  optimal=opt.ctypes.data)
    _check(L.fate_solve_batch(C.byref(a), C.byref(o)), "fate_solve_batch")
    return BatchSolution(n_sel[:n], sel[:n], obj[:n], opt[:n], float(o.wall_s), int(o.threads))
