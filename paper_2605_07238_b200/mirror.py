"""Device-resident incremental execution-state mirror + GPU ready set
(``csrc/fate_mirror.cu``).

The reference snapshots the whole ``ExecutionState`` every wave
(``executor.py:200``) and the scorer would repack and re-upload it.  Here the
state of the running instance stays in HBM: :class:`DeviceMirror` follows the
live state's transitions (``commit_stage``, ``on_task_start``,
``on_task_complete``; reference ``state.py:130-181``) as events, applies them
on the device once per wave, and hands ``fate_score`` the mirror itself as its
one-scenario ``fate_state``.  :class:`MirrorScorer` is a drop-in for
``planner.GpuScorer`` that scores from the mirror; ``compat.install(mirror=...)``
hooks it into the unchanged reference executor.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi, pack
from .planner import GpuScorer, WaveScores, wave_scores
from .runtime import DeviceBank, _check, load_library

EV_COMMIT, EV_START, EV_COMPLETE = 0, 1, 2


class _Event(C.Structure):
    _fields_ = [("kind", C.c_int32), ("stage", C.c_int32), ("device", C.c_int32),
                ("slots", C.c_int32), ("time", C.c_double), ("q0", C.c_int32),
                ("nq", C.c_int32)]


def _lib():
    L = load_library()
    if not getattr(L, "_mirror_bound", False):
        L.fate_mirror_create.restype = C.c_int
        L.fate_mirror_create.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                         C.c_void_p, C.c_int32, C.c_void_p,
                                         C.POINTER(C.c_void_p)]
        L.fate_mirror_destroy.restype = C.c_int
        L.fate_mirror_destroy.argtypes = [C.c_void_p]
        L.fate_mirror_apply.restype = C.c_int
        L.fate_mirror_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                        C.c_int32, C.c_void_p]
        L.fate_mirror_state.restype = C.c_int
        L.fate_mirror_state.argtypes = [C.c_void_p, C.c_void_p]
        L.fate_mirror_ready.restype = C.c_int
        L.fate_mirror_ready.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32),
                                        C.c_void_p]
        L._mirror_bound = True
    return L


class DeviceMirror:
    """The scorer state of one running instance, resident on the GPU."""

    def __init__(self, dbank: DeviceBank, inst_index: int = 0, kappa_cap: int = 16):
        torch = dbank.torch
        L = _lib()
        self.dbank = dbank
        self.L = L
        packed = dbank.packed
        inst = packed.instances[inst_index]
        self.inst_index = inst_index
        self.sindex = packed.stage_index[inst_index]
        self.stage_ids = packed.stage_ids[inst_index]
        self.goff = int(packed.inst_stage_off[inst_index])
        self.dev_index = packed.dev_index
        self.qindex = {q.query_id: i for i, q in enumerate(inst.queries)}
        qg = np.array([packed.group_id(q.prefix_group) for q in inst.queries] or [-1],
                      dtype=np.int32)
        qt = np.array([int(inst.prefix_groups.get(q.prefix_group, q.prompt_tokens))
                       if q.prefix_group is not None else 0 for q in inst.queries] or [0],
                      dtype=np.int32)
        self.kappa_cap = kappa_cap
        h = C.c_void_p()
        s = torch.cuda.current_stream(dbank.device)
        _check(L.fate_mirror_create(C.byref(dbank.cbank), inst_index, kappa_cap,
                                    qg.ctypes.data, qt.ctypes.data, packed.model_id(""),
                                    C.c_void_p(s.cuda_stream), C.byref(h)), "fate_mirror_create")
        self.handle = h
        self.cstate = abi.FateState()
        _check(L.fate_mirror_state(self.handle, C.byref(self.cstate)), "fate_mirror_state")
        self.pending: list = []
        self.pending_q: list = []
        n = len(self.stage_ids)
        self._ready = torch.empty(max(n, 1), dtype=torch.int32, device=dbank.device)
        self.events_applied = 0

    # -- following the live state -------------------------------------------------

    def attach(self, state) -> None:
        """Record the live state's transitions (call the original, then log)."""
        commit, start, complete = state.commit_stage, state.on_task_start, state.on_task_complete

        def commit_stage(stage_id, total_slots):
            commit(stage_id, total_slots)
            self.pending.append((EV_COMMIT, self._g(stage_id), -1, int(total_slots), 0.0, 0, 0))

        def on_task_start(task):
            start(task)
            self.pending.append((EV_START, self._g(task.stage_id), self.dev_index[task.device_id],
                                 0, float(task.finish_time), 0, 0))

        def on_task_complete(task, finish):
            complete(task, finish)
            q0 = len(self.pending_q)
            self.pending_q += [self.qindex[q] for q in task.queries]
            self.pending.append((EV_COMPLETE, self._g(task.stage_id),
                                 self.dev_index[task.device_id], 0, float(finish), q0,
                                 len(task.queries)))

        state.commit_stage = commit_stage
        state.on_task_start = on_task_start
        state.on_task_complete = on_task_complete

    def _g(self, stage_id) -> int:
        return self.goff + self.sindex[stage_id]

    def flush(self, stream=None) -> None:
        if not self.pending:
            return
        torch = self.dbank.torch
        s = stream or torch.cuda.current_stream(self.dbank.device)
        ev = (_Event * len(self.pending))(*[_Event(*e) for e in self.pending])
        q = np.array(self.pending_q or [0], dtype=np.int32)
        _check(self.L.fate_mirror_apply(self.handle, C.cast(ev, C.c_void_p), len(self.pending),
                                        q.ctypes.data, len(self.pending_q),
                                        C.c_void_p(s.cuda_stream)), "fate_mirror_apply")
        # the host arrays must outlive the async copy
        torch.cuda.current_stream(self.dbank.device).synchronize()
        self.events_applied += len(self.pending)
        self.pending, self.pending_q = [], []

    def ready(self, stream=None) -> list:
        """GPU ready set (reference model.py:306-319), as sorted stage ids."""
        self.flush(stream)
        torch = self.dbank.torch
        s = stream or torch.cuda.current_stream(self.dbank.device)
        n = C.c_int32(0)
        _check(self.L.fate_mirror_ready(self.handle, C.c_void_p(self._ready.data_ptr()),
                                        C.byref(n), C.c_void_p(s.cuda_stream)), "fate_mirror_ready")
        # the kernel compacts per warp in completion order; ids ascend after a sort
        idx = np.sort(self._ready[: n.value].cpu().numpy())
        return [self.stage_ids[int(g) - self.goff] for g in idx]

    def download(self) -> dict:
        """Host copy of the mirror's fate_state arrays (tests)."""
        self.flush()
        D = self.dbank.packed.scalars["n_devices"]
        n = len(self.stage_ids)
        cs = self.cstate
        out = {}
        for name, count, typestr in (
                ("residency", D, "<i4"), ("dev_free", D, "<f8"), ("kappa_n", D, "<i4"),
                ("kappa", D * cs.kappa_cap * 4, "<i4"), ("loc", max(n, 1), "<i4"),
                ("scen_clock", 1, "<f8"), ("scen_done_level", 1, "<i4")):
            out[name] = _device_view(self.dbank.torch, getattr(cs, name), count, typestr)
        return out

    def close(self):
        if getattr(self, "handle", None):
            self.L.fate_mirror_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _device_view(torch, ptr: int, count: int, typestr: str) -> np.ndarray:
    """Host copy of ``count`` elements at a raw device pointer (through a
    zero-copy __cuda_array_interface__ view)."""

    class _View:
        __cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                    "data": (int(ptr), False), "version": 3}

    torch.cuda.synchronize()
    return torch.as_tensor(_View(), device="cuda").cpu().numpy().copy()


class MirrorScorer(GpuScorer):
    """``GpuScorer`` drop-in that scores from the device-resident mirror of the
    running instance instead of packing the per-wave snapshot.  Pass it both as
    the policy's scorer and to ``compat.install(mirror=scorer)``, which attaches
    the reference executor's live state to it."""

    def __init__(self, device=None, kappa_cap: int = 16, check_ready: bool = False,
                 gpu_frontier: bool = False):
        """``check_ready``: assert the GPU ready set equals the executor's
        frontier every wave.  ``gpu_frontier``: the executor takes each wave's
        frontier from the GPU ready set (``frontier()``) once the mirror exists
        (from the first scored wave on)."""
        super().__init__(device=device)
        self.kappa_cap = kappa_cap
        self.check_ready = check_ready
        self.provides_frontier = gpu_frontier
        self.mirror: DeviceMirror | None = None
        self._instance = None
        self._live = None
        self.ready_checks = 0
        self.gpu_frontiers = 0

    def attach_live(self, state) -> None:
        """Follow a live executor state.  The device mirror is created at the
        first scored wave (when the catalog is known); the executor commits
        nothing before its first wave, so no transition is missed."""
        if self.mirror is not None:
            self.mirror.close()
            self.mirror = None
        self._live = state
        self._instance = state.instance

    def _ensure_mirror(self, cost_model) -> None:
        if self.mirror is None and self._live is not None:
            dbank = self.bank_for(self._instance, cost_model.models, cost_model.topo,
                                  cost_model.weights)
            self.mirror = DeviceMirror(dbank, 0, self.kappa_cap)
            self.mirror.attach(self._live)

    def follows(self, dag) -> bool:
        return self.mirror is not None and self._instance is not None and \
            self._instance.dag is dag

    def frontier(self) -> set:
        """The next wave's frontier: the GPU ready set (model.py:306-319)."""
        self.gpu_frontiers += 1
        return set(self.mirror.ready())

    def score_wave(self, frontier, state, cost_model, dag=None) -> WaveScores:
        if self._live is None or state.instance is not self._instance:
            return super().score_wave(frontier, state, cost_model, dag)
        self._ensure_mirror(cost_model)
        dbank = self.mirror.dbank
        packed = dbank.packed
        m = self.mirror
        m.flush()
        if self.check_ready:
            got = m.ready()
            if set(got) != set(frontier):
                raise AssertionError(f"GPU ready set {got} != executor frontier {sorted(frontier)}")
            self.ready_checks += 1
        sids = sorted(frontier)
        work = pack.make_work(packed, [(0, packed.global_index(0, s)) for s in sids],
                              dbank.no_shard)
        dwork = dbank.upload_work(work)
        out = dbank.alloc_out(work, extras=True, timing=True)

        class _S:
            cstate = m.cstate

        res = dbank.score_into(_S, dwork, out)
        return wave_scores(packed, sids, work, res)
