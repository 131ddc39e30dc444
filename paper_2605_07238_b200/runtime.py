"""Device runtime: loads ``libfate.so`` (the sm_100a kernels behind the C ABI of
``include/fate.h``) and drives it with PyTorch-owned device buffers.

There is no CPU fallback: if the library is missing, or CUDA is unavailable,
every entry point raises :class:`FateUnavailable`.  PyTorch is plumbing only
(device memory, streams, pinned host buffers); all scoring arithmetic runs in
the library's kernels.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import abi
from .pack import PackedBank, PackedStates, WorkList, pack_state_into, weights_record

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfate.so")


class FateUnavailable(RuntimeError):
    """The CUDA scorer cannot run here (library not built, or no GPU)."""


class FateError(RuntimeError):
    """A C-ABI call returned a nonzero status."""


_lib = None


def load_library():
    """Load ``libfate.so`` (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FateUnavailable(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    L.fate_abi_version.restype = C.c_int
    L.fate_last_error.restype = C.c_char_p
    L.fate_launch_count.restype = C.c_int64
    L.fate_windows_count_host.restype = C.c_int
    L.fate_windows_count_host.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_int32, C.POINTER(C.c_int64)]
    L.fate_windows_build_host.restype = C.c_int
    L.fate_windows_build_host.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_int32, C.c_void_p, C.c_void_p]
    L.fate_window_parents_host.restype = C.c_int
    L.fate_window_parents_host.argtypes = [C.c_int32, C.c_int32] + [C.c_void_p] * 6 + [
        C.POINTER(C.c_int64)]
    L.fate_template_count.restype = C.c_int
    L.fate_template_count.argtypes = [C.c_void_p] * 6
    L.fate_prepare.restype = C.c_int
    L.fate_prepare.argtypes = [C.c_void_p] * 5
    L.fate_score.restype = C.c_int
    L.fate_score.argtypes = [C.c_void_p] * 8
    L.fate_pipeline_create.restype = C.c_int
    L.fate_pipeline_create.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    L.fate_pipeline_destroy.restype = C.c_int
    L.fate_pipeline_destroy.argtypes = [C.c_void_p]
    L.fate_pipeline_score.restype = C.c_int
    L.fate_pipeline_score.argtypes = [C.c_void_p] * 10
    L.fate_pipeline_capture.restype = C.c_int
    L.fate_pipeline_capture.argtypes = [C.c_void_p] * 9
    L.fate_pipeline_replay.restype = C.c_int
    L.fate_pipeline_replay.argtypes = [C.c_void_p, C.c_void_p]
    L.fate_pipeline_bytes.restype = C.c_int
    L.fate_pipeline_bytes.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.fate_pipeline_device_psi.restype = C.c_int
    L.fate_pipeline_device_psi.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    if L.fate_abi_version() != 3:
        raise FateUnavailable("libfate.so ABI version mismatch")
    _lib = L
    return L


def _check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load_library().fate_last_error().decode(errors="replace")
        if rc < 0:
            raise ValueError(f"{what}: {msg} (status {rc})")
        raise FateError(f"{what}: {msg} (cuda error {rc})")


def launch_count() -> int:
    return int(load_library().fate_launch_count())


def build_windows(packed: PackedBank, levels: int):
    """Horizon-window CSR via the native host builder (cached on the bank)."""
    if levels in packed.windows:
        return packed.windows[levels]
    L = load_library()
    a = packed.arrays
    n = packed.n_stages
    ch_ptr = np.ascontiguousarray(a["ch_ptr"])
    ch_idx = np.ascontiguousarray(a["ch_idx"])
    level = np.ascontiguousarray(a["st_level"])
    cnt = C.c_int64(0)
    _check(L.fate_windows_count_host(n, ch_ptr.ctypes.data, ch_idx.ctypes.data,
                                     level.ctypes.data, levels, C.byref(cnt)), "windows_count")
    ptr = np.zeros(n * levels + 1, dtype=np.int64)
    idx = np.zeros(max(cnt.value, 1), dtype=np.int32)
    _check(L.fate_windows_build_host(n, ch_ptr.ctypes.data, ch_idx.ctypes.data,
                                     level.ctypes.data, levels, ptr.ctypes.data,
                                     idx.ctypes.data), "windows_build")
    packed.windows[levels] = (ptr, idx)
    return ptr, idx


def build_window_parents(packed: PackedBank, levels: int):
    """Distinct window parents per (stage, level) via the native builder."""
    key = ("wpar", levels)
    if key in packed.windows:
        return packed.windows[key]
    L = load_library()
    ptr, idx = build_windows(packed, levels)
    a = packed.arrays
    n = packed.n_stages
    par_ptr = np.ascontiguousarray(a["par_ptr"])
    par_idx = np.ascontiguousarray(a["par_idx"])
    cnt = C.c_int64(0)
    _check(L.fate_window_parents_host(n, levels, ptr.ctypes.data, idx.ctypes.data,
                                      par_ptr.ctypes.data, par_idx.ctypes.data, None, None,
                                      C.byref(cnt)), "window_parents_count")
    wptr = np.zeros(n * levels + 1, dtype=np.int64)
    widx = np.zeros(max(cnt.value, 1), dtype=np.int32)
    _check(L.fate_window_parents_host(n, levels, ptr.ctypes.data, idx.ctypes.data,
                                      par_ptr.ctypes.data, par_idx.ctypes.data, wptr.ctypes.data,
                                      widx.ctypes.data, C.byref(cnt)), "window_parents_build")
    packed.windows[key] = (wptr, widx)
    return wptr, widx


def window_parent_min_level(packed: PackedBank, levels: int) -> np.ndarray:
    """Per (stage, level): the lowest level among the window parents
    (INT32_MAX when the list is empty)."""
    key = ("wpar_min", levels)
    if key in packed.windows:
        return packed.windows[key]
    n = packed.n_stages * levels
    out = np.full(max(n, 1), np.iinfo(np.int32).max, dtype=np.int32)
    if n:
        wptr, widx = build_window_parents(packed, levels)
        cnt = (wptr[1:] - wptr[:-1])
        if int(wptr[-1]) > 0:
            lv = packed.arrays["st_level"][widx[: int(wptr[-1])]]
            nz = cnt > 0
            starts = wptr[:-1][nz]
            out[:n][nz] = np.minimum.reduceat(lv, starts)
    packed.windows[key] = out
    return out


def max_level_ops(packed: PackedBank, levels: int) -> int:
    """Largest per-(stage, level) op count of the tail: sum over the bucket of
    (model op + prefix op + parent edges); sizes the kernel's op buffer."""
    if levels == 0:
        return 0
    key = ("ops", levels)
    if key in packed.windows:
        return packed.windows[key]
    ptr, idx = build_windows(packed, levels)
    a = packed.arrays
    npar = (a["par_ptr"][1:] - a["par_ptr"][:-1]).astype(np.int64)
    n_items = int(ptr[-1])
    if n_items == 0:
        packed.windows[key] = 0
        return 0
    per_item = 2 + npar[idx[:n_items]]
    csum = np.concatenate([[0], np.cumsum(per_item)])
    per_bucket = csum[ptr[1:]] - csum[ptr[:-1]]
    out = int(per_bucket.max()) if per_bucket.size else 0
    packed.windows[key] = out
    return out


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise FateUnavailable("CUDA is not available: the FATE scorer has no CPU path")
    return torch


def _to_dev(torch, arr: np.ndarray, device):
    arr = np.ascontiguousarray(arr)
    if arr.dtype == np.uint64:
        arr = arr.view(np.int64)
    return torch.from_numpy(arr).to(device)


@dataclass
class ScoreResult:
    psi: object          # torch float64 [n_psi]
    sched: object        # torch float64 [W*D] or None
    tail: object
    completion: object
    timing: object = None  # torch float64 [W*D*3] (switch, transfer, compute) or None


class DeviceBank:
    """Static SoA resident in HBM for one (bank, weights) pair, plus the
    prologue tables (windows, mean_base, demand, split penalty, edge terms)."""

    def __init__(self, packed: PackedBank, weights, device=None, stream=None):
        torch = _torch()
        L = load_library()
        self.torch = torch
        self.packed = packed
        self.weights = weights
        self.device = torch.device(device or "cuda")
        self.wrec = weights_record(weights)
        self.cweights = abi.make_weights(self.wrec)
        eff = self.wrec["eff_horizon"]
        self.levels = eff - 1 if eff > 1 else 0
        self.no_shard = bool(self.wrec["ablation"] & 16)
        self.t = {k: _to_dev(torch, v, self.device) for k, v in packed.arrays.items()}
        self.cbank = abi.fill_struct(
            abi.FateBank(),
            {k: packed.scalars[k] for k in abi.BANK_INTS if k in packed.scalars}
            | {"beta_default": packed.scalars["beta_default"]},
            {k: self.t[k].data_ptr() for k in abi.BANK_PTRS})
        ptr, idx = build_windows(packed, self.levels)
        self.win_ptr = _to_dev(torch, ptr, self.device)
        self.win_idx = _to_dev(torch, idx, self.device)
        wptr, widx = build_window_parents(packed, self.levels)
        self.wpar_ptr = _to_dev(torch, wptr, self.device)
        self.wpar_idx = _to_dev(torch, widx, self.device)
        self.wpar_minlvl = _to_dev(torch, window_parent_min_level(packed, self.levels),
                                   self.device)
        self.cwin = abi.FateWindows(levels=self.levels,
                                    max_level_ops=max_level_ops(packed, self.levels),
                                    ptr=self.win_ptr.data_ptr(), idx=self.win_idx.data_ptr(),
                                    wpar_ptr=self.wpar_ptr.data_ptr(),
                                    wpar_idx=self.wpar_idx.data_ptr(),
                                    wpar_minlvl=self.wpar_minlvl.data_ptr())
        n, e = packed.n_stages, packed.scalars["n_edges"]
        f64 = dict(dtype=torch.float64, device=self.device)
        self.mean_base = torch.empty(max(n, 1), **f64)
        self.demand = torch.empty(max(n * self.levels, 1), **f64)
        self.split_penalty = torch.empty(max(n, 1), **f64)
        self.edge_sigma = torch.empty(max(e, 1), **f64)
        self.edge_term = torch.empty(max(e, 1), **f64)
        self.row_sums = torch.empty(max(n * 6, 1), **f64)
        self.inst_qgroups = torch.empty(max(packed.scalars["n_instances"], 1), dtype=torch.int32,
                                        device=self.device)
        self.tail_sum = torch.empty(max(n * (packed.scalars["n_models"] + 1), 1), **f64)
        n_static = n * self.levels * (packed.scalars["n_models"] + 1)
        self.tail_static = torch.empty(max(n_static, 1), **f64)
        self.stage_rec = torch.empty(max(n, 1) * 112, dtype=torch.uint8, device=self.device)
        self.tok_vals = torch.empty(max(n, 1) * 4, dtype=torch.int32, device=self.device)
        self.tok_sums = torch.empty(max(n, 1) * 9, **f64)
        self.cder = abi.FateDerived(mean_base=self.mean_base.data_ptr(),
                                    demand=self.demand.data_ptr(),
                                    split_penalty=self.split_penalty.data_ptr(),
                                    edge_sigma=self.edge_sigma.data_ptr(),
                                    edge_term=self.edge_term.data_ptr(),
                                    row_sums=self.row_sums.data_ptr(),
                                    inst_qgroups=self.inst_qgroups.data_ptr(),
                                    tail_sum=self.tail_sum.data_ptr(),
                                    tail_static=self.tail_static.data_ptr(),
                                    stage_rec=self.stage_rec.data_ptr(),
                                    tok_vals=self.tok_vals.data_ptr(),
                                    tok_sums=self.tok_sums.data_ptr())
        s = stream or torch.cuda.current_stream(self.device)
        # op templates of the tail (v6 kernel): count per (stage, level), scan, fill
        nvl = n * self.levels
        self.tmpl_ptr = torch.zeros(nvl + 1, dtype=torch.int64, device=self.device)
        if nvl:
            counts = torch.empty(nvl, dtype=torch.int64, device=self.device)
            _check(L.fate_template_count(C.byref(self.cbank), C.byref(self.cweights),
                                         C.byref(self.cwin), C.byref(self.cder),
                                         C.c_void_p(counts.data_ptr()), C.c_void_p(s.cuda_stream)),
                   "fate_template_count")
            with torch.cuda.stream(s):
                torch.cumsum(counts, 0, out=self.tmpl_ptr[1:])
        n_tmpl = int(self.tmpl_ptr[-1].item()) if nvl else 0
        if nvl:
            # the longest op template bounds every level's op list; the v6
            # kernel sizes its (chunked) op buffer by min(this, its cap)
            longest = int((self.tmpl_ptr[1:] - self.tmpl_ptr[:-1]).max().item())
            self.cwin.max_level_ops = min(self.cwin.max_level_ops, max(longest, 1))
        self.tmpl = torch.empty(max(n_tmpl, 1) * 16, dtype=torch.uint8, device=self.device)
        self.cder.tmpl_ptr = self.tmpl_ptr.data_ptr()
        self.cder.tmpl = self.tmpl.data_ptr()
        _check(L.fate_prepare(C.byref(self.cbank), C.byref(self.cweights), C.byref(self.cwin),
                              C.byref(self.cder), C.c_void_p(s.cuda_stream)), "fate_prepare")

    # -- per-call inputs -------------------------------------------------------

    def upload_states(self, states: PackedStates, non_blocking: bool = False) -> "DeviceStates":
        return DeviceStates(self, states, non_blocking=non_blocking)

    def upload_work(self, work: WorkList, non_blocking: bool = False) -> "DeviceWork":
        return DeviceWork(self, work, non_blocking=non_blocking)

    def alloc_out(self, work: WorkList, extras: bool = True, timing: bool = False) -> ScoreResult:
        torch = self.torch
        n_dev = self.packed.scalars["n_devices"]
        f64 = dict(dtype=torch.float64, device=self.device)
        psi = torch.empty(max(work.n_psi, 1), **f64)
        mk = (lambda: torch.empty(max(work.n_items * n_dev, 1), **f64)) if extras else (lambda: None)
        tm = torch.empty(max(work.n_items * n_dev * 3, 1), **f64) if timing else None
        return ScoreResult(psi=psi, sched=mk(), tail=mk(), completion=mk(), timing=tm)

    def score_into(self, dstates: "DeviceStates", dwork: "DeviceWork", out: ScoreResult,
                   stream=None) -> ScoreResult:
        torch = self.torch
        s = stream or torch.cuda.current_stream(self.device)
        cout = abi.FateOut(
            psi=out.psi.data_ptr(),
            sched=out.sched.data_ptr() if out.sched is not None else None,
            tail=out.tail.data_ptr() if out.tail is not None else None,
            completion=out.completion.data_ptr() if out.completion is not None else None,
            timing=out.timing.data_ptr() if out.timing is not None else None)
        if hasattr(dwork, "queue_for"):
            dwork.cwork.queue = dwork.queue_for(s)
        _check(load_library().fate_score(
            C.byref(self.cbank), C.byref(self.cweights), C.byref(self.cwin), C.byref(self.cder),
            C.byref(dstates.cstate), C.byref(dwork.cwork), C.byref(cout),
            C.c_void_p(s.cuda_stream)), "fate_score")
        return out

    def score(self, states: PackedStates, work: WorkList, extras: bool = True,
              timing: bool = False) -> ScoreResult:
        ds = self.upload_states(states)
        dw = self.upload_work(work)
        out = self.alloc_out(work, extras, timing)
        return self.score_into(ds, dw, out)


class DeviceStates:
    def __init__(self, dbank: DeviceBank, states: PackedStates, non_blocking: bool = False):
        torch = dbank.torch
        self.states = states
        self.t = {}
        for k, v in states.arrays.items():
            src = torch.from_numpy(np.ascontiguousarray(v))
            self.t[k] = src.to(dbank.device, non_blocking=non_blocking)
        self.cstate = abi.fill_struct(
            abi.FateState(), {"n_scenarios": states.n_scenarios, "kappa_cap": states.kappa_cap},
            {k: self.t[k].data_ptr() for k in abi.STATE_PTRS})


class DeviceWork:
    def __init__(self, dbank: DeviceBank, work: WorkList, non_blocking: bool = False):
        torch = dbank.torch
        self.work = work
        self.t = {k: torch.from_numpy(np.ascontiguousarray(getattr(work, k))).to(
            dbank.device, non_blocking=non_blocking) for k in ("scen", "stage", "psi_off")}
        self.cwork = abi.fill_struct(abi.FateWork(), {"n_items": work.n_items},
                                     {k: v.data_ptr() for k, v in self.t.items()})
        self._torch = torch
        self._device = dbank.device
        self._queues: dict = {}

    def queue_for(self, stream) -> int:
        """This work list's self-resetting ticket counter for launches on
        ``stream`` (fate_work.queue): launches on one stream are ordered, so a
        counter per (work list, stream) is never shared by two launches in
        flight, however many streams and work lists are active."""
        key = int(stream.cuda_stream)
        q = self._queues.get(key)
        if q is None:
            # zero-filled on `stream` itself, so ordered before its first launch
            with self._torch.cuda.stream(stream):
                q = self._queues[key] = self._torch.zeros(2, dtype=self._torch.int32,
                                                          device=self._device)
        return q.data_ptr()


class HostPipeline:
    """Reference-facing call with HOST buffers (``fate_pipeline_score``): each
    call copies the step's scenario states and work list host->device from
    pinned memory (the wire format of ``fate_host_batch``: fixed-size scenario
    records, loc rows, 16-byte items), scores, and copies Psi (and optionally
    S / completion) device->host into pinned memory.  The static bank stays
    HBM-resident (uploaded once, like model weights).

    The native pipeline cuts the batch into ``n_chunks`` scenario-aligned
    chunks issued round-robin on ``n_streams`` CUDA streams, so the H2D copy
    of chunk i+1, the scoring of chunk i and the D2H copy of chunk i-1 overlap
    (copy engines and SMs run concurrently).  Items must be scenario-major (as
    every work list built by this package is).

    ``graph=True`` captures the whole pipeline once into a CUDA graph
    (``fate_pipeline_capture``: validation, chunking and sizing happen once)
    and ``run()`` replays it: one launch per step, no per-copy host work on
    the critical path.  Refill ``h_rec`` / ``h_loc`` / ``h_items`` in place
    between replays to score new inputs of the same shape."""

    def __init__(self, dbank: DeviceBank, states: PackedStates, work: WorkList,
                 extras: bool = False, n_chunks: int = 8, n_streams: int = 1,
                 graph: bool = False):
        from .pack import host_batch

        torch = dbank.torch
        L = load_library()
        self.dbank = dbank
        self.L = L
        D = dbank.packed.scalars["n_devices"]
        hb = host_batch(states, work, D)
        pin = (lambda a: torch.from_numpy(a).pin_memory())
        self.h_rec = pin(hb.rec)
        self.h_loc = pin(hb.loc if hb.loc.size else np.zeros(1, np.int8))
        self.h_items = pin(hb.items.view(np.uint8))
        self.batch = abi.FateHostBatch(
            n_scenarios=hb.n_scenarios, kappa_cap=hb.kappa_cap, n_loc=int(hb.loc.size),
            scen_rec=self.h_rec.data_ptr(), loc=self.h_loc.data_ptr(), n_items=work.n_items,
            n_psi=work.n_psi, items=self.h_items.data_ptr())
        f64 = dict(dtype=torch.float64, pin_memory=True)
        self.host_psi = torch.empty(max(work.n_psi, 1), **f64)
        self.host_sched = torch.empty(max(work.n_items * D, 1), **f64) if extras else None
        self.host_completion = torch.empty(max(work.n_items * D, 1), **f64) if extras else None
        h = C.c_void_p()
        dev = dbank.device.index if dbank.device.index is not None else torch.cuda.current_device()
        _check(L.fate_pipeline_create(dev, n_chunks, n_streams, C.byref(h)),
               "fate_pipeline_create")
        self.handle = h
        self.graph = False
        if graph:
            ptr = (lambda t: C.c_void_p(t.data_ptr()) if t is not None else None)
            _check(L.fate_pipeline_capture(
                self.handle, C.byref(dbank.cbank), C.byref(dbank.cweights), C.byref(dbank.cwin),
                C.byref(dbank.cder), C.byref(self.batch), ptr(self.host_psi),
                ptr(self.host_sched), ptr(self.host_completion)), "fate_pipeline_capture")
            self.graph = True
        self.run()  # sizes the workspaces; records the byte counts
        torch.cuda.synchronize(dbank.device)
        a, b = C.c_int64(0), C.c_int64(0)
        _check(L.fate_pipeline_bytes(self.handle, C.byref(a), C.byref(b)), "fate_pipeline_bytes")
        self.h2d_bytes, self.d2h_bytes = int(a.value), int(b.value)

    def run(self, stream=None):
        torch = self.dbank.torch
        s = stream or torch.cuda.current_stream(self.dbank.device)
        d = self.dbank
        if self.graph:
            _check(self.L.fate_pipeline_replay(self.handle, C.c_void_p(s.cuda_stream)),
                   "fate_pipeline_replay")
            return self.host_psi
        ptr = (lambda t: C.c_void_p(t.data_ptr()) if t is not None else None)
        _check(self.L.fate_pipeline_score(
            self.handle, C.byref(d.cbank), C.byref(d.cweights), C.byref(d.cwin),
            C.byref(d.cder), C.byref(self.batch), ptr(self.host_psi),
            ptr(self.host_sched), ptr(self.host_completion), C.c_void_p(s.cuda_stream)),
            "fate_pipeline_score")
        return self.host_psi

    def device_psi(self):
        """The pipeline's device Psi rows as a torch tensor view (no copy)."""
        torch = self.dbank.torch
        ptr = C.c_void_p()
        _check(self.L.fate_pipeline_device_psi(self.handle, C.byref(ptr)),
               "fate_pipeline_device_psi")
        n = max(int(self.batch.n_psi), 1)

        class _View:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                        "data": (int(ptr.value), False), "version": 3}

        return torch.as_tensor(_View(), device=self.dbank.device)

    def close(self):
        if getattr(self, "handle", None):
            self.L.fate_pipeline_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class WaveStaging:
    """Grow-only staging shared by the :class:`WaveRunner` of every bank of a
    scorer (waves are scored one at a time): one pinned host input block and
    one device input block (``fate_state`` + ``fate_work`` SoA at offsets set
    per wave), one device output block and its pinned host mirror, and the
    ticket counter of the work list (self-resetting, fate_work.queue).
    Pinned allocations are slow, so blocks are reused and only regrown (x2)."""

    def __init__(self, torch, device):
        self.torch = torch
        self.device = device
        self.in_bytes = 0
        self.out_len = 0
        self.queue = torch.zeros(2, dtype=torch.int32, device=device)

    def ensure(self, in_bytes: int, out_len: int) -> None:
        torch = self.torch
        if in_bytes > self.in_bytes or out_len > self.out_len:
            torch.cuda.current_stream(self.device).synchronize()
        if in_bytes > self.in_bytes:
            self.in_bytes = max(in_bytes, 2 * self.in_bytes, 4096)
            self.h_in = torch.empty(self.in_bytes, dtype=torch.uint8, pin_memory=True)
            self.h_in_np = self.h_in.numpy()
            self.d_in = torch.empty(self.in_bytes, dtype=torch.uint8, device=self.device)
        if out_len > self.out_len:
            self.out_len = max(out_len, 2 * self.out_len, 4096)
            self.h_out = torch.empty(self.out_len, dtype=torch.float64, pin_memory=True)
            self.h_out_np = self.h_out.numpy()
            self.d_out = torch.empty(self.out_len, dtype=torch.float64, device=self.device)


class WaveRunner:
    """One scenario of one bank instance, scored per wave with the fewest
    host<->device round trips (the drop-in's hot loop: ``build_problem`` is
    called once per executor wave, reference ``policies.py:62``).

    Per wave: the snapshot is written straight into the pinned staging block
    (``pack.pack_state_into``, the single-scenario form of
    ``pack.pack_states``) with the work list, then one H2D copy, one
    ``fate_score`` launch, one D2H copy of Psi | S | completion | tail |
    timing and one stream synchronize."""

    _IN = (("scen_inst", np.int32, "1"), ("scen_clock", np.float64, "1"),
           ("scen_loc_off", np.int64, "1"), ("scen_done_level", np.int32, "1"),
           ("residency", np.int32, "D"), ("dev_free", np.float64, "D"),
           ("kappa_n", np.int32, "D"), ("kappa", np.int32, "K"), ("loc", np.int32, "N"),
           ("scen", np.int32, "W"), ("stage", np.int32, "W"), ("psi_off", np.int64, "W"))

    def __init__(self, dbank: DeviceBank, staging: WaveStaging, inst: int = 0):
        p = dbank.packed
        self.dbank = dbank
        self.staging = staging
        self.L = load_library()
        self.inst = inst
        self.D = p.scalars["n_devices"]
        self.g0 = int(p.inst_stage_off[inst])
        self.n_local = len(p.stage_ids[inst])
        self.sindex = p.stage_index[inst]
        g = np.arange(self.g0, self.g0 + self.n_local)
        if dbank.no_shard:
            self.bounds = np.ones(self.n_local, dtype=np.int32)
        else:
            from .pack import popcount64

            self.bounds = np.minimum(p.arrays["st_shard"][g],
                                     popcount64(p.arrays["st_elig"][g])).astype(np.int32)
        self.elig = p.arrays["st_elig"][g]
        self.cap = 1

    def _layout(self, cap: int, n_items: int) -> tuple:
        sizes = {"1": 1, "D": self.D, "K": self.D * cap * 4, "N": max(self.n_local, 1),
                 "W": max(n_items, 1)}
        off, offs = 0, {}
        for name, dt, n in self._IN:
            offs[name] = (off, dt, sizes[n])
            off += (sizes[n] * np.dtype(dt).itemsize + 15) & ~15
        return offs, off

    def run(self, st, sids) -> dict:
        """Score the frontier ``sids`` (sorted stage ids) of snapshot ``st``;
        returns host copies: psi (slot-major rows per stage), psi_off, bounds,
        stage (global), sched / completion / tail [n, D], timing [n, D, 3]."""
        stg = self.staging
        torch = stg.torch
        D = self.D
        need = max((len(e) for e in st.prefix_store.values()), default=0)
        if need > 64:
            raise ValueError(f"{need} prefix entries per device exceed 64")
        cap = max(self.cap, need)
        self.cap = cap
        n = len(sids)
        loc = np.fromiter((self.sindex[s] for s in sids), dtype=np.int64, count=n)
        bounds = self.bounds[loc]
        off = np.zeros(n, dtype=np.int64)
        if n:
            np.cumsum(bounds[:-1].astype(np.int64) * D, out=off[1:])
        n_psi = int(bounds.astype(np.int64).sum()) * D
        nd = n * D
        total = n_psi + 6 * nd
        offs, in_bytes = self._layout(cap, n)
        stg.ensure(in_bytes, total)
        buf = stg.h_in_np
        v = {k: buf[o: o + m * np.dtype(dt).itemsize].view(dt) for k, (o, dt, m) in offs.items()}
        pack_state_into(self.dbank.packed, self.inst, st, v, cap)
        v["scen"][:n] = 0
        v["stage"][:n] = loc + self.g0
        v["psi_off"][:n] = off
        base = stg.d_in.data_ptr()
        cstate = abi.FateState(n_scenarios=1, kappa_cap=cap)
        for k in abi.STATE_PTRS:
            setattr(cstate, k, base + offs[k][0])
        cwork = abi.FateWork(n_items=n, scen=base + offs["scen"][0],
                             stage=base + offs["stage"][0], psi_off=base + offs["psi_off"][0],
                             queue=stg.queue.data_ptr())
        o_s, o_c, o_t, o_m = n_psi, n_psi + nd, n_psi + 2 * nd, n_psi + 3 * nd
        ob = stg.d_out.data_ptr()
        cout = abi.FateOut(psi=ob, sched=ob + 8 * o_s, completion=ob + 8 * o_c,
                           tail=ob + 8 * o_t, timing=ob + 8 * o_m)
        s = torch.cuda.current_stream(self.dbank.device)
        d = self.dbank
        stg.d_in[:in_bytes].copy_(stg.h_in[:in_bytes], non_blocking=True)
        if n:
            _check(self.L.fate_score(C.byref(d.cbank), C.byref(d.cweights), C.byref(d.cwin),
                                     C.byref(d.cder), C.byref(cstate), C.byref(cwork),
                                     C.byref(cout), C.c_void_p(s.cuda_stream)), "fate_score")
            stg.h_out[:total].copy_(stg.d_out[:total], non_blocking=True)
        s.synchronize()
        h = stg.h_out_np[:total].copy()
        return {"psi": h[:n_psi], "psi_off": off, "bounds": bounds, "stage": loc + self.g0,
                "sched": h[o_s:o_c].reshape(n, D), "completion": h[o_c:o_t].reshape(n, D),
                "tail": h[o_t:o_m].reshape(n, D), "timing": h[o_m:total].reshape(n, D, 3)}
