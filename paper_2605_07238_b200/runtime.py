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
from .pack import PackedBank, PackedStates, WorkList, weights_record

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
    L.fate_prepare.restype = C.c_int
    L.fate_prepare.argtypes = [C.c_void_p] * 5
    L.fate_score.restype = C.c_int
    L.fate_score.argtypes = [C.c_void_p] * 8
    if L.fate_abi_version() != 1:
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
        self.cder = abi.FateDerived(mean_base=self.mean_base.data_ptr(),
                                    demand=self.demand.data_ptr(),
                                    split_penalty=self.split_penalty.data_ptr(),
                                    edge_sigma=self.edge_sigma.data_ptr(),
                                    edge_term=self.edge_term.data_ptr(),
                                    row_sums=self.row_sums.data_ptr(),
                                    inst_qgroups=self.inst_qgroups.data_ptr(),
                                    tail_sum=self.tail_sum.data_ptr(),
                                    tail_static=self.tail_static.data_ptr())
        s = stream or torch.cuda.current_stream(self.device)
        _check(L.fate_prepare(C.byref(self.cbank), C.byref(self.cweights), C.byref(self.cwin),
                              C.byref(self.cder), C.c_void_p(s.cuda_stream)), "fate_prepare")

    # -- per-call inputs -------------------------------------------------------

    def upload_states(self, states: PackedStates, non_blocking: bool = False) -> "DeviceStates":
        return DeviceStates(self, states, non_blocking=non_blocking)

    def upload_work(self, work: WorkList, non_blocking: bool = False) -> "DeviceWork":
        return DeviceWork(self, work, non_blocking=non_blocking)

    def alloc_out(self, work: WorkList, extras: bool = True) -> ScoreResult:
        torch = self.torch
        n_dev = self.packed.scalars["n_devices"]
        f64 = dict(dtype=torch.float64, device=self.device)
        psi = torch.empty(max(work.n_psi, 1), **f64)
        mk = (lambda: torch.empty(max(work.n_items * n_dev, 1), **f64)) if extras else (lambda: None)
        return ScoreResult(psi=psi, sched=mk(), tail=mk(), completion=mk())

    def score_into(self, dstates: "DeviceStates", dwork: "DeviceWork", out: ScoreResult,
                   stream=None) -> ScoreResult:
        torch = self.torch
        s = stream or torch.cuda.current_stream(self.device)
        cout = abi.FateOut(
            psi=out.psi.data_ptr(),
            sched=out.sched.data_ptr() if out.sched is not None else None,
            tail=out.tail.data_ptr() if out.tail is not None else None,
            completion=out.completion.data_ptr() if out.completion is not None else None)
        _check(load_library().fate_score(
            C.byref(self.cbank), C.byref(self.cweights), C.byref(self.cwin), C.byref(self.cder),
            C.byref(dstates.cstate), C.byref(dwork.cwork), C.byref(cout),
            C.c_void_p(s.cuda_stream)), "fate_score")
        return out

    def score(self, states: PackedStates, work: WorkList, extras: bool = True) -> ScoreResult:
        ds = self.upload_states(states)
        dw = self.upload_work(work)
        out = self.alloc_out(work, extras)
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


class HostPipeline:
    """Reference-facing call with HOST buffers: each call copies the step's
    scenario states and work list host->device from pinned memory, scores,
    and copies Psi device->host into pinned memory.  The static bank stays
    HBM-resident (uploaded once, like model weights).

    The batch is split into ``n_chunks`` scenario-aligned chunks issued
    round-robin on ``n_streams`` CUDA streams, so the H2D copy of chunk i+1,
    the scoring of chunk i and the D2H copy of chunk i-1 overlap (copy engines
    and SMs run concurrently).  Items must be scenario-major (as every work
    list built by this package is)."""

    def __init__(self, dbank: DeviceBank, states: PackedStates, work: WorkList,
                 extras: bool = False, n_chunks: int = 8, n_streams: int = 3):
        torch = dbank.torch
        self.dbank = dbank
        D = dbank.packed.scalars["n_devices"]
        cap4 = states.kappa_cap * 4
        sc = np.asarray(work.scen)
        if sc.size and np.any(np.diff(sc) < 0):
            raise ValueError("HostPipeline needs a scenario-major work list")
        if work.n_items and np.any(np.diff(work.psi_off) < 0):
            raise ValueError("HostPipeline needs increasing psi offsets")
        sa = states.arrays
        self.host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
                     for k, v in sa.items()}
        for k in ("scen", "stage", "psi_off"):
            self.host["w:" + k] = torch.from_numpy(
                np.ascontiguousarray(getattr(work, k))).pin_memory()
        self.dev = {k: torch.empty_like(v, device=dbank.device) for k, v in self.host.items()}
        self.cstate = abi.fill_struct(
            abi.FateState(), {"n_scenarios": states.n_scenarios, "kappa_cap": states.kappa_cap},
            {k: self.dev[k].data_ptr() for k in abi.STATE_PTRS})
        self.out = dbank.alloc_out(work, extras=extras)
        self.host_psi = torch.empty(self.out.psi.shape, dtype=torch.float64).pin_memory()
        # scenario-aligned chunks
        n = work.n_items
        bounds = [0]
        if n:
            for c in range(1, n_chunks):
                i = (n * c) // n_chunks
                while 0 < i < n and sc[i] == sc[i - 1]:
                    i += 1
                if bounds[-1] < i < n:
                    bounds.append(i)
            bounds.append(n)
        loc_off = np.asarray(sa["scen_loc_off"])
        n_loc = sa["loc"].size
        self.chunks = []
        for i0, i1 in zip(bounds[:-1], bounds[1:]):
            s0, s1 = int(sc[i0]), int(sc[i1 - 1]) + 1
            l0 = int(loc_off[s0])
            l1 = int(loc_off[s1]) if s1 < states.n_scenarios else n_loc
            p0 = int(work.psi_off[i0])
            p1 = int(work.psi_off[i1]) if i1 < n else work.n_psi
            sl = {"scen_inst": (s0, s1), "scen_clock": (s0, s1), "scen_loc_off": (s0, s1),
                  "scen_done_level": (s0, s1),
                  "loc": (l0, l1), "residency": (s0 * D, s1 * D), "dev_free": (s0 * D, s1 * D),
                  "kappa_n": (s0 * D, s1 * D), "kappa": (s0 * D * cap4, s1 * D * cap4),
                  "w:scen": (i0, i1), "w:stage": (i0, i1), "w:psi_off": (i0, i1)}
            cw = abi.fill_struct(abi.FateWork(), {"n_items": i1 - i0}, {
                k: self.dev["w:" + k].data_ptr() + i0 * self.dev["w:" + k].element_size()
                for k in ("scen", "stage", "psi_off")})
            self.chunks.append((sl, cw, (p0, p1)))
        self.streams = [torch.cuda.Stream(dbank.device) for _ in range(max(1, n_streams))]
        self.h2d_bytes = sum(v.numel() * v.element_size() for v in self.host.values())
        self.d2h_bytes = work.n_psi * 8

    def run(self, stream=None):
        torch = self.dbank.torch
        main = stream or torch.cuda.current_stream(self.dbank.device)
        start = torch.cuda.Event()
        start.record(main)
        d = self.dbank
        L = load_library()
        cout = abi.FateOut(psi=self.out.psi.data_ptr(),
                           sched=self.out.sched.data_ptr() if self.out.sched is not None else None,
                           tail=self.out.tail.data_ptr() if self.out.tail is not None else None,
                           completion=(self.out.completion.data_ptr()
                                       if self.out.completion is not None else None))
        for c, (sl, cw, (p0, p1)) in enumerate(self.chunks):
            s = self.streams[c % len(self.streams)]
            s.wait_event(start)
            with torch.cuda.stream(s):
                for k, (a, b_) in sl.items():
                    if b_ > a:
                        self.dev[k][a:b_].copy_(self.host[k][a:b_], non_blocking=True)
                _check(L.fate_score(C.byref(d.cbank), C.byref(d.cweights), C.byref(d.cwin),
                                    C.byref(d.cder), C.byref(self.cstate), C.byref(cw),
                                    C.byref(cout), C.c_void_p(s.cuda_stream)), "fate_score")
                if p1 > p0:
                    self.host_psi[p0:p1].copy_(self.out.psi[p0:p1], non_blocking=True)
        for s in self.streams:
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        return self.host_psi
