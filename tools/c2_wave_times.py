"""Per-wave time distribution of the drop-in's snapshot path (runtime.WaveRunner)
over the 96 config-2 FATE runs through the reference executor: host packing vs
the GPU round trip (H2D, launch, D2H, synchronize).  Diagnoses run-to-run
variance of bench.py's c2_fate_runs key.   usage: python tools/c2_wave_times.py [reps]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

bench.reference_on_path()
import wfsched.executor as RE  # noqa: E402
import wfsched.harness as RH  # noqa: E402
from wfsched.config import default_config  # noqa: E402

from paper_2605_07238_b200 import runtime  # noqa: E402
from paper_2605_07238_b200.planner import FateGpuPolicy, GpuScorer  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
man = RH.default_manifest()
cfg = default_config(man.num_devices)
reg = RH.materialize_workloads(man, cfg)
keys = sorted(k for k, inst in reg.items() if inst.dag.family not in ("prefix_reuse", "conflict"))
times = []
orig = runtime.WaveRunner.run


events = []
kev = []


def timed(self, st, sids):
    import torch as _t
    e0 = _t.cuda.Event(enable_timing=True)
    e1 = _t.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    r = orig(self, st, sids)
    e1.record()
    times.append(time.perf_counter() - t0)
    events.append((e0, e1, self.inst, len(sids), id(self.dbank)))
    return r


runtime.WaveRunner.run = timed
sub = {"ensure": [], "sync": [], "launch": []}
_ens = runtime.WaveStaging.ensure


def _ensure(self, a, b):
    t0 = time.perf_counter()
    _ens(self, a, b)
    sub["ensure"].append(time.perf_counter() - t0)


runtime.WaveStaging.ensure = _ensure
import torch  # noqa: E402

_sync = torch.cuda.Stream.synchronize


def _tsync(self):
    t0 = time.perf_counter()
    _sync(self)
    sub["sync"].append(time.perf_counter() - t0)


torch.cuda.Stream.synchronize = _tsync
_L = runtime.load_library()
_score = _L.fate_score


class _Lib:
    def __getattr__(self, k):
        return getattr(_L, k)

    def fate_score(self, *a):
        ka = torch.cuda.Event(enable_timing=True)
        kb = torch.cuda.Event(enable_timing=True)
        ka.record()
        t0 = time.perf_counter()
        r = _score(*a)
        sub["launch"].append(time.perf_counter() - t0)
        kb.record()
        kev.append((ka, kb))
        return r


_orig_init = runtime.WaveRunner.__init__


def _init(self, *a, **k):
    _orig_init(self, *a, **k)
    self.L = _Lib()


runtime.WaveRunner.__init__ = _init
cev = []
_copy = torch.Tensor.copy_


def _tcopy(self, src, non_blocking=False):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    r = _copy(self, src, non_blocking=non_blocking)
    b.record()
    cev.append(("h2d" if self.is_cuda else "d2h", a, b))
    return r


if os.environ.get("C2_TIME_COPIES"):
    torch.Tensor.copy_ = _tcopy
import gc  # noqa: E402

gc_pauses = []
_gc_t0 = [0.0]


def _gc_cb(phase, info):
    if phase == "start":
        _gc_t0[0] = time.perf_counter()
    else:
        gc_pauses.append((info.get("generation"), time.perf_counter() - _gc_t0[0]))


gc.callbacks.append(_gc_cb)
if os.environ.get("C2_GC_FREEZE"):
    gc.collect()
    gc.freeze()
sc = GpuScorer()
RE.run(FateGpuPolicy(scorer=sc), reg[keys[0]], cfg)
idle = float(os.environ.get("C2_IDLE_S", "0"))  # GPU-idle seconds before each pass
fresh = bool(os.environ.get("C2_FRESH"))          # a new scorer (bank setup) per pass
for rep in range(reps):
    if idle:
        time.sleep(idle)
    if fresh:
        sc = GpuScorer()
    times.clear()
    events.clear()
    kev.clear()
    cev.clear()
    gc_pauses.clear()
    for v in sub.values():
        v.clear()
    t0 = time.perf_counter()
    for k in keys:
        RE.run(FateGpuPolicy(scorer=sc), reg[k], cfg)
    wall = time.perf_counter() - t0
    a = np.array(times) * 1e3
    torch.cuda.synchronize()
    gpu = np.array([e0.elapsed_time(e1) for e0, e1, *_ in events])
    kt = np.array([x.elapsed_time(y) for x, y in kev])
    for kind in ("h2d", "d2h"):
        ct = np.array([x.elapsed_time(y) for k, x, y in cev if k == kind] or [0.0])
        print(json.dumps({"rep": rep, "copy": kind, "n": int(len(ct)), "sum_ms": float(ct.sum()),
                          "max_ms": float(ct.max()), "p50_ms": float(np.percentile(ct, 50))}),
              flush=True)
    print(json.dumps({"rep": rep, "kernel_ms_sum": float(kt.sum()), "kernel_ms_max": float(kt.max()),
                      "kernel_ms_p50": float(np.percentile(kt, 50)),
                      "kernel_top5": sorted(kt.tolist())[-5:]}), flush=True)
    worst = np.argsort(-a)[:5]
    print(json.dumps({"rep": rep, "worst": [{"wave": int(i), "host_ms": float(a[i]),
                                             "gpu_event_ms": float(gpu[i]),
                                             "n": events[i][3]} for i in worst],
                      "gpu_event_sum_ms": float(gpu.sum()), "gpu_event_max_ms": float(gpu.max())}),
          flush=True)
    print(json.dumps({"rep": rep, "idle_s": idle, "fresh": fresh, "wall_s": wall, "waves": len(a), "sum_ms": float(a.sum()),
                      "p50_ms": float(np.percentile(a, 50)), "p90_ms": float(np.percentile(a, 90)),
                      "p99_ms": float(np.percentile(a, 99)), "max_ms": float(a.max()),
                      "top10_ms": sorted(a.tolist())[-10:],
                      "gc_s": sum(p for _, p in gc_pauses),
                      "gc_max_s": max((p for _, p in gc_pauses), default=0.0),
                      "gc_gen2": sum(1 for g, _ in gc_pauses if g == 2),
                      **{f"{k}_sum_ms": 1e3 * sum(v) for k, v in sub.items()},
                      **{f"{k}_max_ms": 1e3 * max(v, default=0.0) for k, v in sub.items()}}),
          flush=True)
