#!/usr/bin/env python
"""FATE candidate-scoring benchmark (B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fate|reference]
                    [--workload c5|c4] [--mode frontier|sweep] [--gather]

One *step* = one pass of the hot path (horizon-aware candidate scoring +
state-conditional cost estimation, i.e. ``build_problem``'s Psi matrix plus
the S and completion matrices) over one batch of synthetic input.

Default workload (BASELINE.json configs[4], "c5"): 4096 independent
synthetic workflow instances (500 stages, 32 devices, H=3) per GPU, one
canonical scenario state each, every ready-frontier (stage x slot x device)
candidate scored -- 5.72 M Psi per GPU per step.  Multi-GPU: one process per
GPU (torchrun), each rank scores its own 4096 instances (instance seeds offset
by rank): independent units, no data-path collective, weak scaling.
``--gather`` adds an NCCL all-gather of the per-rank Psi slabs to every rank.

Also measured in the same run (N=1): config 4 ("c4_sweep": the 10k-stage,
64-device, 8-model, H=4 DAG, all stages x 8 scenario states, 9.0 M Psi per
step), the north-star roofline kernel.

Timing: CUDA events on the launching stream around each scoring launch,
inputs HBM-resident, L2 flushed (256 MiB write) between steps outside the
events; max over ranks.  ``e2e`` = the same work through the host-buffer call
``fate_pipeline`` (pinned H2D of the step's scenario records, loc rows and
work items, unpack + scoring kernels, D2H of Psi), captured once into a CUDA
graph and replayed every step.
``cpu_baseline`` / ``--impl reference`` = the C oracle port of the
reference scorer on the host cores (test-infrastructure checker, never the
product path).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "candidate assignments scored/sec (stage×device×horizon)"
UNIT = "candidates/s"
PER_GPU_INSTANCES = 4096
C5_SHAPE = dict(depth=20, width=25, density=0.12, batch=16)
C4_SCENARIOS = 8
HBM_FALLBACK_GBS = 6650.0


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def shard_plan(rank: int, world: int, per_gpu: int = PER_GPU_INSTANCES) -> dict:
    """Weak scaling: rank r owns instances [r*per_gpu, (r+1)*per_gpu); config-5
    instance i uses synth seed 1000+i and scenario seed i."""
    first = rank * per_gpu
    return {"first": first, "count": per_gpu, "seed0": 1000 + first, "scen0": first}


def reduce_max(value: float, world: int, device=None) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(value: float, world: int, device=None) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_slabs(psi, world: int):
    """NCCL all-gather of per-rank Psi slabs (padded to the largest)."""
    import torch
    import torch.distributed as dist

    n = torch.tensor([psi.numel()], dtype=torch.int64, device=psi.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    m = int(max(int(s.item()) for s in sizes))
    pad = torch.full((m,), float("nan"), dtype=psi.dtype, device=psi.device)
    pad[: psi.numel()] = psi
    out = torch.empty(world * m, dtype=psi.dtype, device=psi.device)
    dist.all_gather_into_tensor(out, pad)
    return out, [int(s.item()) for s in sizes]


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML polling thread)
# ---------------------------------------------------------------------------


class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, index: int):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception as exc:  # pragma: no cover - depends on the box
            self.error = str(exc)

    def _loop(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self) -> dict:
        if not self._ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "samples": 0}
        s = sorted(self.samples)
        names = [n for n, bit in self.REASONS.items() if self.reasons & bit]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(s)}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------


def build_c5(rank: int, world: int, mode: str):
    from paper_2605_07238_b200 import fastgen, pack, scenarios

    plan = shard_plan(rank, world)
    cfg = scenarios.config_c5()
    fb = fastgen.synth_batch(cfg, plan["count"], plan["seed0"], plan["scen0"],
                             C5_SHAPE["depth"], C5_SHAPE["width"], C5_SHAPE["density"],
                             C5_SHAPE["batch"])
    sc, g = fb.frontier_items() if mode == "frontier" else fb.sweep_items()
    work = pack.make_work(fb.bank, zip(sc.tolist(), g.tolist()), cfg.weights.ablation.no_shard)
    return cfg, fb.bank, fb.states, work, plan


def build_c4(mode: str = "sweep", n_scen: int = C4_SCENARIOS, first_scen: int = 0):
    """Config 4 from the native generator: one 10k-stage instance (seed 1),
    scenario states s = first_scen .. first_scen+n_scen-1 (ranks shard the
    scenario seeds)."""
    import numpy as np

    from paper_2605_07238_b200 import fastgen, pack, scenarios

    cfg = scenarios.config_c4_catalog()
    parts = [fastgen.synth_batch(cfg, 1, 1, s, 100, 100, 0.03, 16)
             for s in range(first_scen, first_scen + n_scen)]
    bank = parts[0].bank
    cap = max(p.states.kappa_cap for p in parts)
    arrays = {}
    for k in parts[0].states.arrays:
        arrays[k] = np.concatenate([p.states.arrays[k] for p in parts])
    arrays["scen_inst"][:] = 0
    arrays["scen_loc_off"][:] = 0
    V, D = bank.n_stages, bank.scalars["n_devices"]
    kap = [p.states.arrays["kappa"].reshape(D, p.states.kappa_cap, 4) for p in parts]
    kk = np.zeros((n_scen, D, cap, 4), dtype=np.int32)
    for s, a in enumerate(kap):
        kk[s, :, : a.shape[1]] = a
    arrays["kappa"] = kk.ravel()
    arrays["loc"] = np.concatenate([p.states.arrays["loc"] for p in parts])
    arrays["scen_loc_off"] = (np.arange(n_scen, dtype=np.int64) * V)
    states = pack.PackedStates(arrays=arrays, n_scenarios=n_scen, kappa_cap=cap)
    items = []
    for s, p in enumerate(parts):
        if mode == "sweep":
            items += [(s, g) for g in range(V)]
        else:
            _, g = p.frontier_items()
            items += [(s, int(x)) for x in g]
    work = pack.make_work(bank, items, cfg.weights.ablation.no_shard)
    return cfg, bank, states, work


# ---------------------------------------------------------------------------
# measurement
# ---------------------------------------------------------------------------


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def traffic_for(key: str):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


def issue_ceiling(key: str, ms: float, sm_mhz) -> dict | None:
    """The binding ceiling of this gather/fp64 kernel: warp-instruction issue.
    Instructions per launch come from the committed ncu capture
    (profiles/ncu_instructions.json, smsp__inst_executed.sum); the peak is
    148 SMs x 4 schedulers x 1 warp-instruction per cycle at the sampled SM
    clock."""
    path = os.path.join(ROOT, "profiles", "ncu_instructions.json")
    try:
        with open(path) as fh:
            inst = json.load(fh).get(key)
    except Exception:
        inst = None
    if not inst or not sm_mhz:
        return None
    peak = 148 * 4 * float(sm_mhz) * 1e6
    achieved = inst / (ms / 1e3)
    out = {"bound": "issue", "warp_instructions_per_launch": inst,
           "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "G warp-inst/s",
           "frac": achieved / peak, "source": "profiles/ncu_instructions.json"}
    # single-pipe ceilings measured by tools/issue_probe.cu on this pool's B200
    # (the integer ALU and FP64 pipes each retire a warp instruction every
    # other cycle per scheduler; a mixed stream is needed to pass ~52 %)
    try:
        with open(os.path.join(ROOT, "profiles", "r01_issue_probe.json")) as fh:
            probe = json.load(fh)
        out["measured_pipes"] = {k: probe[k] for k in
                                 ("int_issue_ginst_s", "dadd_ginst_s",
                                  "walk_fma01_warp_ops_g_per_s") if k in probe}
        out["measured_pipes"]["source"] = "profiles/r01_issue_probe.json"
    except Exception:
        pass
    return out


def time_device(torch, dbank, dstates, dwork, out, steps, warmup, flush, world, device,
                gather=False, clocks=None):
    """Per-step kernel time (CUDA events on the launching stream), L2 flushed
    between steps outside the events.  Returns (ms_per_step, launches)."""
    import torch.distributed as dist

    from paper_2605_07238_b200 import runtime

    stream = torch.cuda.current_stream(device)
    for _ in range(warmup):
        flush.fill_(1.0)
        dbank.score_into(dstates, dwork, out)
        if gather:
            gather_slabs(out.psi, world)
    torch.cuda.synchronize(device)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)
    launches0 = runtime.launch_count()
    ctx = clocks if clocks is not None else _Null()
    with ctx:
        for i in range(steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            dbank.score_into(dstates, dwork, out)
            if gather:
                gather_slabs(out.psi, world)
            ev[i][1].record(stream)
        torch.cuda.synchronize(device)
    launches = runtime.launch_count() - launches0
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    return ms, launches


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def time_e2e(torch, pipe, steps, warmup, world, device, blocks: int = 5):
    """ms per step of the host-buffer pipeline: ``steps`` back-to-back replays
    timed with CUDA events in ``blocks`` equal blocks; the median block is
    reported (PCIe transfers see occasional host-side hiccups) together with
    every block's value."""
    import torch.distributed as dist

    stream = torch.cuda.current_stream(device)
    for _ in range(warmup):
        pipe.run()
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)
    per = max(1, steps // blocks)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(blocks + 1)]
    ev[0].record(stream)
    for b in range(blocks):
        for _ in range(per):
            pipe.run()
        ev[b + 1].record(stream)
    torch.cuda.synchronize(device)
    ms = sorted(ev[b].elapsed_time(ev[b + 1]) / per for b in range(blocks))
    return ms[len(ms) // 2], ms


def measure_host_solve(bank, work, psi_host, n_inst: int = 16) -> dict:
    """Host frontier solve of the first ``n_inst`` config-5 instances on the
    GPU cost matrix (outside every timed region): the reference's solve
    restated in Python vs the native ``fate_solve_frontier``, both at budget 0
    (option enumeration + deterministic greedy -- a full search of a 25-stage,
    32-device frontier does not finish in either), selections compared."""
    import numpy as np

    from paper_2605_07238_b200 import solver as native
    from paper_2605_07238_b200.wf import frontier as MF

    D = bank.scalars["n_devices"]
    elig = bank.arrays["st_elig"]
    sc = np.asarray(work.scen)
    devs = tuple(f"d{j:02d}" for j in range(D))
    t_py = t_nat = 0.0
    same = True
    n_cand = 0
    for inst in range(n_inst):
        cands, bounds = [], {}
        for w in np.nonzero(sc == inst)[0]:
            g = int(work.stage[w])
            sid = f"s{g:08d}"
            bounds[sid] = int(work.bounds[w])
            m = int(elig[g])
            base = int(work.psi_off[w])
            for k in range(bounds[sid]):
                for d in range(D):
                    if m >> d & 1:
                        cands.append(MF.Candidate(sid, k, devs[d], float(psi_host[base + k * D + d])))
        prob = MF.FrontierProblem(tuple(cands), bounds, devs)
        n_cand += len(cands)
        t0 = time.perf_counter()
        a = MF.solve_frontier(prob, budget_s=0.0)
        t1 = time.perf_counter()
        b = native.solve_frontier(prob, budget_s=0.0)
        t2 = time.perf_counter()
        t_py += t1 - t0
        t_nat += t2 - t1
        same &= (a.selected, a.objective.hex(), a.optimal) == (b.selected, b.objective.hex(),
                                                               b.optimal)
    return {"instances": n_inst, "candidates_per_instance": n_cand / n_inst, "budget_s": 0.0,
            "python_ms_per_instance": 1e3 * t_py / n_inst,
            "native_ms_per_instance": 1e3 * t_nat / n_inst, "identical": bool(same),
            "note": "host solve timed separately (north star); reference semantics restated"}


def cpu_sample_rate(bank, weights, states, work, target_s: float = 12.0, threads: int = 0):
    """The C oracle port of the reference scorer on a bounded sample of the
    workload's work items (first items in order), all host threads."""
    import numpy as np

    import oracle
    from paper_2605_07238_b200 import pack

    threads = threads or oracle.max_threads()

    def sub(n_items):
        w = pack.WorkList(scen=work.scen[:n_items].copy(), stage=work.stage[:n_items].copy(),
                          psi_off=work.psi_off[:n_items].copy(),
                          bounds=work.bounds[:n_items].copy(), n_psi=0)
        D = bank.scalars["n_devices"]
        w.psi_off = np.zeros(n_items, dtype=np.int64)
        if n_items:
            w.psi_off[1:] = np.cumsum(w.bounds[:-1].astype(np.int64) * D)
        w.n_psi = int(w.bounds.astype(np.int64).sum() * D)
        return w

    wrec = pack.weights_record(weights)
    n = min(64, work.n_items)
    w = sub(n)
    t0 = time.perf_counter()
    oracle.score(bank, wrec, states, w, n_threads=threads, with_extras=False)
    dt = time.perf_counter() - t0
    n2 = int(min(work.n_items, max(n, n * target_s / max(dt, 1e-6))))
    w = sub(n2)
    t0 = time.perf_counter()
    oracle.score(bank, wrec, states, w, n_threads=threads, with_extras=False)
    dt = time.perf_counter() - t0
    return {"value": w.n_psi / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {n2} of {work.n_items} work items ({w.n_psi} Psi) in {dt:.1f} s; "
                      f"C oracle (faithful port of CostModel.plan_score), OpenMP"}


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------


def run_reference(args):
    """Reference arm: the reference's CPU scorer (C oracle port) on the host
    cores, same workload/metric; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    from paper_2605_07238_b200 import fastgen, pack, scenarios

    plan = shard_plan(0, 1)
    cfg = scenarios.config_c5()
    fb = fastgen.synth_batch(cfg, plan["count"], plan["seed0"], plan["scen0"],
                             C5_SHAPE["depth"], C5_SHAPE["width"], C5_SHAPE["density"],
                             C5_SHAPE["batch"])
    sc, g = fb.frontier_items() if args.mode == "frontier" else fb.sweep_items()
    wrec = pack.weights_record(cfg.weights)
    threads = oracle.max_threads()
    per_step = args.ref_instances
    inst_of = sc

    def step_work(i):
        lo = (i * per_step) % plan["count"]
        sel = (inst_of >= lo) & (inst_of < lo + per_step)
        return pack.make_work(fb.bank, zip(sc[sel].tolist(), g[sel].tolist()), False)

    for i in range(args.warmup):
        oracle.score(fb.bank, wrec, fb.states, step_work(i), n_threads=threads, with_extras=False)
    works = [step_work(args.warmup + i) for i in range(args.steps)]
    n_psi = 0
    t0 = time.perf_counter()
    for w in works:
        oracle.score(fb.bank, wrec, fb.states, w, n_threads=threads, with_extras=False)
        n_psi += w.n_psi
    dt = time.perf_counter() - t0
    value = n_psi / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (config-5 generator, canonical scenario states)",
        "config": {"workload": f"c5_{args.mode}", "instances_per_step": per_step,
                   "stages_per_instance": 500, "devices": 32, "batch": 16, "horizon": 3},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{per_step} instances' {args.mode} items per step, "
                                   f"{n_psi} Psi over {args.steps} steps; C oracle port of "
                                   f"CostModel.plan_score (OpenMP)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_fate(args):
    import torch
    import torch.distributed as dist

    from paper_2605_07238_b200 import pack, runtime

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    device = torch.device(f"cuda:{local}")
    torch.cuda.set_device(device)

    if args.workload == "c5":
        cfg, bank, states, work, plan = build_c5(rank, world, args.mode)
    else:
        cfg, bank, states, work = build_c4(args.mode, first_scen=rank * C4_SCENARIOS)
        plan = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample_rate(bank, cfg.weights, states, work, target_s=args.cpu_seconds)

    t_bank = time.perf_counter()
    dbank = runtime.DeviceBank(bank, cfg.weights, device=device)
    torch.cuda.synchronize(device)
    bank_setup_s = time.perf_counter() - t_bank  # once per (bank, weights), not per step
    dstates = dbank.upload_states(states)
    dwork = dbank.upload_work(work)
    out = dbank.alloc_out(work, extras=True)
    out.tail = None  # diagnostic only; Psi + S + completion are what FATE consumes
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=device)  # 256 MiB
    torch.cuda.synchronize(device)

    clocks = ClockSampler(local)
    # one rank has nothing to gather (and no process group at N = 1)
    ms, launches = time_device(torch, dbank, dstates, dwork, out, args.steps, args.warmup, flush,
                               world, device, gather=args.gather and world > 1, clocks=clocks)
    ms_max = reduce_max(ms, world, device)
    psi_total = reduce_sum(float(work.n_psi), world, device)
    value = psi_total / (ms_max / 1e3)

    levels = dbank.levels
    nbytes = pack.compulsory_bytes(bank, work, states, levels, runtime.build_windows(bank, levels))
    ach = nbytes / (ms / 1e3) / 1e9
    peak, peak_src = hbm_peak()
    key = f"{args.workload}_{args.mode}"
    roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic_for(key), "peak_source": peak_src,
                "bytes_per_launch": nbytes, "bytes_per_candidate": nbytes / work.n_psi,
                "kernel": "fate_score_kernel"}
    csum = clocks.summary()
    ceil = issue_ceiling(key, ms, csum.get("sm_mhz") or csum.get("sm_max_mhz"))
    if ceil is not None:
        roofline["issue_ceiling"] = ceil

    pipe = runtime.HostPipeline(dbank, states, work, extras=False, n_chunks=4, graph=True)
    e2e_ms, e2e_blocks = time_e2e(torch, pipe, max(10, args.steps), min(args.warmup, 3), world,
                                  device)
    e2e_max = reduce_max(e2e_ms, world, device)
    e2e = {"value": psi_total / (e2e_max / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": pipe.h2d_bytes, "d2h_bytes_per_step": pipe.d2h_bytes,
           "ms_per_step": e2e_max, "block_ms": e2e_blocks,
           "path": "fate_pipeline_capture/replay: 4 scenario-aligned chunks, H2D / scoring / "
                   "D2H overlapped on 3 streams, one CUDA-graph launch per step"}

    host_solve = None
    if rank == 0 and world == 1 and args.workload == "c5" and args.mode == "frontier":
        host_solve = measure_host_solve(bank, work, out.psi.cpu().numpy())

    c4 = None
    if world == 1 and args.workload == "c5" and not args.no_c4:
        c4 = measure_c4(torch, device, args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (config-5 generator + canonical scenario states, SURVEY §8(d))",
            "config": {
                "workload": f"{args.workload}_{args.mode}",
                "instances_per_gpu": plan["count"] if plan else 1,
                "stages_per_instance": bank.n_stages // max(1, bank.scalars["n_instances"]),
                "devices": bank.scalars["n_devices"], "batch": bank.scalars["max_queries"],
                "horizon": cfg.weights.horizon, "psi_per_gpu_step": work.n_psi,
                "work_items_per_gpu_step": work.n_items,
                "l2": "flushed between steps (256 MiB write, outside the events)",
                "bank_setup_s": round(bank_setup_s, 3),
                "parallelism": f"dp{world}: "
                               + ("instances" if args.workload == "c5" else "scenario seeds")
                               + " sharded by rank, no data-path collective"
                               + (" + NCCL all-gather of Psi" if args.gather and world > 1
                                  else ""),
            },
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        if c4 is not None:
            line["c4_sweep"] = c4
        if host_solve is not None:
            line["host_solve"] = host_solve
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def measure_c4(torch, device, args) -> dict:
    from paper_2605_07238_b200 import pack, runtime

    cfg, bank, states, work = build_c4("sweep")
    dbank = runtime.DeviceBank(bank, cfg.weights, device=device)
    dstates = dbank.upload_states(states)
    dwork = dbank.upload_work(work)
    out = dbank.alloc_out(work, extras=True)
    out.tail = None
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=device)
    clocks = ClockSampler(device.index or 0)
    ms, launches = time_device(torch, dbank, dstates, dwork, out, max(5, args.steps // 4),
                               min(args.warmup, 3), flush, 1, device, clocks=clocks)
    nbytes = pack.compulsory_bytes(bank, work, states, dbank.levels,
                                   runtime.build_windows(bank, dbank.levels))
    peak, _ = hbm_peak()
    ach = nbytes / (ms / 1e3) / 1e9
    return {"workload": "c4_sweep (10k stages x 8 scenarios, 64 devices, 8 models, H=4)",
            "value": work.n_psi / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "psi_per_step": work.n_psi,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "traffic": traffic_for("c4_sweep"),
                         "bytes_per_launch": nbytes, "bytes_per_candidate": nbytes / work.n_psi,
                         "issue_ceiling": issue_ceiling(
                             "c4_sweep", ms, clocks.summary().get("sm_mhz")
                             or clocks.summary().get("sm_max_mhz"))},
            "clocks": clocks.summary(), "gpu_launches": launches}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("fate", "reference"), default="fate")
    ap.add_argument("--workload", choices=("c5", "c4"), default="c5")
    ap.add_argument("--mode", choices=("frontier", "sweep"), default="frontier")
    ap.add_argument("--gather", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-instances", type=int, default=16)
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_fate(args)


if __name__ == "__main__":
    sys.exit(main())
