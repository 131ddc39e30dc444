"""Executor-side realized durations on the GPU.

The reference executor prices every task it issues with
``CostModel.realized_duration(stage, [(device, task.queries)], state, dag)``
(``executor.py:231-233``, ``costs.py:383-416``) on its *live* state.
:class:`GpuCostModel` is the caller's ``wfsched.costs.CostModel`` with that
method answered by ``fate_realized`` (one small kernel per call): the state is
the device-resident mirror of the running instance when one follows it
(``compat.install(mirror=..., durations=True)``; its pending transitions are
applied first), otherwise the state is packed and uploaded.  Everything else
is the reference's own code.  ``compat.install(durations=True)`` makes the
executor construct this class (``executor.py:168``).

The reference's contract checks (overlapping shards, ineligible device,
``costs.py:391-401``) run on the host first and raise its ``ValueError``.
"""

from __future__ import annotations

import ctypes as C
import importlib

import numpy as np

from . import pack
from .runtime import _check, load_library

_COSTS = importlib.import_module("wfsched.costs")

_source = {"scorer": None}


def set_source(scorer) -> None:
    """The scorer whose banks (and, for a MirrorScorer, live mirror) price
    durations; ``None``: the planner's default scorer."""
    _source["scorer"] = scorer


def _scorer():
    s = _source["scorer"]
    if s is None:
        from .planner import default_scorer

        s = default_scorer()
    return s


class _Task(C.Structure):
    _fields_ = [("stage", C.c_int32), ("device", C.c_int32), ("q0", C.c_int32),
                ("nq", C.c_int32)]


def _lib():
    L = load_library()
    if not getattr(L, "_realized_bound", False):
        L.fate_realized.restype = C.c_int
        L.fate_realized.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L._realized_bound = True
    return L


def realized_on_gpu(cost_model, stage, shard_assignment, state):
    """ShardTimings of ``shard_assignment`` (list of (device, query ids)) for
    ``stage`` on ``state``, computed by ``fate_realized``."""
    scorer = _scorer()
    inst = state.instance
    mirror = None
    if getattr(scorer, "_live", None) is state and state.instance is scorer._instance:
        scorer._ensure_mirror(cost_model)
        mirror = scorer.mirror
        dbank = mirror.dbank
    else:
        dbank = scorer.bank_for(inst, cost_model.models, cost_model.topo, cost_model.weights)
    torch = dbank.torch
    packed = dbank.packed
    g = packed.global_index(0, stage.id)
    qindex = {q.query_id: i for i, q in enumerate(inst.queries)}
    tasks, tq = [], []
    for dev, qids in shard_assignment:
        tasks.append((g, packed.dev_index[dev], len(tq), len(qids)))
        tq += [qindex[q] for q in qids]
    t_host = np.asarray(tasks, dtype=np.int32).reshape(-1, 4)
    q_host = np.asarray(tq or [0], dtype=np.int32)
    dev = dbank.device
    d_tasks = torch.from_numpy(t_host).to(dev)
    d_q = torch.from_numpy(q_host).to(dev)
    d_out = torch.empty(3 * len(tasks), dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    if mirror is not None:
        mirror.flush(s)  # the live state's transitions so far
        cstate = mirror.cstate
        keep = None
    else:
        keep = dbank.upload_states(pack.pack_states(packed, [(0, state)]))
        cstate = keep.cstate
    _check(_lib().fate_realized(C.byref(dbank.cbank), C.byref(dbank.cweights), C.byref(cstate),
                                0, len(tasks), C.c_void_p(d_tasks.data_ptr()),
                                C.c_void_p(d_q.data_ptr()), C.c_void_p(d_out.data_ptr()),
                                C.c_void_p(s.cuda_stream)), "fate_realized")
    out = d_out.cpu().numpy().reshape(-1, 3)
    del keep
    return [_COSTS.ShardTiming(device_id=dev_id, queries=tuple(qids), switch_s=float(o[0]),
                               transfer_s=float(o[1]), compute_s=float(o[2]))
            for (dev_id, qids), o in zip(shard_assignment, out)]


class GpuCostModel(_COSTS.CostModel):
    """``wfsched.costs.CostModel`` whose ``realized_duration`` runs on the GPU."""

    def realized_duration(self, stage, shard_assignment, state, dag=None):
        seen: set = set()
        for _, qids in shard_assignment:  # costs.py:391-396
            dup = seen.intersection(qids)
            if dup:
                raise ValueError(f"overlapping shards share queries {sorted(dup)}")
            seen.update(qids)
        for device_id, _ in shard_assignment:  # costs.py:400-401
            if stage.eligible_devices and device_id not in stage.eligible_devices:
                raise ValueError(f"device {device_id} not eligible for stage {stage.id}")
        if not shard_assignment:
            return []
        return realized_on_gpu(self, stage, shard_assignment, state)
