"""World-size-2 (gloo, CPU) run of bench.py's exact multi-GPU plan (SURVEY
§8(e)): contiguous instance ranges per rank (strong scaling), each rank
scores its shard (the oracle stands in for the kernel on CPU), solves its
frontiers with the native batch solve, and all-gathers its Psi slab and its
assignment triples with bench.SlabGather.  The gathered slabs must equal the
per-rank results, and their concatenation must equal one process scoring and
solving the whole batch."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

TOTAL = 6


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard(plan):
    import bench
    import oracle
    from paper_2605_07238_b200 import pack

    cfg, bank, states, work = bench.build_c5(plan, "frontier")
    res = oracle.score(bank, pack.weights_record(cfg.weights), states, work, n_threads=1,
                       with_extras=False)
    summary, sol = bench.host_solve_all(bank, work, res["psi"], threads=2, repeats=1)
    D = bank.scalars["n_devices"]
    n = len(sol.n_sel)
    trip = np.zeros((n, D * 3 + 1), dtype=np.int32)
    trip[:, 0] = sol.n_sel
    trip[:, 1:] = sol.sel.reshape(n, D * 3)
    # work-item indices are rank-local; make them instance-global stage ids
    sel = [[(int(bank.arrays["st_inst"][int(work.stage[a])]) + plan["first"],
             int(work.stage[a]) - int(bank.inst_stage_off[int(bank.arrays["st_inst"][int(work.stage[a])])]),
             int(b), int(c)) for a, b, c in sol.selected(p)] for p in range(n)]
    return res["psi"], trip.ravel(), sel, work.n_psi, summary


def _worker(rank, world, port, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = bench.shard_plan(rank, world, total=TOTAL)
        psi, trip, sel, n_psi, summary = _shard(plan)
        mx = bench.reduce_max(1.0 + rank, world)
        tot = bench.reduce_sum(float(n_psi), world)
        g_psi = bench.SlabGather(torch, n_psi, torch.float64, "cpu", world, fill=float("nan"))
        g_psi(torch.from_numpy(psi.copy()))
        g_as = bench.SlabGather(torch, trip.size, torch.int32, "cpu", world)
        g_as(torch.from_numpy(trip.copy()))
        q.put((rank, plan, mx, tot, psi, [g_psi.part(r).numpy().copy() for r in range(world)],
               trip, [g_as.part(r).numpy().copy() for r in range(world)], sel,
               bench.c4_plan(rank, world), summary["problems"]))
    finally:
        dist.destroy_process_group()


def test_two_rank_plan_gathers_and_solves():
    import bench

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1 = out
    # contiguous, disjoint, covering instance ranges (strong scaling)
    assert (r0[1]["first"], r0[1]["count"], r1[1]["first"], r1[1]["count"]) == (0, 3, 3, 3)
    assert r0[2] == r1[2] == 2.0                                 # max over ranks
    assert r0[3] == r1[3] == float(len(r0[4]) + len(r1[4]))      # whole-job Psi
    assert r0[10] == r1[10] == 3                                 # problems per rank
    # every rank holds every rank's Psi slab and assignment triples, unchanged
    for rank_out in out:
        for r in range(2):
            assert np.array_equal(rank_out[5][r].view(np.uint64), out[r][4].view(np.uint64))
            assert np.array_equal(rank_out[7][r], out[r][6])
    # C4: every scenario on every rank, stages split by residue mod world
    assert r0[9] == {"first": 0, "count": 8, "stage_rank": 0, "stage_world": 2}
    assert r1[9] == {"first": 0, "count": 8, "stage_rank": 1, "stage_world": 2}
    # the union equals one process doing the whole batch
    psi_all, _, sel_all, _, _ = _shard(bench.shard_plan(0, 1, total=TOTAL))
    assert np.array_equal(np.concatenate([r0[4], r1[4]]).view(np.uint64),
                          psi_all.view(np.uint64))
    assert r0[8] + r1[8] == sel_all
