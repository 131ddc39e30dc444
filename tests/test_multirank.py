"""World-size-2 (gloo, CPU) coverage of bench.py's multi-GPU plumbing: the
instance sharding plan, max/sum reductions over ranks, the optional Psi
all-gather, and the oracle on each rank's shard (every rank scores disjoint,
complete instances: no data-path exchange is needed)."""

from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


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
        plan = bench.shard_plan(rank, world, per_gpu=3)
        # each rank builds its own shard with the mirror generators and scores it
        import numpy as np

        import oracle
        from paper_2605_07238_b200 import pack, scenarios

        cfg = scenarios.config_c5()
        insts = [scenarios.c5_instance(plan["first"] + i, cfg) for i in range(plan["count"])]
        bank = pack.pack_bank(insts, cfg.models, cfg.topology)
        states = pack.pack_states(bank, [(i, scenarios.build_scenario(inst, cfg, plan["scen0"] + i))
                                         for i, inst in enumerate(insts)])
        items = [(i, bank.global_index(i, sid)) for i, inst in enumerate(insts)
                 for sid in scenarios.scenario_frontier(inst, states_obj(inst, cfg, plan, i))]
        work = pack.make_work(bank, items, False)
        res = oracle.score(bank, pack.weights_record(cfg.weights), states, work, n_threads=1)
        local_ms = 1.0 + rank
        mx = bench.reduce_max(local_ms, world)
        tot = bench.reduce_sum(float(work.n_psi), world)
        psi = torch.from_numpy(res["psi"].copy())
        gathered, sizes = bench.gather_slabs(psi, world)
        q.put((rank, plan, mx, tot, work.n_psi, sizes, gathered.numpy().tolist()[:4],
               [i.dag.workflow_id for i in insts], np.isfinite(res["psi"]).all()))
    finally:
        dist.destroy_process_group()


def states_obj(inst, cfg, plan, i):
    from paper_2605_07238_b200 import scenarios

    return scenarios.build_scenario(inst, cfg, plan["scen0"] + i)


def test_two_rank_sharding_and_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, plan0, mx0, tot0, n0, sizes0, g0, ids0, fin0), (r1, plan1, mx1, tot1, n1, sizes1, g1, ids1,
                                                           fin1) = out
    assert plan0["first"] == 0 and plan1["first"] == 3
    assert not set(ids0) & set(ids1)            # disjoint instances (weak scaling)
    assert mx0 == mx1 == 2.0                    # max over ranks
    assert tot0 == tot1 == float(n0 + n1)       # whole-job candidate count
    assert sizes0 == sizes1 == [n0, n1]
    assert fin0 and fin1
