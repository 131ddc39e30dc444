"""GPU kernel vs the CPU oracle, bit for bit, through the C ABI.

Covers every branch of the scorer (edge_case: transfer overrides, device
speeds, base_cost_override, restricted/empty eligibility, shard bounds 1-4,
stages without model/role/group, query prefix groups, foreign-model and
empty-model prefix entries, idle and busy devices), every ablation, horizons
0-6, and the canonical config-4/5 scenario states (frontier and sweep).
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

import oracle
from paper_2605_07238_b200 import pack, runtime
from paper_2605_07238_b200.wf.weights import AblationFlags

from cases import (ALL_ABLATIONS, bits, c4_case, c5_case, edge_case, small_case, token_case,
                   wide_case)

pytestmark = pytest.mark.gpu


def _gpu(case):
    dbank = runtime.DeviceBank(case.bank, case.weights)
    res = dbank.score(case.states, case.work, extras=True)
    n = case.work.n_items * case.bank.scalars["n_devices"]
    return {"psi": res.psi.cpu().numpy()[: case.work.n_psi],
            "sched": res.sched.cpu().numpy()[:n], "tail": res.tail.cpu().numpy()[:n],
            "completion": res.completion.cpu().numpy()[:n]}


def assert_parity(case):
    got = _gpu(case)
    want = oracle.score(case.bank, case.wrec, case.states, case.work)
    for k in ("psi", "sched", "tail", "completion"):
        g, w = bits(got[k]), bits(want[k])
        bad = np.flatnonzero(g != w)
        assert bad.size == 0, (
            f"{case} {k}: {bad.size} of {g.size} differ; first at {bad[:5]}: "
            f"gpu {got[k][bad[:3]]} oracle {want[k][bad[:3]]}")


@pytest.mark.parametrize("horizon", [0, 1, 2, 3, 4, 6])
def test_edge_case_horizons(horizon):
    assert_parity(edge_case(horizon=horizon))


@pytest.mark.parametrize("flag", ALL_ABLATIONS)
def test_edge_case_ablations(flag):
    assert_parity(edge_case(horizon=3, ablation=AblationFlags.from_names([flag])))


def test_edge_case_default_beta():
    assert_parity(edge_case(horizon=4, overrides=False))


def test_lifted_scenarios():
    assert_parity(small_case())


def test_prefix_suite_scenarios():
    assert_parity(small_case(prefix=True))


@pytest.mark.parametrize("horizon", [0, 3])
def test_partial_hit_token_classes(horizon):
    """Tabulated partial-hit prefix classes (tok_vals / tok_sums) next to
    untabulated ones, full hits and misses."""
    assert_parity(token_case(horizon=horizon))


def test_c5_frontier():
    assert_parity(c5_case(n_inst=6))


def test_c5_sweep():
    assert_parity(c5_case(n_inst=2, first=10, sweep=True))


def test_bank_file_scores_like_the_packed_bank(tmp_path):
    """A bank reloaded from its ``fate.bank@1`` file (no instance objects)
    scores bit-identically to the oracle."""
    case = edge_case(horizon=3)
    pack.save_bank(case.bank, tmp_path / "bank.npz")
    case.bank = pack.load_bank(tmp_path / "bank.npz")
    assert case.bank.instances == []
    assert_parity(case)


def test_c4_frontier_and_sweep_sample():
    assert_parity(c4_case(scen=(0, 3), sweep_stride=97))


def test_long_levels_walk_in_chunks():
    """Config-4 levels are longer than the production op buffer (64 entries),
    so their op lists are compacted and walked in several chunks: still
    bit-identical."""
    from paper_2605_07238_b200 import runtime

    case = c4_case(scen=(1,), sweep_stride=211)
    dbank = runtime.DeviceBank(case.bank, case.weights)
    assert dbank.cwin.max_level_ops > 64
    assert_parity(case)


def test_ab_knobs_are_not_in_the_production_library():
    """The production build runs one kernel generation: the A/B environment
    overrides of experiment builds (-DFATE_AB) change nothing."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "import conftest, test_gpu_parity as T\n"
            "from cases import c4_case, edge_case\n"
            "T.assert_parity(edge_case(horizon=4))\n"
            "T.assert_parity(c4_case(scen=(1,), sweep_stride=401))\n"
            "print('ok')\n" % (here, os.path.dirname(here)))
    env = dict(os.environ, FATE_SCORE_KERNEL="v5", FATE_MINB="7", FATE_V6_OPCAP="32",
               FATE_V6_FETCH="0", FATE_V6_DYNLAYOUT="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


WIDE = [
    (64, 40, 6, True, 4),     # two device slots, overrides, runtime layout (B > 16)
    (64, 16, 2, False, 4),    # two device slots, device-mask walk, static layout
    (33, 16, 3, False, 3),    # first two-slot size: one live device in slot 1
    (32, 256, 12, True, 5),   # last one-slot size, MAX_QUERIES queries
    (48, 24, 4, False, 6),    # two slots, runtime layout, horizon 6
    (8, 16, 64, True, 4),     # MAX_KAPPA prefix entries on a device
    (1, 1, 1, False, 2),      # one device, one query
]


@pytest.mark.parametrize("args", WIDE, ids=lambda a: "d%d-b%d-k%d-o%d-h%d" % a)
def test_wide_shapes(args):
    assert_parity(wide_case(*args))


@pytest.mark.parametrize("uniform", [True, False])
@pytest.mark.parametrize("n_dev", [32, 64])
def test_no_query_groups_lean_and_general_kernels(uniform, n_dev):
    """Banks without query prefix groups: uniform speed runs the lean
    instantiation (FATE_BANK_NO_QGROUPS + FATE_BANK_UNIFORM_SPEED), mixed
    speeds the general one; both bit-identical."""
    case = wide_case(n_dev, 16, 4, False, 4, seed=9, uniform_speed=uniform, qgroups=False)
    flags = case.bank.scalars["flags"]
    assert flags & pack.BANK_NO_QGROUPS
    assert bool(flags & pack.BANK_UNIFORM_SPEED) == uniform
    assert_parity(case)


def test_wide_shapes_uniform_speed_ablations():
    for flag in ALL_ABLATIONS:
        case = wide_case(64, 16, 3, False, 4, seed=5, uniform_speed=True)
        case.weights = replace(case.weights, ablation=AblationFlags.from_names([flag]))
        case.wrec = pack.weights_record(case.weights)
        case.work = pack.make_work(case.bank, [(int(s), int(g)) for s, g in
                                               zip(case.work.scen, case.work.stage)],
                                   case.weights.ablation.no_shard)
        assert_parity(case)


def test_empty_work_list_is_a_no_op():
    case = edge_case(horizon=3)
    dbank = runtime.DeviceBank(case.bank, case.weights)
    empty = pack.make_work(case.bank, [], False)
    before = runtime.launch_count()
    res = dbank.score(case.states, empty, extras=True)
    assert res.psi.numel() >= 0 and empty.n_psi == 0
    assert runtime.launch_count() == before


def test_library_is_native():
    """The scorer ran from the in-tree libfate.so, and launched kernels."""
    before = runtime.launch_count()
    _gpu(edge_case(horizon=2))
    assert runtime.launch_count() > before
    assert runtime.LIB_PATH.endswith("paper_2605_07238_b200/libfate.so")


def test_host_pipeline_chunks_match_device_path():
    """The pinned host-buffer call (native fate_pipeline_score, chunked over 3
    streams) returns exactly the device-resident result, S and completion
    included, and exactly the oracle."""
    import torch

    case = c5_case(n_inst=5)
    dbank = runtime.DeviceBank(case.bank, case.weights)
    res = dbank.score(case.states, case.work, extras=True)
    n = case.work.n_psi
    for chunks, streams, graph in ((4, 3, False), (1, 1, False), (64, 2, False), (8, 1, True),
                                   (3, 2, True)):
        pipe = runtime.HostPipeline(dbank, case.states, case.work, extras=True,
                                    n_chunks=chunks, n_streams=streams, graph=graph)
        pipe.host_psi.fill_(0.0)
        before = runtime.launch_count()
        got = pipe.run()
        torch.cuda.synchronize()
        assert runtime.launch_count() > before
        assert np.array_equal(bits(got.numpy()[:n]), bits(res.psi.cpu().numpy()[:n]))
        m = case.work.n_items * case.bank.scalars["n_devices"]
        assert np.array_equal(bits(pipe.host_sched.numpy()[:m]), bits(res.sched.cpu().numpy()[:m]))
        assert np.array_equal(bits(pipe.host_completion.numpy()[:m]),
                              bits(res.completion.cpu().numpy()[:m]))
        assert pipe.d2h_bytes == 8 * n + 16 * m
        pipe.close()
    want = oracle.score(case.bank, case.wrec, case.states, case.work)["psi"]
    assert np.array_equal(bits(got.numpy()[:n]), bits(want))


@pytest.mark.parametrize("args", [WIDE[0], WIDE[3], WIDE[5]],
                         ids=lambda a: "d%d-b%d-k%d-o%d-h%d" % a)
def test_host_pipeline_wide_shapes_match_oracle(args):
    """Host wire records at their largest (64 devices x 6 entries, 64
    entries per device, 256 queries) through the pipeline equal the oracle."""
    import torch

    case = wide_case(*args)
    dbank = runtime.DeviceBank(case.bank, case.weights)
    pipe = runtime.HostPipeline(dbank, case.states, case.work, extras=True, n_chunks=2,
                                graph=True)
    got = pipe.run()
    torch.cuda.synchronize()
    want = oracle.score(case.bank, case.wrec, case.states, case.work)
    n = case.work.n_psi
    m = case.work.n_items * case.bank.scalars["n_devices"]
    assert np.array_equal(bits(got.numpy()[:n]), bits(want["psi"]))
    assert np.array_equal(bits(pipe.host_sched.numpy()[:m]), bits(want["sched"]))
    assert np.array_equal(bits(pipe.host_completion.numpy()[:m]), bits(want["completion"]))
    pipe.close()


def test_host_pipeline_graph_replays_fresh_inputs():
    """A captured pipeline re-reads the pinned inputs on every replay."""
    import torch

    case = c5_case(n_inst=4)
    dbank = runtime.DeviceBank(case.bank, case.weights)
    pipe = runtime.HostPipeline(dbank, case.states, case.work, n_chunks=2, graph=True)
    first = pipe.run().clone()
    torch.cuda.synchronize()
    # perturb every scenario clock in the pinned wire records, replay, compare to oracle
    D = case.bank.scalars["n_devices"]
    rb = pack.scen_rec_bytes(D, case.states.kappa_cap)
    rec = pipe.h_rec.numpy().reshape(-1, rb)
    clocks = rec[:, 0:8].copy().view("<f8").ravel() + 7.25
    rec[:, 0:8] = clocks.reshape(-1, 1).view(np.uint8)
    got = pipe.run()
    torch.cuda.synchronize()
    arrays = dict(case.states.arrays)
    arrays["scen_clock"] = clocks
    st2 = pack.PackedStates(arrays=arrays, n_scenarios=case.states.n_scenarios,
                            kappa_cap=case.states.kappa_cap)
    want = oracle.score(case.bank, case.wrec, st2, case.work)["psi"]
    n = case.work.n_psi
    assert np.array_equal(bits(got.numpy()[:n]), bits(want))
    assert not np.array_equal(bits(got.numpy()[:n]), bits(first.numpy()[:n]))


def test_host_pipeline_skips_scenarios_without_items():
    """Scenarios no item reads are not copied; results still exact."""
    import torch

    case = c5_case(n_inst=6)
    keep = np.isin(case.work.scen, [1, 4])
    sub = pack.make_work(case.bank, zip(case.work.scen[keep].tolist(),
                                        case.work.stage[keep].tolist()), False)
    dbank = runtime.DeviceBank(case.bank, case.weights)
    pipe = runtime.HostPipeline(dbank, case.states, sub, n_chunks=3, n_streams=2)
    got = pipe.run()
    torch.cuda.synchronize()
    want = oracle.score(case.bank, case.wrec, case.states, sub)["psi"]
    assert np.array_equal(bits(got.numpy()[: sub.n_psi]), bits(want))
    full = sum(v.nbytes for v in case.states.arrays.values())
    assert pipe.h2d_bytes < full


def test_host_pipeline_rejects_contract_violations():
    """Unsorted items / out-of-range scenarios fail with ValueError (status < 0)
    before any copy is enqueued."""
    import ctypes as C

    from paper_2605_07238_b200 import abi

    case = c5_case(n_inst=2)
    dbank = runtime.DeviceBank(case.bank, case.weights)
    pipe = runtime.HostPipeline(dbank, case.states, case.work, n_chunks=2)
    items = pipe.h_items.numpy().view(pack.ITEM_DTYPE)
    saved = items.copy()
    items["scen"][0], items["scen"][-1] = items["scen"][-1], items["scen"][0]
    with pytest.raises(ValueError):
        pipe.run()
    items[:] = saved
    items["scen"][0] = case.states.n_scenarios + 5
    with pytest.raises(ValueError):
        pipe.run()
    items[:] = saved
    pipe.run()  # valid again
    pipe.close()


def test_concurrent_launches_on_streams_and_graph_replay():
    """Scoring launches in flight on several streams at once, next to a
    captured host pipeline, each keep their own work-queue counter: every
    result equals the oracle."""
    import torch

    case = c5_case(n_inst=6)
    want = oracle.score(case.bank, case.wrec, case.states, case.work)["psi"]
    n = case.work.n_psi
    dbank = runtime.DeviceBank(case.bank, case.weights)
    ds, dw = dbank.upload_states(case.states), dbank.upload_work(case.work)
    outs = [dbank.alloc_out(case.work, extras=False) for _ in range(6)]
    streams = [torch.cuda.Stream() for _ in outs]
    pipe = runtime.HostPipeline(dbank, case.states, case.work, n_chunks=3, graph=True)
    torch.cuda.synchronize()
    for _ in range(5):
        for o, s in zip(outs, streams):
            o.psi.fill_(0.0)
        torch.cuda.synchronize()
        for o, s in zip(outs, streams):
            dbank.score_into(ds, dw, o, stream=s)
        pipe.run()
        torch.cuda.synchronize()
        for o in outs:
            assert np.array_equal(bits(o.psi.cpu().numpy()[:n]), bits(want))
        assert np.array_equal(bits(pipe.host_psi.numpy()[:n]), bits(want))
    pipe.close()


def test_captured_pipeline_invalidated_by_larger_batch():
    """A direct call that outgrows the captured workspaces invalidates the
    graph: replay then refuses (status < 0) instead of using freed memory;
    a new capture works."""
    import ctypes as C

    import torch

    small, big = c5_case(n_inst=2), c5_case(n_inst=6)
    dbank = runtime.DeviceBank(big.bank, big.weights)
    sub = pack.make_work(big.bank, [(s, g) for s, g in zip(big.work.scen, big.work.stage)
                                    if s < 2], False)
    pipe = runtime.HostPipeline(dbank, big.states, sub, n_chunks=2, graph=True)
    other = runtime.HostPipeline(dbank, big.states, big.work, n_chunks=2)
    L = runtime.load_library()
    s = torch.cuda.current_stream()
    rc = L.fate_pipeline_score(pipe.handle, C.byref(dbank.cbank), C.byref(dbank.cweights),
                               C.byref(dbank.cwin), C.byref(dbank.cder), C.byref(other.batch),
                               C.c_void_p(other.host_psi.data_ptr()), None, None,
                               C.c_void_p(s.cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match="capture again"):
        pipe.run()
    other.close()
    pipe.close()


def test_bench_batches_in_full():
    """The bench's own batches, in full, bit-identical to the oracle: every
    Psi, S and completion of the config-5 frontier batch (4096 instances,
    5.72 M Psi, bench.build_c5) and every Psi of the config-4 sweep (all 8
    scenario states x 10 000 stages, 9.0 M Psi, bench.build_c4)."""
    import bench

    cfg, bank, states, work = bench.build_c5(bench.shard_plan(0, 1), "frontier")
    want = oracle.score(bank, pack.weights_record(cfg.weights), states, work)
    res = runtime.DeviceBank(bank, cfg.weights).score(states, work, extras=True)
    assert work.n_psi == 5_722_208
    for k in ("psi", "sched", "completion"):
        got = getattr(res, k).cpu().numpy()[: want[k].size]
        assert np.array_equal(bits(got), bits(want[k])), k

    cfg, bank, states, work = bench.build_c4("sweep")
    want = oracle.score(bank, pack.weights_record(cfg.weights), states, work,
                        with_extras=False)["psi"]
    got = runtime.DeviceBank(bank, cfg.weights).score(states, work, extras=False).psi
    assert work.n_psi == 9_003_008
    assert np.array_equal(bits(got.cpu().numpy()[: work.n_psi]), bits(want))


def test_prepare_rejects_false_bank_declarations_and_nonfinite_ops():
    """fate_prepare verifies what a bank declares (FATE_BANK_NO_QGROUPS,
    FATE_BANK_UNIFORM_SPEED -- the lean kernel relies on both) and that every
    tail op value is finite (the exact walk's skipped op is fma(v, 0, a)):
    a false declaration or a non-finite weight is a status < 0, not wrong Psi."""
    import copy

    case = small_case()
    qg = copy.deepcopy(case.bank)
    qg.arrays["q_group"] = qg.arrays["q_group"].copy()
    qg.arrays["q_group"][0] = 0
    qg.scalars["flags"] |= pack.BANK_NO_QGROUPS
    with pytest.raises(ValueError, match="NO_QGROUPS"):
        runtime.DeviceBank(qg, case.weights)
    sp = copy.deepcopy(case.bank)
    sp.arrays["dev_speed"] = sp.arrays["dev_speed"].copy()
    sp.arrays["dev_speed"][-1] = 1.5
    sp.scalars["flags"] |= pack.BANK_UNIFORM_SPEED
    with pytest.raises(ValueError, match="UNIFORM_SPEED"):
        runtime.DeviceBank(sp, case.weights)
    with pytest.raises(ValueError, match="non-finite"):
        runtime.DeviceBank(case.bank, replace(case.weights, switch_x=float("inf")))
    big = replace(case.weights, switch_x=1e308, state_scale=1e308)  # finite weights, inf ops
    if any(float(case.bank.arrays["model_switch"][m]) > 0 for m in range(len(case.bank.arrays["model_switch"]))):
        with pytest.raises(ValueError, match="non-finite"):
            runtime.DeviceBank(case.bank, big)
    runtime.DeviceBank(case.bank, case.weights)  # the honest bank still prepares


def test_more_concurrent_launches_than_rotating_counter_slots():
    """160 launches in flight on 160 streams (more than the library's 128
    rotating ticket counters): each (work list, stream) brings its own
    counter (fate_work.queue), so every result equals the oracle."""
    import torch

    case = c5_case(n_inst=2)
    want = bits(oracle.score(case.bank, case.wrec, case.states, case.work)["psi"])
    n = case.work.n_psi
    dbank = runtime.DeviceBank(case.bank, case.weights)
    ds, dw = dbank.upload_states(case.states), dbank.upload_work(case.work)
    from cuda.bindings import runtime as cudart

    outs = [dbank.alloc_out(case.work, extras=False) for _ in range(160)]
    # 160 distinct CUDA streams (torch's own stream pool recycles 32)
    raw = []
    for _ in outs:
        err, h = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
        assert err == cudart.cudaError_t.cudaSuccess
        raw.append(h)
    streams = [torch.cuda.ExternalStream(int(h)) for h in raw]
    gate = torch.cuda.Event()
    hold = torch.cuda.current_stream()
    torch.cuda._sleep(20_000_000)  # keep the streams' launches queued together
    gate.record(hold)
    for o, s in zip(outs, streams):
        s.wait_event(gate)
        dbank.score_into(ds, dw, o, stream=s)
    torch.cuda.synchronize()
    assert len(dw._queues) == 160
    for o in outs:
        assert np.array_equal(bits(o.psi.cpu().numpy()[:n]), want)
    for h in raw:
        cudart.cudaStreamDestroy(h)


@pytest.mark.parametrize("g", [2, 4, 8])
def test_strong_scaling_shards_match_oracle(g):
    """Rank 0's shard at g ranks (bench.shard_plan / bench.c4_plan) scored on
    the GPU equals the oracle bit for bit.  The shards put the launch in
    every scheduling regime of the persistent grid: a static first share
    with multi-item tickets (2-way), a short static share with 2-item
    tickets (4-way) and single-item tickets (8-way)."""
    import bench

    cfg, bank, states, work = bench.build_c5(bench.shard_plan(0, g), "frontier")
    want = oracle.score(bank, pack.weights_record(cfg.weights), states, work,
                        with_extras=False)["psi"]
    got = runtime.DeviceBank(bank, cfg.weights).score(states, work, extras=False).psi
    assert np.array_equal(bits(got.cpu().numpy()[: work.n_psi]), bits(want))

    p = bench.c4_plan(0, g)
    cfg, bank, states, work = bench.build_c4("sweep", n_scen=p["count"], first_scen=p["first"],
                                             stage_rank=p["stage_rank"],
                                             stage_world=p["stage_world"])
    want = oracle.score(bank, pack.weights_record(cfg.weights), states, work,
                        with_extras=False)["psi"]
    got = runtime.DeviceBank(bank, cfg.weights).score(states, work, extras=False).psi
    assert np.array_equal(bits(got.cpu().numpy()[: work.n_psi]), bits(want))
