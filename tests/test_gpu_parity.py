"""GPU kernel vs the CPU oracle, bit for bit, through the C ABI.

Covers every branch of the scorer (edge_case: transfer overrides, device
speeds, base_cost_override, restricted/empty eligibility, shard bounds 1-4,
stages without model/role/group, query prefix groups, foreign-model and
empty-model prefix entries, idle and busy devices), every ablation, horizons
0-6, and the canonical config-4/5 scenario states (frontier and sweep).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2605_07238_b200 import runtime
from paper_2605_07238_b200.wf.weights import AblationFlags

from cases import ALL_ABLATIONS, bits, c4_case, c5_case, edge_case, small_case

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


def test_c5_frontier():
    assert_parity(c5_case(n_inst=6))


def test_c5_sweep():
    assert_parity(c5_case(n_inst=2, first=10, sweep=True))


def test_c4_frontier_and_sweep_sample():
    assert_parity(c4_case(scen=(0, 3), sweep_stride=97))


def test_library_is_native():
    """The scorer ran from the in-tree libfate.so, and launched kernels."""
    before = runtime.launch_count()
    _gpu(edge_case(horizon=2))
    assert runtime.launch_count() > before
    assert runtime.LIB_PATH.endswith("paper_2605_07238_b200/libfate.so")


def test_host_pipeline_chunks_match_device_path():
    """The pinned host-buffer call (chunked over 3 streams) returns exactly the
    device-resident result."""
    case = c5_case(n_inst=5)
    dbank = runtime.DeviceBank(case.bank, case.weights)
    want = dbank.score(case.states, case.work, extras=False).psi.cpu().numpy()[: case.work.n_psi]
    pipe = runtime.HostPipeline(dbank, case.states, case.work, n_chunks=4, n_streams=3)
    got = pipe.run()
    import torch

    torch.cuda.synchronize()
    assert np.array_equal(bits(got.numpy()[: case.work.n_psi]), bits(want))
    assert len(pipe.chunks) >= 2
