"""CPU oracle for the FATE scorer -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/libfate_oracle.so`` (built from
``oracle/fate_oracle.c`` by ``oracle/Makefile``), a scalar C restatement of
the reference scorer (``/root/reference/pkg/src/wfsched/costs.py:70-416``).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; the product package never does.

Parity pinning: ``tests/test_oracle_golden.py`` checks this oracle bit-for-bit
against Psi vectors captured from the reference itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2605_07238_b200 import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfate_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        try:  # incremental: rebuilds when fate_oracle.c or include/fate.h changed
            build()
        except (OSError, subprocess.CalledProcessError):
            if not os.path.exists(_LIB_PATH):
                raise
        L = C.CDLL(_LIB_PATH)
        L.oracle_score.restype = C.c_int
        L.oracle_score.argtypes = [C.c_void_p] * 5 + [C.c_int]
        L.oracle_plan_score.restype = C.c_double
        L.oracle_plan_score.argtypes = [C.c_void_p] * 3 + [C.c_int, C.c_int32, C.c_int, C.c_int]
        L.oracle_pysum.restype = C.c_double
        L.oracle_pysum.argtypes = [C.c_void_p, C.c_int64]
        L.oracle_max_threads.restype = C.c_int
        _lib = L
    return _lib


class HostArgs:
    """Host-pointer fate_* structs over packed numpy arrays (keeps them alive)."""

    def __init__(self, bank, weights_rec, states, work):
        self._keep = []
        a = {k: np.ascontiguousarray(v) for k, v in bank.arrays.items()}
        self._keep.append(a)
        self.bank = abi.fill_struct(
            abi.FateBank(), {k: bank.scalars[k] for k in abi.BANK_INTS if k in bank.scalars}
            | {"beta_default": bank.scalars["beta_default"]},
            {k: abi.host_ptr(a[k]) for k in abi.BANK_PTRS})
        self.weights = abi.make_weights(weights_rec)
        sa = {k: np.ascontiguousarray(v) for k, v in states.arrays.items()}
        self._keep.append(sa)
        self.state = abi.fill_struct(abi.FateState(), {"n_scenarios": states.n_scenarios,
                                                       "kappa_cap": states.kappa_cap},
                                     {k: abi.host_ptr(sa[k]) for k in abi.STATE_PTRS})
        wa = dict(scen=np.ascontiguousarray(work.scen), stage=np.ascontiguousarray(work.stage),
                  psi_off=np.ascontiguousarray(work.psi_off))
        self._keep.append(wa)
        self.work = abi.fill_struct(abi.FateWork(), {"n_items": work.n_items},
                                    {k: abi.host_ptr(v) for k, v in wa.items()})


def score(bank, weights_rec, states, work, n_threads: int = 0, with_extras: bool = True):
    """Oracle Psi (+ S, tail, completion) in fate_score's output layout."""
    args = HostArgs(bank, weights_rec, states, work)
    n_dev = bank.scalars["n_devices"]
    psi = np.empty(max(work.n_psi, 1), dtype=np.float64)
    extras = {k: np.empty(max(work.n_items * n_dev * (3 if k == "timing" else 1), 1),
                          dtype=np.float64)
              for k in ("sched", "tail", "completion", "timing")} if with_extras else {}
    out = abi.FateOut(psi=psi.ctypes.data,
                      sched=extras["sched"].ctypes.data if extras else None,
                      tail=extras["tail"].ctypes.data if extras else None,
                      completion=extras["completion"].ctypes.data if extras else None,
                      timing=extras["timing"].ctypes.data if extras else None)
    rc = lib().oracle_score(C.byref(args.bank), C.byref(args.weights), C.byref(args.state),
                            C.byref(args.work), C.byref(out), int(n_threads))
    if rc != 0:
        raise RuntimeError(f"oracle_score failed: {rc}")
    res = {"psi": psi[: work.n_psi]}
    for k, v in extras.items():
        res[k] = v[: work.n_items * n_dev * (3 if k == "timing" else 1)]
    return res


def pysum(values) -> float:
    x = np.ascontiguousarray(values, dtype=np.float64)
    return lib().oracle_pysum(x.ctypes.data, x.size)


def max_threads() -> int:
    return lib().oracle_max_threads()
