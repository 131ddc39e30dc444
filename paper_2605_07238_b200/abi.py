"""ctypes mirror of ``include/fate.h`` (the C ABI structs).

Pointer fields are filled from tensor ``data_ptr()`` (device) by
:mod:`.runtime`, or from numpy arrays (host) by the test-side oracle wrapper.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

MAX_HORIZON = 32

_p = C.c_void_p


class FateWeights(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "lambda_q", "lambda_s", "lambda_tr", "lambda_c", "lambda_p", "lambda_r",
        "gamma", "kappa_prefix", "locality_coeff", "shard_overhead_frac", "demand_coeff",
        "state_scale", "locality_scale", "prefix_scale", "switch_x", "transfer_x", "prefix_x",
    )] + [
        ("gamma_pow", C.c_double * MAX_HORIZON),
        ("horizon", C.c_int32),
        ("eff_horizon", C.c_int32),
        ("ablation", C.c_uint32),
        ("reserved", C.c_int32),
    ]


BANK_INTS = ("n_devices", "n_models", "n_roles", "has_overrides", "n_instances", "n_stages",
             "n_edges", "n_queries", "max_queries", "flags")
BANK_PTRS = ("dev_speed", "dev_topo_order", "beta", "model_prefill", "model_decode",
             "model_switch", "role_cplx", "role_prefill", "role_decode", "role_comm",
             "inst_stage_off", "inst_n_stages", "inst_query_off", "inst_n_queries",
             "st_inst", "st_model", "st_role", "st_prompt", "st_out", "st_group", "st_flags",
             "st_shard", "st_level", "st_override", "st_elig", "par_ptr", "par_idx", "ch_ptr",
             "ch_idx", "override_cost", "override_mask", "q_prompt", "q_group")


class FateBank(C.Structure):
    _fields_ = ([(n, C.c_int32) for n in BANK_INTS] + [("beta_default", C.c_double)]
                + [(n, _p) for n in BANK_PTRS])


STATE_PTRS = ("scen_inst", "scen_clock", "scen_loc_off", "scen_done_level", "loc", "residency",
              "dev_free", "kappa_n", "kappa")


class FateState(C.Structure):
    _fields_ = [("n_scenarios", C.c_int32), ("kappa_cap", C.c_int32)] + [(n, _p) for n in STATE_PTRS]


class FateHostBatch(C.Structure):
    _fields_ = [("n_scenarios", C.c_int32), ("kappa_cap", C.c_int32), ("n_loc", C.c_int64),
                ("scen_rec", _p), ("loc", _p), ("n_items", C.c_int32), ("reserved", C.c_int32),
                ("n_psi", C.c_int64), ("items", _p)]


class FateWork(C.Structure):
    _fields_ = [("n_items", C.c_int32), ("reserved", C.c_int32), ("scen", _p), ("stage", _p),
                ("psi_off", _p), ("queue", _p)]


class FateWindows(C.Structure):
    _fields_ = [("levels", C.c_int32), ("max_level_ops", C.c_int32), ("ptr", _p), ("idx", _p),
                ("wpar_ptr", _p), ("wpar_idx", _p), ("wpar_minlvl", _p)]


class FateDerived(C.Structure):
    _fields_ = [(n, _p) for n in ("mean_base", "demand", "split_penalty", "edge_sigma",
                                  "edge_term", "row_sums", "inst_qgroups", "tail_sum", "tail_static",
                                  "stage_rec", "tmpl_ptr", "tmpl", "tok_vals", "tok_sums")]


class FateOut(C.Structure):
    _fields_ = [(n, _p) for n in ("psi", "sched", "tail", "completion", "timing")]


def make_weights(rec: dict) -> FateWeights:
    w = FateWeights()
    for name, _ in FateWeights._fields_:
        if name in ("gamma_pow", "reserved"):
            continue
        setattr(w, name, rec[name])
    for i, g in enumerate(rec["gamma_pow"]):
        w.gamma_pow[i] = g
    return w


def fill_struct(struct, scalars: dict, pointers: dict):
    for k, v in scalars.items():
        setattr(struct, k, v)
    for k, v in pointers.items():
        setattr(struct, k, v)
    return struct


def host_ptr(a: np.ndarray) -> int:
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data
