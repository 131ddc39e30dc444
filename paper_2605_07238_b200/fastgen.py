"""Batch generator for layered synthetic workloads straight into SoA form.

Python front end of ``csrc/fate_synth.cpp``: builds thousands of config-5
style instances (``synth_generate`` + ``make_instance`` + the canonical
scenario state) directly as a :class:`~.pack.PackedBank` /
:class:`~.pack.PackedStates`, bit-identical to packing the Python objects
(``tests/test_fastgen.py``), without materialising per-stage objects.
This is the "workload and format path at scale" row of SURVEY.md §8(f).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .pack import PackedBank, PackedStates, _role_key
from .runtime import _check, load_library
from .wf.dagmodel import ROLE_KINDS


class _Catalog(C.Structure):
    _fields_ = [("n_devices", C.c_int32), ("device_names", C.POINTER(C.c_char_p)),
                ("n_models", C.c_int32)] + [
        (n, C.c_int32 * 11) for n in ("role_row", "role_shard", "role_max_tok", "role_out_tok",
                                      "role_keep", "role_reuse")] + [
        ("role_models_ptr", C.c_void_p), ("role_models", C.c_void_p)]


_OUT_I32 = ("st_model", "st_role", "st_prompt", "st_out", "st_group", "st_flags", "st_shard",
            "st_level", "par_ptr", "par_idx", "ch_ptr", "ch_idx", "q_prompt", "frontier_level",
            "loc", "residency", "kappa_n", "kappa")


class _Out(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n_instances", "n_stages_per", "n_edges", "batch",
                                         "n_devices", "kappa_cap")] + [
        ("st_model", C.POINTER(C.c_int32)), ("st_role", C.POINTER(C.c_int32)),
        ("st_prompt", C.POINTER(C.c_int32)), ("st_out", C.POINTER(C.c_int32)),
        ("st_group", C.POINTER(C.c_int32)), ("st_flags", C.POINTER(C.c_int32)),
        ("st_shard", C.POINTER(C.c_int32)), ("st_level", C.POINTER(C.c_int32)),
        ("par_ptr", C.POINTER(C.c_int32)), ("par_idx", C.POINTER(C.c_int32)),
        ("ch_ptr", C.POINTER(C.c_int32)), ("ch_idx", C.POINTER(C.c_int32)),
        ("q_prompt", C.POINTER(C.c_int32)), ("clock", C.POINTER(C.c_double)),
        ("frontier_level", C.POINTER(C.c_int32)), ("loc", C.POINTER(C.c_int32)),
        ("residency", C.POINTER(C.c_int32)), ("dev_free", C.POINTER(C.c_double)),
        ("kappa_n", C.POINTER(C.c_int32)), ("kappa", C.POINTER(C.c_int32))]


def _lib():
    L = load_library()
    if not getattr(L, "_synth_ready", False):
        L.fate_synth_layered.restype = C.c_int
        L.fate_synth_layered.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                         C.c_double, C.c_int32, C.POINTER(_Catalog),
                                         C.POINTER(C.POINTER(_Out))]
        L.fate_synth_free.argtypes = [C.POINTER(_Out)]
        L._synth_ready = True
    return L


class SyntheticBatch:
    """A generated batch: packed bank + one scenario per instance + frontier."""

    def __init__(self, bank: PackedBank, states: PackedStates, frontier_level: np.ndarray,
                 width: int):
        self.bank = bank
        self.states = states
        self.frontier_level = frontier_level
        self.width = width

    def frontier_items(self):
        """(scenario, global stage) work items: scenario i <-> instance i,
        frontier = the whole layer at the scenario's cut level."""
        lvl = self.bank.arrays["st_level"]
        inst = self.bank.arrays["st_inst"]
        sel = lvl == self.frontier_level[inst]
        g = np.flatnonzero(sel).astype(np.int32)
        return inst[g].astype(np.int32), g

    def sweep_items(self):
        g = np.arange(self.bank.n_stages, dtype=np.int32)
        return self.bank.arrays["st_inst"][g].astype(np.int32), g


def synth_batch(cfg, n_inst: int, seed0: int, scen0: int, depth: int, width: int,
                density: float, batch: int = 16) -> SyntheticBatch:
    """``n_inst`` instances; instance i = synth_generate(seed=seed0+i) +
    make_instance(batch, seed0+i) + scenario seed scen0+i."""
    L = _lib()
    topo = cfg.topology
    device_ids = sorted(topo.device_ids)
    D = len(device_ids)
    catalog = sorted(cfg.models)
    model_index = {m: i for i, m in enumerate(catalog)}
    names = (C.c_char_p * D)(*[d.encode() for d in device_ids])
    cat = _Catalog()
    cat.n_devices, cat.device_names, cat.n_models = D, names, len(catalog)
    roles = {(1.0, 1.0, 1.0, 1.0): 0}
    rm_ptr, rm = [0], []
    for k, kind in enumerate(ROLE_KINDS):
        role = cfg.roles[kind]
        key = _role_key(role)
        roles.setdefault(key, len(roles))
        cat.role_row[k] = roles[key]
        cat.role_shard[k] = int(role.shard_eligible)
        cat.role_max_tok[k] = role.max_token_proxy
        cat.role_out_tok[k] = role.output_size_proxy
        cat.role_keep[k] = int(role.default_keep_cache)
        cat.role_reuse[k] = int(role.default_cache_reuse)
        rm += [model_index[a] for a in cfg.role_models.get(kind, ())]
        rm_ptr.append(len(rm))
    rm_ptr_a = np.asarray(rm_ptr, dtype=np.int32)
    rm_a = np.asarray(rm or [0], dtype=np.int32)
    cat.role_models_ptr, cat.role_models = rm_ptr_a.ctypes.data, rm_a.ctypes.data
    out = C.POINTER(_Out)()
    _check(L.fate_synth_layered(n_inst, seed0, scen0, depth, width, density, batch,
                                C.byref(cat), C.byref(out)), "fate_synth_layered")
    try:
        o = out.contents
        V, E, cap = o.n_stages_per, o.n_edges, o.kappa_cap
        NS = n_inst * V
        sizes = {"st_model": NS, "st_role": NS, "st_prompt": NS, "st_out": NS, "st_group": NS,
                 "st_flags": NS, "st_shard": NS, "st_level": NS, "par_ptr": NS + 1,
                 "par_idx": max(E, 1), "ch_ptr": NS + 1, "ch_idx": max(E, 1),
                 "q_prompt": max(n_inst * batch, 1), "frontier_level": n_inst, "loc": NS,
                 "residency": n_inst * D, "kappa_n": n_inst * D, "kappa": n_inst * D * cap * 4}
        got = {k: np.ctypeslib.as_array(getattr(o, k), shape=(n,)).copy()
               for k, n in sizes.items()}
        clock = np.ctypeslib.as_array(o.clock, shape=(n_inst,)).copy()
        free = np.ctypeslib.as_array(o.dev_free, shape=(n_inst * D,)).copy()
    finally:
        L.fate_synth_free(out)

    role_rows = sorted(roles.items(), key=lambda kv: kv[1])
    arrays = {k: got[k] for k in ("st_model", "st_role", "st_prompt", "st_out", "st_group",
                                  "st_flags", "st_shard", "st_level", "par_ptr", "par_idx",
                                  "ch_ptr", "ch_idx", "q_prompt")}
    arrays["st_inst"] = np.repeat(np.arange(n_inst, dtype=np.int32), V)
    arrays["st_override"] = np.full(NS, -1, dtype=np.int32)
    arrays["st_elig"] = np.full(NS, (1 << D) - 1 if D < 64 else (1 << 64) - 1, dtype=np.uint64)
    arrays["q_group"] = np.full(max(n_inst * batch, 1), -1, dtype=np.int32)
    arrays["override_cost"] = np.zeros(D, dtype=np.float64)
    arrays["override_mask"] = np.zeros(1, dtype=np.uint64)
    arrays["dev_speed"] = np.array([float(topo.speed_factor(d)) for d in device_ids])
    arrays["dev_topo_order"] = np.array([device_ids.index(d) for d in topo.device_ids],
                                        dtype=np.int32)
    beta = np.array([[topo.transfer_coeff(a, b) for b in device_ids] for a in device_ids])
    arrays["beta"] = beta.ravel()
    arrays["model_prefill"] = np.array([float(cfg.models[m].prefill_coeff) for m in catalog])
    arrays["model_decode"] = np.array([float(cfg.models[m].decode_coeff) for m in catalog])
    arrays["model_switch"] = np.array([float(cfg.models[m].switch_penalty) for m in catalog])
    arrays["role_cplx"] = np.array([k[0] for k, _ in role_rows])
    arrays["role_prefill"] = np.array([k[1] for k, _ in role_rows])
    arrays["role_decode"] = np.array([k[2] for k, _ in role_rows])
    arrays["role_comm"] = np.array([k[3] for k, _ in role_rows])
    arrays["inst_stage_off"] = (np.arange(n_inst, dtype=np.int32) * V).astype(np.int32)
    arrays["inst_n_stages"] = np.full(n_inst, V, dtype=np.int32)
    arrays["inst_query_off"] = (np.arange(n_inst, dtype=np.int32) * batch).astype(np.int32)
    arrays["inst_n_queries"] = np.full(n_inst, batch, dtype=np.int32)
    scalars = dict(n_devices=D, n_models=len(catalog), n_roles=len(role_rows),
                   has_overrides=1 if len(topo.transfer_overrides) else 0, n_instances=n_inst,
                   n_stages=NS, n_edges=E, n_queries=n_inst * batch, max_queries=batch,
                   flags=(1 if bool(np.all(arrays["dev_speed"] == arrays["dev_speed"][0])) else 0)
                   | (2 if not np.any(arrays["q_group"] != -1) else 0),
                   beta_default=float(topo.default_transfer_coeff))
    sids = sorted(f"s{n:02d}" for n in range(V))
    sindex = {s: i for i, s in enumerate(sids)}
    bank = PackedBank(device_ids=device_ids, dev_index={d: i for i, d in enumerate(device_ids)},
                      model_index=dict(model_index), n_models=len(catalog),
                      group_index={f"pg:{m}": i for i, m in enumerate(catalog)}, arrays=arrays,
                      scalars=scalars, instances=[None] * n_inst, stage_ids=[sids] * n_inst,
                      stage_index=[sindex] * n_inst, inst_stage_off=arrays["inst_stage_off"])
    loc2 = got["loc"].reshape(n_inst, V)
    lvl2 = arrays["st_level"].reshape(n_inst, V)
    done = np.where(loc2 >= 0, lvl2, -1).max(axis=1).astype(np.int32)
    st_arrays = dict(scen_inst=np.arange(n_inst, dtype=np.int32), scen_clock=clock,
                     scen_loc_off=(np.arange(n_inst, dtype=np.int64) * V),
                     scen_done_level=done, loc=got["loc"],
                     residency=got["residency"], dev_free=free, kappa_n=got["kappa_n"],
                     kappa=got["kappa"])
    states = PackedStates(arrays=st_arrays, n_scenarios=n_inst, kappa_cap=cap)
    return SyntheticBatch(bank, states, got["frontier_level"], width)
