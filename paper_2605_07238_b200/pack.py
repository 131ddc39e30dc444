"""Host packer: scheduler objects -> structure-of-arrays (the C-ABI format).

Turns ``(models, topology, weights)`` + workflow instances into the static
``fate_bank`` arrays and execution-state snapshots into ``fate_state`` arrays
(``include/fate.h``).  Duck-typed on the reference's field names, so it packs
both the reference's own objects (``wfsched.model`` / ``wfsched.state``) and
this package's mirror (:mod:`paper_2605_07238_b200.wf`).

Index conventions (SURVEY.md §7.1 rule 2): stage index = rank in
``sorted(stage_ids)`` (offset per instance), device index = rank in
``sorted(device_ids)``.  Every ``sorted(...)`` iteration of the reference
therefore becomes ascending-index order on the device.

Reference read-side semantics packed here:
* ``output_device`` -- plurality device of a completed stage's output shards,
  ties to the smallest id (``state.py:96-108``); computed with the state's own
  method so reference states are packed by the reference's rule;
* ``cached_tokens`` -- prefix entries ``(group, tokens, model)`` per device
  (``state.py:110-123``); groups and model strings are dictionary-encoded, so
  matching is exact equality with no hashing collisions;
* ``residency`` / ``device_free`` / ``clock`` (``state.py:45-57``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MAX_DEVICES = 64
MAX_HORIZON = 32
MAX_QUERIES = 256
MAX_KAPPA = 64

ABL_BITS = {
    "no_future_planning": 1,
    "no_locality": 2,
    "no_same_model": 4,
    "no_prefix": 8,
    "no_shard": 16,
}
BANK_UNIFORM_SPEED = 1
BANK_NO_QGROUPS = 2  # no query prefix group anywhere in the bank (lean kernel)
STAGE_CACHE_REUSE = 1
STAGE_KEEP_CACHE = 2

_NEUTRAL_ROLE = (1.0, 1.0, 1.0, 1.0)  # StageRole(kind="worker") defaults (costs.py:19)


def weights_record(weights) -> dict:
    """``ScoreWeights`` -> plain values of ``fate_weights``."""
    eff = weights.effective_horizon()
    if weights.horizon >= MAX_HORIZON or eff >= MAX_HORIZON:
        raise ValueError(f"horizon {weights.horizon} exceeds the supported {MAX_HORIZON - 1}")
    abl = 0
    for name, bit in ABL_BITS.items():
        if getattr(weights.ablation, name):
            abl |= bit
    names = ("lambda_q", "lambda_s", "lambda_tr", "lambda_c", "lambda_p", "lambda_r", "gamma",
             "kappa_prefix", "locality_coeff", "shard_overhead_frac", "demand_coeff",
             "state_scale", "locality_scale", "prefix_scale", "switch_x", "transfer_x",
             "prefix_x")
    rec = {n: float(getattr(weights, n)) for n in names}
    # gamma ** l exactly as the reference evaluates it (float ** int, costs.py:349)
    rec["gamma_pow"] = [weights.gamma ** l for l in range(MAX_HORIZON)]
    rec["horizon"] = int(weights.horizon)
    rec["eff_horizon"] = int(eff)
    rec["ablation"] = abl
    return rec


@dataclass
class PackedBank:
    """Static SoA for one RunConfig and a batch of instances (host numpy)."""

    device_ids: list
    dev_index: dict
    model_index: dict          # model string -> id (catalog first, sorted)
    n_models: int
    group_index: dict          # prefix-group string -> id
    arrays: dict               # name -> np.ndarray (fate_bank fields)
    scalars: dict
    instances: list            # the packed instance objects
    stage_ids: list            # per instance: sorted stage ids
    stage_index: list          # per instance: id -> local index
    inst_stage_off: np.ndarray
    windows: dict = field(default_factory=dict)  # levels -> (ptr, idx)

    @property
    def n_stages(self) -> int:
        return int(self.scalars["n_stages"])

    def global_index(self, inst: int, stage_id: str) -> int:
        return int(self.inst_stage_off[inst]) + self.stage_index[inst][stage_id]

    def model_id(self, name, grow: bool = True) -> int:
        if name is None:
            return -1
        mid = self.model_index.get(name)
        if mid is None:
            if not grow:
                return -2
            mid = len(self.model_index)
            self.model_index[name] = mid
        return mid

    def group_id(self, name) -> int:
        if name is None:
            return -1
        return self.group_index.get(name, -2)


def _role_key(role) -> tuple:
    if role is None:
        return _NEUTRAL_ROLE
    return (float(role.complexity), float(role.prefill_scale), float(role.decode_scale),
            float(role.comm_weight))


def pack_bank(instances, models, topo) -> PackedBank:
    """Pack the static side: catalog + a batch of instances sharing it."""
    device_ids = sorted(topo.device_ids)
    n_dev = len(device_ids)
    if n_dev == 0 or n_dev > MAX_DEVICES:
        raise ValueError(f"device count {n_dev} outside 1..{MAX_DEVICES}")
    dev_index = {d: i for i, d in enumerate(device_ids)}
    catalog = sorted(models)
    model_index = {m: i for i, m in enumerate(catalog)}
    speed = np.array([float(topo.speed_factor(d)) for d in device_ids], dtype=np.float64)
    topo_order = np.array([dev_index[d] for d in topo.device_ids], dtype=np.int32)
    beta = np.zeros((n_dev, n_dev), dtype=np.float64)
    for i, src in enumerate(device_ids):
        for j, dst in enumerate(device_ids):
            beta[i, j] = topo.transfer_coeff(src, dst)
    has_over = 1 if len(topo.transfer_overrides) else 0

    group_index: dict = {}

    def gid(name):
        if name is None:
            return -1
        if name not in group_index:
            group_index[name] = len(group_index)
        return group_index[name]

    roles: dict = {_NEUTRAL_ROLE: 0}
    cols = {k: [] for k in ("st_inst", "st_model", "st_role", "st_prompt", "st_out", "st_group",
                            "st_flags", "st_shard", "st_level", "st_override")}
    elig: list = []
    over_rows: list = []
    over_mask: list = []
    par_lists: list = []
    ch_lists: list = []
    q_prompt: list = []
    q_group: list = []
    inst_stage_off, inst_n_stages, inst_query_off, inst_n_queries = [], [], [], []
    stage_ids_all, stage_index_all = [], []
    g0 = 0
    max_q = 0
    for ii, inst in enumerate(instances):
        dag = inst.dag
        if dag.annotations is None:
            raise ValueError("plan_score requires an annotated dag")
        sids = sorted(dag.stages)
        sindex = {s: i for i, s in enumerate(sids)}
        stage_ids_all.append(sids)
        stage_index_all.append(sindex)
        inst_stage_off.append(g0)
        inst_n_stages.append(len(sids))
        inst_query_off.append(len(q_prompt))
        inst_n_queries.append(len(inst.queries))
        max_q = max(max_q, len(inst.queries))
        if len(inst.queries) > MAX_QUERIES:
            raise ValueError(f"batch of {len(inst.queries)} queries exceeds {MAX_QUERIES}")
        level = dag.annotations.level
        for sid in sids:
            st = dag.stages[sid]
            if st.model is not None and st.model not in model_index:
                raise KeyError(f"model alias {st.model!r} not in catalog")
            rk = _role_key(st.role)
            if rk not in roles:
                roles[rk] = len(roles)
            cols["st_inst"].append(ii)
            cols["st_model"].append(-1 if st.model is None else model_index[st.model])
            cols["st_role"].append(roles[rk])
            cols["st_prompt"].append(int(st.prompt_token_proxy))
            cols["st_out"].append(int(st.output_token_proxy))
            cols["st_group"].append(gid(st.shared_prefix_group))
            cols["st_flags"].append((STAGE_CACHE_REUSE if st.cache_reuse else 0)
                                    | (STAGE_KEEP_CACHE if st.keep_cache else 0))
            cols["st_shard"].append(int(st.shard_bound))
            cols["st_level"].append(int(level[sid]))
            mask = 0
            for d in st.eligible_devices:
                if d not in dev_index:
                    raise ValueError(f"stage {sid}: unknown device {d}")
                mask |= 1 << dev_index[d]
            elig.append(mask)
            ov = st.base_cost_override
            if ov is not None:
                row = np.zeros(n_dev, dtype=np.float64)
                omask = 0
                for d, val in ov.items():
                    if d in dev_index:
                        row[dev_index[d]] = float(val)
                        omask |= 1 << dev_index[d]
                cols["st_override"].append(len(over_rows))
                over_rows.append(row)
                over_mask.append(omask)
            else:
                cols["st_override"].append(-1)
        ups = [[] for _ in sids]
        downs = [[] for _ in sids]
        for src, dst in dag.edges:
            ups[sindex[dst]].append(sindex[src] + g0)
            downs[sindex[src]].append(sindex[dst] + g0)
        for lst in ups:
            lst.sort()
        for lst in downs:
            lst.sort()
        par_lists.extend(ups)
        ch_lists.extend(downs)
        for q in inst.queries:
            q_prompt.append(int(q.prompt_tokens))
            q_group.append(gid(q.prefix_group))
        g0 += len(sids)

    role_rows = sorted(roles.items(), key=lambda kv: kv[1])
    arrays = {k: np.asarray(v, dtype=np.int32) for k, v in cols.items()}
    arrays["st_elig"] = np.asarray(elig, dtype=np.uint64)
    arrays["par_ptr"], arrays["par_idx"] = _csr(par_lists)
    arrays["ch_ptr"], arrays["ch_idx"] = _csr(ch_lists)
    arrays["override_cost"] = (np.stack(over_rows) if over_rows
                               else np.zeros((1, n_dev))).astype(np.float64).ravel()
    arrays["override_mask"] = np.asarray(over_mask or [0], dtype=np.uint64)
    arrays["q_prompt"] = np.asarray(q_prompt or [0], dtype=np.int32)
    arrays["q_group"] = np.asarray(q_group or [-1], dtype=np.int32)
    arrays["dev_speed"] = speed
    arrays["dev_topo_order"] = topo_order
    arrays["beta"] = beta.ravel()
    arrays["model_prefill"] = np.array([float(models[m].prefill_coeff) for m in catalog] or [1.0])
    arrays["model_decode"] = np.array([float(models[m].decode_coeff) for m in catalog] or [0.0])
    arrays["model_switch"] = np.array([float(models[m].switch_penalty) for m in catalog] or [0.0])
    arrays["role_cplx"] = np.array([k[0] for k, _ in role_rows])
    arrays["role_prefill"] = np.array([k[1] for k, _ in role_rows])
    arrays["role_decode"] = np.array([k[2] for k, _ in role_rows])
    arrays["role_comm"] = np.array([k[3] for k, _ in role_rows])
    arrays["inst_stage_off"] = np.asarray(inst_stage_off, dtype=np.int32)
    arrays["inst_n_stages"] = np.asarray(inst_n_stages, dtype=np.int32)
    arrays["inst_query_off"] = np.asarray(inst_query_off, dtype=np.int32)
    arrays["inst_n_queries"] = np.asarray(inst_n_queries, dtype=np.int32)
    scalars = dict(
        n_devices=n_dev, n_models=len(catalog), n_roles=len(role_rows), has_overrides=has_over,
        n_instances=len(instances), n_stages=g0, n_edges=int(arrays["par_idx"].size),
        n_queries=len(q_prompt), max_queries=max_q, beta_default=float(topo.default_transfer_coeff),
        flags=(BANK_UNIFORM_SPEED if bool(np.all(speed == speed[0])) else 0)
        | (BANK_NO_QGROUPS if not np.any(arrays["q_group"] != -1) else 0),
    )
    return PackedBank(
        device_ids=device_ids, dev_index=dev_index, model_index=model_index,
        n_models=len(catalog), group_index=group_index, arrays=arrays, scalars=scalars,
        instances=list(instances), stage_ids=stage_ids_all, stage_index=stage_index_all,
        inst_stage_off=arrays["inst_stage_off"],
    )


def _csr(lists):
    ptr = np.zeros(len(lists) + 1, dtype=np.int32)
    if lists:
        ptr[1:] = np.cumsum([len(x) for x in lists])
    flat = [i for lst in lists for i in lst]
    idx = np.asarray(flat or [0], dtype=np.int32)
    return ptr, idx


def bound_of(bank: PackedBank, g: int, no_shard: bool) -> int:
    """Slots per stage (planner.py:88): 1 if no_shard else min(R, |A(v)|)."""
    if no_shard:
        return 1
    return min(int(bank.arrays["st_shard"][g]), int(bank.arrays["st_elig"][g]).bit_count())


# ---------------------------------------------------------------------------
# state snapshots
# ---------------------------------------------------------------------------


# ---------------------------------------------------------------------------
# binary bank format: pack once, score many
# ---------------------------------------------------------------------------

BANK_FORMAT = "fate.bank@1"


def _json_default(x):
    if isinstance(x, np.integer):
        return int(x)
    if isinstance(x, np.floating):
        return float(x)
    raise TypeError(f"{type(x).__name__} is not serialisable")


def save_bank(bank: PackedBank, path) -> None:
    """Write the packed static side as one ``.npz``: every ``fate_bank``
    array verbatim plus the index dictionaries, so a batch packed once (from
    instance JSON or the generators) is reloaded without touching the
    instance objects.  Horizon windows are not stored; the native builder
    derives them from the CSR on first use."""
    import json

    ids = [sid for per_inst in bank.stage_ids for sid in per_inst]
    if any("\n" in sid for sid in ids):
        raise ValueError("stage ids containing a newline cannot be stored")
    meta = dict(format=BANK_FORMAT, device_ids=list(bank.device_ids),
                model_index=bank.model_index, n_models=bank.n_models,
                group_index=bank.group_index, scalars=bank.scalars,
                n_stage_ids=[len(s) for s in bank.stage_ids])
    blobs = {f"a.{k}": np.ascontiguousarray(v) for k, v in bank.arrays.items()}
    blobs["meta"] = np.frombuffer(json.dumps(meta, default=_json_default).encode(), np.uint8)
    blobs["ids"] = np.frombuffer("\n".join(ids).encode(), np.uint8)
    with open(path, "wb") as fh:
        np.savez(fh, **blobs)


def load_bank(path) -> PackedBank:
    """Inverse of :func:`save_bank`; ``instances`` is empty on the result."""
    import json

    with np.load(path, allow_pickle=False) as z:
        meta = json.loads(bytes(z["meta"]).decode())
        if meta.get("format") != BANK_FORMAT:
            raise ValueError(f"unsupported bank format {meta.get('format')!r}")
        arrays = {k[2:]: z[k] for k in z.files if k.startswith("a.")}
        flat = bytes(z["ids"]).decode().split("\n") if z["ids"].size else []
    stage_ids = []
    pos = 0
    for n in meta["n_stage_ids"]:
        stage_ids.append(flat[pos: pos + n])
        pos += n
    if pos != len(flat):
        raise ValueError("bank file: stage id table does not match the instance sizes")
    device_ids = list(meta["device_ids"])
    return PackedBank(
        device_ids=device_ids, dev_index={d: i for i, d in enumerate(device_ids)},
        model_index=dict(meta["model_index"]), n_models=int(meta["n_models"]),
        group_index=dict(meta["group_index"]), arrays=arrays, scalars=dict(meta["scalars"]),
        instances=[], stage_ids=stage_ids,
        stage_index=[{sid: i for i, sid in enumerate(ids)} for ids in stage_ids],
        inst_stage_off=arrays["inst_stage_off"],
    )


@dataclass
class PackedStates:
    arrays: dict
    n_scenarios: int
    kappa_cap: int


def pack_states(bank: PackedBank, scenarios, kappa_cap: int | None = None) -> PackedStates:
    """Pack ``[(instance_index, state), ...]`` into ``fate_state`` arrays."""
    n_dev = bank.scalars["n_devices"]
    dev_index = bank.dev_index
    n_s = len(scenarios)
    caps = [max((len(ents) for ents in st.prefix_store.values()), default=0)
            for _, st in scenarios]
    cap = max(caps, default=0)
    if kappa_cap is not None:
        if kappa_cap < cap:
            raise ValueError(f"kappa_cap {kappa_cap} < live prefix entries {cap}")
        cap = kappa_cap
    cap = max(cap, 1)
    if cap > MAX_KAPPA:
        raise ValueError(f"{cap} prefix entries per device exceed {MAX_KAPPA}")
    scen_inst = np.zeros(n_s, dtype=np.int32)
    clock = np.zeros(n_s, dtype=np.float64)
    loc_off = np.zeros(n_s, dtype=np.int64)
    residency = np.full(n_s * n_dev, -1, dtype=np.int32)
    free = np.zeros(n_s * n_dev, dtype=np.float64)
    kap_n = np.zeros(n_s * n_dev, dtype=np.int32)
    kap = np.zeros((n_s * n_dev, cap, 4), dtype=np.int32)
    locs = []
    done_level = np.full(n_s, -1, dtype=np.int32)
    off = 0
    lvl_all = bank.arrays["st_level"]
    for s, (ii, st) in enumerate(scenarios):
        scen_inst[s] = ii
        clock[s] = float(st.clock)
        loc_off[s] = off
        sindex = bank.stage_index[ii]
        row = np.full(len(sindex), -1, dtype=np.int32)
        for sid in st.parent_loc:
            dev = st.output_device(sid)
            if dev is not None and sid in sindex:
                row[sindex[sid]] = dev_index[dev]
        locs.append(row)
        if np.any(row >= 0):
            g0 = int(bank.inst_stage_off[ii])
            done_level[s] = int(lvl_all[g0: g0 + len(sindex)][row >= 0].max())
        off += len(sindex)
        base = s * n_dev
        for dev, di in dev_index.items():
            res = st.residency.get(dev)
            residency[base + di] = bank.model_id(res)
            free[base + di] = float(st.device_free.get(dev, 0.0))
            ents = st.prefix_store.get(dev, {})
            kap_n[base + di] = len(ents)
            for k, ent in enumerate(ents.values()):
                kap[base + di, k, 0] = bank.group_id(ent.group)
                kap[base + di, k, 1] = int(ent.tokens)
                kap[base + di, k, 2] = bank.model_id(ent.model)
    arrays = dict(
        scen_inst=scen_inst, scen_clock=clock, scen_loc_off=loc_off, scen_done_level=done_level,
        loc=np.concatenate(locs) if locs else np.zeros(1, dtype=np.int32),
        residency=residency, dev_free=free, kappa_n=kap_n, kappa=kap.ravel(),
    )
    return PackedStates(arrays=arrays, n_scenarios=n_s, kappa_cap=cap)


def pack_state_into(bank: PackedBank, inst: int, st, v: dict, cap: int) -> None:
    """:func:`pack_states` for one scenario ``(inst, st)``, written into
    preallocated arrays ``v`` (the fate_state fields; ``loc`` sized to the
    instance, ``kappa`` to ``n_devices * cap * 4``) -- the per-wave form used
    by :class:`~.runtime.WaveRunner`'s pinned staging block."""
    n_dev = bank.scalars["n_devices"]
    v["scen_inst"][0] = inst
    v["scen_clock"][0] = float(st.clock)
    v["scen_loc_off"][0] = 0
    row = v["loc"]
    row.fill(-1)
    dev_index, sindex = bank.dev_index, bank.stage_index[inst]
    g0 = int(bank.inst_stage_off[inst])
    lvl = bank.arrays["st_level"]
    done = -1
    for sid in st.parent_loc:
        dev = st.output_device(sid)
        i = sindex.get(sid)
        if dev is not None and i is not None:
            row[i] = dev_index[dev]
            lv = int(lvl[g0 + i])
            if lv > done:
                done = lv
    v["scen_done_level"][0] = done
    res, free, kn = v["residency"], v["dev_free"], v["kappa_n"]
    kap = v["kappa"][: n_dev * cap * 4].reshape(n_dev, cap, 4)
    kap.fill(0)
    res.fill(-1)
    free.fill(0.0)
    kn.fill(0)
    for dev, di in dev_index.items():
        res[di] = bank.model_id(st.residency.get(dev))
        free[di] = float(st.device_free.get(dev, 0.0))
        ents = st.prefix_store.get(dev, {})
        if len(ents) > cap:
            raise ValueError(f"{len(ents)} prefix entries on {dev} exceed capacity {cap}")
        kn[di] = len(ents)
        for k, ent in enumerate(ents.values()):
            kap[di, k, 0] = bank.group_id(ent.group)
            kap[di, k, 1] = int(ent.tokens)
            kap[di, k, 2] = bank.model_id(ent.model)


# ---------------------------------------------------------------------------
# work lists
# ---------------------------------------------------------------------------


@dataclass
class WorkList:
    scen: np.ndarray
    stage: np.ndarray
    psi_off: np.ndarray
    bounds: np.ndarray
    n_psi: int

    @property
    def n_items(self) -> int:
        return int(self.scen.size)


def make_work(bank: PackedBank, items, no_shard: bool) -> WorkList:
    """``items`` = iterable of (scenario, global stage index)."""
    n_dev = bank.scalars["n_devices"]
    items = list(items)
    scen = np.asarray([s for s, _ in items], dtype=np.int32)
    stage = np.asarray([g for _, g in items], dtype=np.int32)
    if no_shard:
        bounds = np.ones(len(items), dtype=np.int32)
    else:
        shard = bank.arrays["st_shard"][stage] if len(items) else np.zeros(0, np.int32)
        pop = popcount64(bank.arrays["st_elig"][stage]) if len(items) else np.zeros(0, np.int32)
        bounds = np.minimum(shard, pop).astype(np.int32)
    off = np.zeros(len(items), dtype=np.int64)
    if len(items):
        off[1:] = np.cumsum(bounds.astype(np.int64) * n_dev)[:-1]
    n_psi = int(bounds.astype(np.int64).sum() * n_dev)
    return WorkList(scen=scen, stage=stage, psi_off=off, bounds=bounds, n_psi=n_psi)


def popcount64(a: np.ndarray) -> np.ndarray:
    a = np.asarray(a, dtype=np.uint64)
    out = np.zeros(a.shape, dtype=np.int32)
    for shift in range(0, 64, 8):
        out += _POP8[((a >> np.uint64(shift)) & np.uint64(0xFF)).astype(np.int64)]
    return out


_POP8 = np.array([bin(i).count("1") for i in range(256)], dtype=np.int32)


def candidates_from_psi(bank: PackedBank, work: WorkList, psi: np.ndarray, inst: int):
    """Rebuild ``(stage_id, slot, device_id, psi)`` tuples in the reference's
    candidate order (sorted stage -> slot -> sorted eligible device)."""
    n_dev = bank.scalars["n_devices"]
    off0 = int(bank.inst_stage_off[inst])
    sids = bank.stage_ids[inst]
    devs = bank.device_ids
    elig_all = bank.arrays["st_elig"]
    out = []
    for w in range(work.n_items):
        g = int(work.stage[w])
        sid = sids[g - off0]
        mask = int(elig_all[g])
        base = int(work.psi_off[w])
        for k in range(int(work.bounds[w])):
            row = base + k * n_dev
            for d in range(n_dev):
                if mask >> d & 1:
                    out.append((sid, k, devs[d], float(psi[row + d])))
    return out


def compulsory_bytes(bank: PackedBank, work: WorkList, states: PackedStates, levels: int,
                     windows=None) -> int:
    """Algorithmic (compulsory) bytes of a scoring launch, SURVEY.md §8(d):

    per unit u = (scenario, stage v) with n_c = slots(v)*D candidates
      in(u)  = 32 + 12|Pa(v)| + 8|Ch(v)|[slots>1]
               + sum_{l, bucket nonempty} (8 + sum_{x in bucket} (16 + 12|Pa(x)|))
               + D*(24 + 16*kbar) + 8*B
      out(u) = 8*n_c
    kbar = mean live prefix entries per device of the unit's scenario.
    """
    a = bank.arrays
    n_dev = bank.scalars["n_devices"]
    par_ptr = a["par_ptr"].astype(np.int64)
    ch_ptr = a["ch_ptr"].astype(np.int64)
    npar = par_ptr[1:] - par_ptr[:-1]
    nch = ch_ptr[1:] - ch_ptr[:-1]
    kap_n = states.arrays["kappa_n"].reshape(states.n_scenarios, n_dev)
    kbar = kap_n.mean(axis=1)
    nq = a["inst_n_queries"][states.arrays["scen_inst"]]
    total = 0.0
    win_bytes = np.zeros(bank.n_stages, dtype=np.float64)
    if levels > 0:
        ptr, idx = windows
        for g in np.unique(work.stage):
            b = 0.0
            for l in range(levels):
                lo, hi = int(ptr[g * levels + l]), int(ptr[g * levels + l + 1])
                if hi > lo:
                    xs = idx[lo:hi]
                    b += 8 + float(np.sum(16 + 12 * npar[xs]))
            win_bytes[g] = b
    st = work.stage
    slots = work.bounds
    unit_in = (32 + 12 * npar[st] + 8 * nch[st] * (slots > 1) + win_bytes[st]
               + n_dev * (24 + 16 * kbar[work.scen]) + 8 * nq[work.scen])
    unit_out = 8 * slots.astype(np.float64) * n_dev
    total = float(np.sum(unit_in) + np.sum(unit_out))
    return int(math.floor(total + 0.5))


# per (item, eligible device): the fp64 operations the reference's formulas
# mandate outside the tail walk -- sched_score (costs.py:222-231: 10 products,
# 5 sums, 1 negation), Psi(slot 0) = S + tail, wait, completion (3), prefix
# (2), the tail's per-level combination (5 per nonempty level: divide,
# product, sum, gamma product, accumulate), _parallel_benefit when R > 1 (6)
# and each slot >= 1 of _marginal_shard_score (15).  Divisions count as one
# operation (a lower bound).
FP64_PER_CAND_FIXED = 16 + 1 + 1 + 3 + 2
FP64_PER_LEVEL = 5
FP64_PARALLEL = 6
FP64_MARGINAL = 15


def mandated_fp64_ops(bank: PackedBank, work: WorkList, states: PackedStates, levels: int,
                      windows, sample: int = 3000, seed: int = 0) -> dict:
    """Lower bound on the fp64 operations a scoring launch must execute,
    estimated on a uniform sample of its work items and scaled to the launch:
    the fixed per-candidate arithmetic above plus, for every horizon level with
    a located window parent (the only levels whose chain is state-dependent),
    one add per (op, device it applies to) of the tail's op sequence
    (costs.py:307-348: model op, prefix op, located parent edges other than v).
    Sequential += chains cannot be shared between devices whose op sequences
    differ, so each is an fp64 add per device."""
    a = bank.arrays
    D = bank.scalars["n_devices"]
    M = bank.scalars["n_models"]
    rng = np.random.default_rng(seed)
    n = work.n_items
    pick = np.arange(n) if n <= sample else np.sort(rng.choice(n, sample, replace=False))
    par_ptr, par_idx = a["par_ptr"], a["par_idx"]
    st_model, st_group, st_level = a["st_model"], a["st_group"], a["st_level"]
    ptr, idx = windows if levels else (None, None)
    S = states.arrays
    tot = 0.0
    walk_tot = 0.0
    for w in pick:
        s, v = int(work.scen[w]), int(work.stage[w])
        elig = int(a["st_elig"][v])
        ne = bin(elig).count("1")
        bound = int(work.bounds[w])
        n_lev = 0
        walk = 0.0
        if levels:
            inst = int(a["st_inst"][v])
            off = int(S["scen_loc_off"][s]) - int(bank.inst_stage_off[inst])
            res = S["residency"][s * D:(s + 1) * D]
            mv = int(st_model[v])
            disp = np.array([(r if (r != -1 and r != mv and r < M) else -1) for r in res])
            cls = {x: int(np.sum((disp == x) & np.array([(elig >> d) & 1 for d in range(D)],
                                                        dtype=bool))) for x in range(M)}
            for l in range(levels):
                lo, hi = int(ptr[v * levels + l]), int(ptr[v * levels + l + 1])
                if hi == lo:
                    continue
                n_lev += 1
                xs = idx[lo:hi]
                ops = 0.0
                located = False
                for x in xs:
                    mx = int(st_model[x])
                    if mx != -1:
                        ops += ne if mx == mv else cls.get(mx, 0)
                    if st_group[v] != -1 and st_group[x] == st_group[v]:
                        ops += ne
                    for e in range(int(par_ptr[x]), int(par_ptr[x + 1])):
                        u = int(par_idx[e])
                        if u == v:
                            continue
                        L = int(S["loc"][off + u])
                        if L >= 0:
                            located = True
                            ops += ne - ((elig >> L) & 1)
                if located:
                    walk += ops
        fixed = ne * (FP64_PER_CAND_FIXED + FP64_PER_LEVEL * n_lev
                      + (FP64_PARALLEL if int(a["st_shard"][v]) > 1 else 0)
                      + FP64_MARGINAL * max(0, bound - 1))
        tot += fixed + walk
        walk_tot += walk
    scale = n / max(1, len(pick))
    return {"fp64_ops": tot * scale, "walk_adds": walk_tot * scale,
            "sampled_items": int(len(pick)), "items": int(n)}


# ---------------------------------------------------------------------------
# host wire format of fate_pipeline_score (include/fate.h: fate_host_batch)
# ---------------------------------------------------------------------------

ITEM_DTYPE = np.dtype([("scen", "<i4"), ("stage", "<i4"), ("psi_off", "<i8")])


def scen_rec_bytes(n_dev: int, cap: int) -> int:
    """FATE_SCEN_REC_BYTES(D, cap)."""
    return 32 + 16 * n_dev + 16 * n_dev * cap


@dataclass
class HostBatch:
    rec: np.ndarray      # uint8 [S * rec_bytes]
    loc: np.ndarray      # int8 [n_loc] (device index, -1 = None)
    items: np.ndarray    # ITEM_DTYPE [W]
    n_scenarios: int
    kappa_cap: int
    n_psi: int


def host_batch(states: PackedStates, work: WorkList, n_dev: int) -> HostBatch:
    """Pack scenario states + work list into the pipeline's wire format: one
    fixed-size record per scenario, the loc rows, 16-byte items."""
    a = states.arrays
    S, cap = states.n_scenarios, states.kappa_cap
    rb = scen_rec_bytes(n_dev, cap)
    rec = np.zeros((S, rb), dtype=np.uint8)
    rec[:, 0:8] = np.asarray(a["scen_clock"], dtype="<f8").reshape(S, 1).view(np.uint8)
    rec[:, 8:16] = np.asarray(a["scen_loc_off"], dtype="<i8").reshape(S, 1).view(np.uint8)
    rec[:, 16:20] = np.asarray(a["scen_inst"], dtype="<i4").reshape(S, 1).view(np.uint8)
    rec[:, 20:24] = np.asarray(a["scen_done_level"], dtype="<i4").reshape(S, 1).view(np.uint8)
    o = 32
    for key, dt, width in (("residency", "<i4", n_dev), ("kappa_n", "<i4", n_dev),
                           ("dev_free", "<f8", n_dev), ("kappa", "<i4", n_dev * cap * 4)):
        arr = np.ascontiguousarray(np.asarray(a[key], dtype=dt).reshape(S, width))
        nb = arr.shape[1] * arr.dtype.itemsize
        rec[:, o:o + nb] = arr.view(np.uint8)
        o += nb
    assert o == rb
    items = np.empty(work.n_items, dtype=ITEM_DTYPE)
    items["scen"] = work.scen
    items["stage"] = work.stage
    items["psi_off"] = work.psi_off
    loc = np.asarray(a["loc"])
    if loc.size and (loc.max() >= n_dev or loc.min() < -1 or n_dev > 127):
        raise ValueError("loc entries must be device indices < n_devices <= 127, or -1")
    return HostBatch(rec=rec.reshape(-1), loc=np.ascontiguousarray(loc, dtype=np.int8),
                     items=items, n_scenarios=S, kappa_cap=cap, n_psi=work.n_psi)
