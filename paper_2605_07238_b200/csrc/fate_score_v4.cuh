// fate_score_v4.cuh -- warp-per-item scoring kernel (production path).
//
// Included by fate_kernels.cu (inside its anonymous namespace).
//
// One warp owns one item = (scenario, stage v); lane t owns devices
// t, t+32, ... (DPL = 1 for D <= 32, 2 for D <= 64), so an item never
// synchronises beyond its own warp (__syncwarp only) and items in a CTA run
// independently.  Per item:
//
//   P0  per device: residency, free time, cached stage-group tokens (cs),
//       wait, switch, transfer and colo counts -- the transfer loop walks v's
//       parents once for both device slots (costs.py:107-125, 157-165).
//   P1  row classes: devices with equal (cs, speed) share the cache-aware
//       query_compute row bit for bit (costs.py:70-94); classes found with
//       __match_any_sync.  Instances with query prefix groups use one class
//       per device.  The first RCAP classes get their row in shared memory;
//       further classes are evaluated directly (rare: query groups on > RCAP
//       devices).
//   P2  class rows, then every Neumaier sum the reference takes over them:
//       aware / full-batch compute (costs.py:257, :404) and the shard ranges of
//       the <= 2 shard counts the item uses (:404-405).
//   P3  tail (costs.py:281-352) per level: with no located parent edge in the
//       level the affinity chain depends only on (v, l, displacing resident
//       model) and comes from the static table built by the prologue; else the
//       warp compacts the level into an ordered op list (signed values:
//       a - b == a + (-b) exactly) and each lane walks it for its 1-2 devices
//       at once (the op load is shared, the chains are independent: ILP 2).
//   P4  per device: colo, prefix overlap, parallel benefit, S, tail,
//       Psi(slot 0..bound-1), completion.

constexpr int V4_KT = 4;    // shard counts k <= V4_KT: shard sums tabulated per class
constexpr int V4_RCAP = 8;  // classes with a shared-memory row

struct V4Op {
    double val;
    int key;   // kind 0/2: located device (-1 = applies to all); kind 1: model
    int kind;  // 0: apply iff key != d; 1: apply iff key == displacing model of d;
               // 2: override locality op, apply iff key != d, value = sigma
};

struct V4View {
    double* rows;     // [RCAP*Bmax]
    double* shard;    // [D*2*KT] per class
    double* aware;    // [D] per class
    double* sw;       // [D]
    double* tr;       // [D]
    V4Op* ops;        // [ops_cap]
    int* key;         // [D] cs per device
    int* rowc;        // [D] class per device
    int* rowdev;      // [D] representative per class
    int* slot2cls;    // [RCAP] class of each shared-memory row slot
};

__host__ __device__ inline size_t v4_item_bytes(int D, int Bmax, int ops_cap) {
    size_t dbl = (size_t)V4_RCAP * Bmax + (size_t)D * 2 * V4_KT + 3 * (size_t)D;
    size_t ops = (size_t)ops_cap * sizeof(V4Op);
    size_t ints = 3 * (size_t)D + V4_RCAP;
    return (dbl * 8 + ops + ints * 4 + 15) & ~size_t(15);
}

__device__ inline V4View v4_view(unsigned char* base, int D, int Bmax, int ops_cap) {
    V4View v;
    double* dp = reinterpret_cast<double*>(base);
    v.rows = dp; dp += (size_t)V4_RCAP * Bmax;
    v.shard = dp; dp += (size_t)D * 2 * V4_KT;
    v.aware = dp; dp += D;
    v.sw = dp; dp += D;
    v.tr = dp; dp += D;
    v.ops = reinterpret_cast<V4Op*>(dp);
    int* ip = reinterpret_cast<int*>(v.ops + ops_cap);
    v.key = ip; ip += D;
    v.rowc = ip; ip += D;
    v.rowdev = ip; ip += D;
    v.slot2cls = ip;
    return v;
}

struct V4Item {
    int s, v, q0, nq, m, gv, Pv;
    bool cache_reuse;
    long long dev_row0;
    int cap4;
    const int32_t* kappa;
    const int32_t* kappa_n;
    double pcoef, pscale, decode, cplx;
};

// cache-aware query_compute of query q on device dv (costs.py:70-94)
__device__ __forceinline__ double v4_qc(const fate_bank& b, const V4Item& it, const V4View& V,
                                        int dv, int q) {
    const long long sp = V.key[dv];  // max(0, P(v) - cached stage-group tokens)
    long long qp = b.q_prompt[it.q0 + q];
    const int qg = b.q_group[it.q0 + q];
    if (qg != -1) {
        const long long drow = it.dev_row0 + dv;
        const long long cc = cached_tokens(it.kappa + drow * it.cap4, it.kappa_n[drow], qg, it.m);
        qp = qp - cc > 0 ? qp - cc : 0;
    }
    return qc_value(sp, qp, it.pcoef, it.pscale, it.decode, it.cplx, b.dev_speed[dv]);
}

template <int DPL, int MINB>
__global__ void __launch_bounds__(128, MINB) fate_score_v4_kernel(fate_bank b, fate_weights w,
                                                            fate_windows win, fate_derived der,
                                                            fate_state st, fate_work work,
                                                            fate_out out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int D = b.n_devices, Bmax = b.max_queries, LV = win.levels, OPS = win.max_level_ops;
    const int wi = threadIdx.x >> 5, t = threadIdx.x & 31;
    const long long item = (long long)blockIdx.x * 4 + wi;
    if (item >= work.n_items) return;  // whole warps exit together
    V4View V = v4_view(smem_raw + v4_item_bytes(D, Bmax, OPS) * wi, D, Bmax, OPS);
    const unsigned FULL = 0xffffffffu;
    const bool no_loc = w.ablation & FATE_NO_LOCALITY;
    const bool no_pre = w.ablation & FATE_NO_PREFIX;
    const bool no_same = w.ablation & FATE_NO_SAME_MODEL;
    const bool no_shard = w.ablation & FATE_NO_SHARD;
    const int H = w.eff_horizon;
    const int M1 = b.n_models + 1;

    V4Item it;
    it.s = work.scen[item];
    const int v = work.stage[item];
    it.v = v;
    const int inst = st.scen_inst[it.s];
    it.q0 = b.inst_query_off[inst];
    it.nq = b.inst_n_queries[inst];
    const int nq = it.nq;
    it.m = b.st_model[v];
    const int m = it.m;
    const int R = b.st_shard[v];
    it.gv = b.st_group[v];
    it.Pv = b.st_prompt[v];
    const uint64_t elig = b.st_elig[v];
    const double clock = st.scen_clock[it.s];
    it.cache_reuse = (b.st_flags[v] & FATE_STAGE_CACHE_REUSE) && it.gv != -1;
    const int32_t* loc_row = st.loc + st.scen_loc_off[it.s] - b.inst_stage_off[inst];
    it.dev_row0 = (long long)it.s * D;
    it.cap4 = st.kappa_cap * 4;
    it.kappa = st.kappa;
    it.kappa_n = st.kappa_n;
    {
        const int ri = b.st_role[v];
        it.pcoef = m >= 0 ? b.model_prefill[m] : 1.0;
        const double dcoef = m >= 0 ? b.model_decode[m] : 0.0;
        it.decode = (double)b.st_out[v] * dcoef * b.role_decode[ri];
        it.pscale = b.role_prefill[ri];
        it.cplx = b.role_cplx[ri];
    }
    const int pa0 = b.par_ptr[v], pa1 = b.par_ptr[v + 1];

    // ---- P0: device rows -------------------------------------------------------------
    int dv[DPL], res[DPL], cs[DPL], hit[DPL];
    bool live[DPL], ok[DPL];
    double fr[DPL], trv[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        dv[j] = t + 32 * j;
        live[j] = dv[j] < D;
        ok[j] = live[j] && ((elig >> dv[j]) & 1ull);
        res[j] = -1;
        cs[j] = 0;
        hit[j] = 0;
        fr[j] = 0.0;
        trv[j] = 0.0;
        if (live[j]) {
            const long long row = it.dev_row0 + dv[j];
            res[j] = st.residency[row];
            fr[j] = st.dev_free[row];
            cs[j] = it.Pv;  // effective stage part sp = max(0, P - cached), costs.py:86-88
            if (it.cache_reuse) {
                const int c = cached_tokens(st.kappa + row * it.cap4, st.kappa_n[row], it.gv, m);
                cs[j] = it.Pv - c > 0 ? it.Pv - c : 0;
            }
            V.key[dv[j]] = cs[j];
            V.sw[dv[j]] = (m < 0 || res[j] == m) ? 0.0 : b.model_switch[m] * w.switch_x;
        }
    }
    for (int e = pa0; e < pa1; ++e) {
        const int L = loc_row[b.par_idx[e]];
        if (L < 0) continue;
        const double sg = der.edge_sigma[e];
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            hit[j] += L == dv[j];
            if (live[j] && L != dv[j]) trv[j] += b.beta[(size_t)L * D + dv[j]] * sg;
        }
    }
#pragma unroll
    for (int j = 0; j < DPL; ++j)
        if (live[j]) V.tr[dv[j]] = trv[j] * w.transfer_x;
    const bool per_device_rows = der.inst_qgroups[inst] != 0;
    unsigned long long idle_m = 0ull, ok_m = 0ull;
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        idle_m |= (unsigned long long)__ballot_sync(FULL, ok[j] && fr[j] <= clock + 1e-12) << (32 * j);
        ok_m |= (unsigned long long)__ballot_sync(FULL, ok[j]) << (32 * j);
    }
    __syncwarp();

    // ---- P1: row classes ---------------------------------------------------------------
    int rep[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        const unsigned okj = (unsigned)(ok_m >> (32 * j));
        unsigned same = okj;
        if (!per_device_rows) {
            const unsigned long long spd = __double_as_longlong(b.dev_speed[live[j] ? dv[j] : 0]);
            same &= __match_any_sync(FULL, cs[j]) & __match_any_sync(FULL, spd);
        } else {
            same &= 1u << t;
        }
        rep[j] = ok[j] ? 32 * j + __ffs(same) - 1 : -1;
    }
    if (DPL == 2 && !per_device_rows) {
        // a slot-1 class may already exist among slot-0 devices
        const unsigned reps0 = __ballot_sync(FULL, ok[0] && rep[0] == dv[0]);
        if (ok[DPL - 1]) {
            unsigned rr = reps0;
            const double sp = b.dev_speed[dv[DPL - 1]];
            while (rr) {
                const int e = __ffs(rr) - 1;
                rr &= rr - 1;
                if (V.key[e] == cs[DPL - 1] && b.dev_speed[e] == sp) {
                    rep[DPL - 1] = e;
                    break;
                }
            }
        }
    }
    unsigned long long rep_m = 0ull;
#pragma unroll
    for (int j = 0; j < DPL; ++j)
        rep_m |= (unsigned long long)__ballot_sync(FULL, ok[j] && rep[j] == dv[j]) << (32 * j);
    const int n_cls = __popcll(rep_m);
    int cls[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        cls[j] = ok[j] ? __popcll(rep_m & low_mask(rep[j])) : -1;
        if (ok[j]) {
            V.rowc[dv[j]] = cls[j];
            if (rep[j] == dv[j]) V.rowdev[cls[j]] = dv[j];
        }
    }
    const int n_idle = __popcll(idle_m);
    int kb = 0, ki = 0;
    if (R > 1 && !no_shard) {
        kb = R < 1 + n_idle ? R : 1 + n_idle;
        ki = R < n_idle ? R : n_idle;
    }
    const bool kb_ok = kb >= 2 && kb <= V4_KT;
    const bool ki_ok = ki != kb && ki >= 2 && ki <= V4_KT;
    const int per = 1 + (kb_ok ? kb : 0) + (ki_ok ? ki : 0);
    // static classes (uniform speed, no query prefix groups): the stateless row
    // sp = P (class A) and the full-hit row sp = 0 (class B) have their sums in
    // the prologue table row_sums[v][0..5]
    int cA = -1, cB = -1;
    if ((b.flags & FATE_BANK_UNIFORM_SPEED) && !per_device_rows && kb <= 2 && ki <= 2) {
        unsigned long long am = 0ull, bm = 0ull;
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            const bool r0 = ok[j] && rep[j] == dv[j];
            am |= (unsigned long long)__ballot_sync(FULL, r0 && cs[j] == it.Pv) << (32 * j);
            bm |= (unsigned long long)__ballot_sync(FULL, r0 && cs[j] == 0 && it.Pv > 0) << (32 * j);
        }
        if (am) cA = __popcll(rep_m & low_mask(__ffsll((long long)am) - 1));
        if (bm) cB = __popcll(rep_m & low_mask(__ffsll((long long)bm) - 1));
    }
    // dynamic classes: rows in shared memory for the first RCAP of them
    unsigned long long dyn_m = n_cls >= 64 ? ~0ull : ((1ull << n_cls) - 1ull);
    if (cA >= 0) dyn_m &= ~(1ull << cA);
    if (cB >= 0) dyn_m &= ~(1ull << cB);
    const int n_dyn = __popcll(dyn_m);
    const int n_rows = n_dyn < V4_RCAP ? n_dyn : V4_RCAP;
    if (t == 0) {
        unsigned long long mm = dyn_m;
        for (int r = 0; r < n_rows; ++r) {
            V.slot2cls[r] = __ffsll((long long)mm) - 1;
            mm &= mm - 1;
        }
        const double* z = der.row_sums + (size_t)v * 6;
#pragma unroll
        for (int sidx = 0; sidx < 2; ++sidx) {
            const int c = sidx == 0 ? cA : cB;
            if (c < 0) continue;
            const double* zz = z + 3 * sidx;
            V.aware[c] = zz[0];
            if (kb == 2) {
                V.shard[(c * 2 + 0) * V4_KT + 0] = zz[1];
                V.shard[(c * 2 + 0) * V4_KT + 1] = zz[2];
            }
            if (ki == 2 && ki != kb) {
                V.shard[(c * 2 + 1) * V4_KT + 0] = zz[1];
                V.shard[(c * 2 + 1) * V4_KT + 1] = zz[2];
            }
        }
    }
    __syncwarp();

    // ---- P2: dynamic class rows and sums -----------------------------------------------
    for (int p = t; p < n_rows * nq; p += 32) {
        const int r = p / nq, q = p - r * nq;
        V.rows[r * Bmax + q] = v4_qc(b, it, V, V.rowdev[V.slot2cls[r]], q);
    }
    __syncwarp();
    {
        const int n_row_tasks = n_rows * per;
        const int n_tasks = n_row_tasks + (n_dyn - n_rows);
        for (int p = t; p < n_tasks; p += 32) {
            PySum acc;
            if (p >= n_row_tasks) {  // dynamic class beyond RCAP: direct aware
                unsigned long long mm = dyn_m;
                for (int r = 0; r < n_rows + (p - n_row_tasks); ++r) mm &= mm - 1;
                const int c = __ffsll((long long)mm) - 1;
                const int dd = V.rowdev[c];
                for (int q = 0; q < nq; ++q) acc.add(v4_qc(b, it, V, dd, q));
                V.aware[c] = acc.result();
                continue;
            }
            const int r = p / per;
            const int c = V.slot2cls[r];
            int j = p - r * per;
            const double* row = V.rows + r * Bmax;
            if (j == 0) {
                for (int q = 0; q < nq; ++q) acc.add(row[q]);
                V.aware[c] = acc.result();
            } else {
                j -= 1;
                int kslot = 0, k = kb;
                if (!kb_ok || j >= kb) {
                    if (kb_ok) j -= kb;
                    kslot = 1;
                    k = ki;
                }
                int lo, hi;
                shard_range(nq, k, j, &lo, &hi);
                for (int q = lo; q < hi; ++q) acc.add(row[q]);
                V.shard[(c * 2 + kslot) * V4_KT + j] = acc.result();
            }
        }
    }
    __syncwarp();

    // ---- P3: tail ------------------------------------------------------------------------------
    double tail[DPL];
    int dmc[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        tail[j] = 0.0;
        dmc[j] = (live[j] && res[j] != -1 && res[j] != m && res[j] < b.n_models) ? res[j] : -1;
    }
    if (H > 1) {
        for (int l = 0; l < LV; ++l) {
            const long long lo = win.ptr[(long long)v * LV + l];
            const long long hi = win.ptr[(long long)v * LV + l + 1];
            if (hi == lo) continue;
            const int n_b = (int)(hi - lo);
            const long long vl = (long long)v * LV + l;
            double aff[DPL];
            {
                const double* row = der.tail_static + vl * M1;
#pragma unroll
                for (int j = 0; j < DPL; ++j) aff[j] = row[1 + dmc[j]];
            }
            bool located = false;
            if (!no_loc) {
                const long long w1 = win.wpar_ptr[vl + 1];
                for (long long i = win.wpar_ptr[vl] + t; i < w1; i += 32)
                    located |= loc_row[win.wpar_idx[i]] >= 0;
            }
            if (__any_sync(FULL, located)) {
                int base = 0;
                for (int j0 = 0; j0 < n_b; j0 += 32) {
                    const int jx = j0 + t;
                    int x = -1, mx = -1, cnt = 0;
                    bool same_op = false, disp_op = false, pre_op = false;
                    if (jx < n_b) {
                        x = win.idx[lo + jx];
                        mx = b.st_model[x];
                        if (!no_same && mx != -1) {
                            same_op = mx == m;
                            disp_op = !same_op;
                        }
                        const int gx = b.st_group[x];
                        pre_op = !no_pre && gx != -1 && gx == it.gv;
                        cnt = (same_op || disp_op) + pre_op;
                        for (int e = b.par_ptr[x]; e < b.par_ptr[x + 1]; ++e) {
                            const int pp = b.par_idx[e];
                            cnt += pp != v && loc_row[pp] >= 0;
                        }
                    }
                    int incl = cnt;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(FULL, incl, o);
                        if (t >= o) incl += y;
                    }
                    int pos = base + incl - cnt;
                    base += __shfl_sync(FULL, incl, 31);
                    if (jx < n_b) {
                        if (same_op || disp_op) {
                            const double bonus =
                                w.lambda_s * b.model_switch[mx] * w.switch_x * w.state_scale;
                            V4Op op;
                            op.val = same_op ? bonus : -bonus;
                            op.key = same_op ? -1 : mx;
                            op.kind = same_op ? 0 : 1;
                            V.ops[pos++] = op;
                        }
                        if (pre_op) {
                            const int Px = b.st_prompt[x];
                            const int shared = it.Pv < Px ? it.Pv : Px;
                            V4Op op;
                            op.val = w.lambda_p * w.kappa_prefix * (double)shared / 1000.0 *
                                     w.prefix_x * w.prefix_scale;
                            op.key = -1;
                            op.kind = 0;
                            V.ops[pos++] = op;
                        }
                        for (int e = b.par_ptr[x]; e < b.par_ptr[x + 1]; ++e) {
                            const int pp = b.par_idx[e];
                            if (pp == v) continue;
                            const int L = loc_row[pp];
                            if (L < 0) continue;
                            V4Op op;
                            if (b.has_overrides) {
                                op.val = der.edge_sigma[e];
                                op.kind = 2;
                            } else {
                                op.val = -der.edge_term[e];
                                op.kind = 0;
                            }
                            op.key = L;
                            V.ops[pos++] = op;
                        }
                    }
                }
                __syncwarp();
#pragma unroll
                for (int j = 0; j < DPL; ++j) aff[j] = 0.0;
                if (!b.has_overrides) {
                    // aff starts at +0.0 and, in round-to-nearest, never becomes -0.0, so
                    // adding +0.0 for a skipped op leaves it bit-identical: branch-free walk
#pragma unroll 4
                    for (int o = 0; o < base; ++o) {
                        const V4Op op = V.ops[o];
#pragma unroll
                        for (int j = 0; j < DPL; ++j) {
                            const bool apply = op.kind == 1 ? op.key == dmc[j] : op.key != dv[j];
                            aff[j] += apply ? op.val : 0.0;
                        }
                    }
                } else {
                    for (int o = 0; o < base; ++o) {
                        const V4Op op = V.ops[o];
#pragma unroll
                        for (int j = 0; j < DPL; ++j) {
                            if (op.kind == 0) {
                                if (op.key != dv[j]) aff[j] += op.val;
                            } else if (op.kind == 1) {
                                if (op.key == dmc[j]) aff[j] += op.val;
                            } else if (op.key != dv[j]) {
                                aff[j] -= w.lambda_tr *
                                          b.beta[(size_t)op.key * D + (live[j] ? dv[j] : 0)] *
                                          op.val * w.transfer_x * w.locality_scale;
                            }
                        }
                    }
                }
                __syncwarp();  // op buffer reused by the next level
            }
            const double dem = der.demand[(long long)v * LV + l];
#pragma unroll
            for (int j = 0; j < DPL; ++j)
                tail[j] += w.gamma_pow[l + 1] * (aff[j] / (double)n_b + w.demand_coeff * dem);
        }
    }

    // ---- P4: per-device assembly ---------------------------------------------------------------
    const int n_elig = __popcll(elig);
    const int bound = no_shard ? 1 : (R < n_elig ? R : n_elig);
    double* psi = out.psi + work.psi_off[item];
    double bb = 0.0;
    for (int c = 0; c < n_cls; ++c) bb = (c == 0 || V.aware[c] < bb) ? V.aware[c] : bb;
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        if (!live[j]) continue;
        const int d = dv[j];
        const long long orow = item * D + d;
        if (!ok[j]) {
            const double qnan = __longlong_as_double(0x7ff8000000000000LL);
            for (int k = 0; k < bound; ++k) psi[(long long)k * D + d] = qnan;
            if (out.sched) out.sched[orow] = qnan;
            if (out.tail) out.tail[orow] = qnan;
            if (out.completion) out.completion[orow] = qnan;
            continue;
        }
        const double wait = py_max0(fr[j] - clock);
        const double sw = V.sw[d];
        const double tr = V.tr[d];
        const double here = V.aware[cls[j]];
        const double colo = pa1 > pa0 ? (double)hit[j] / (double)(pa1 - pa0) : 0.0;

        // prefix_overlap_thousands (costs.py:127-145), integer-exact
        long long tokens = 0;
        if (it.cache_reuse) tokens += it.Pv - cs[j];  // min(cached, P) = P - sp
        if (per_device_rows) {
            const long long row = it.dev_row0 + d;
            const int32_t* kap = st.kappa + row * it.cap4;
            const int kn = st.kappa_n[row];
            for (int q = 0; q < nq; ++q) {
                const int qg = b.q_group[it.q0 + q];
                if (qg == -1) continue;
                const long long c = cached_tokens(kap, kn, qg, m);
                const long long qp = b.q_prompt[it.q0 + q];
                tokens += c < qp ? c : qp;
            }
        }
        const double prefix = w.kappa_prefix * ((double)tokens / 1000.0) * w.prefix_x;

        // _parallel_benefit (costs.py:181-201)
        const double full_total = sw + tr + here;
        double parallel = 0.0;
        if (R > 1 && !no_shard) {
            const bool self_idle = (idle_m >> d) & 1ull;
            const int others = n_idle - (self_idle ? 1 : 0);
            const int k = R < 1 + others ? R : 1 + others;
            if (k > 1) {
                const int kslot = (k == kb && kb_ok) ? 0 : 1;
                const bool tab = kslot == 0 || (k == ki && ki_ok);
                unsigned long long rest = idle_m & ~(1ull << d);
                double worst = 0.0;
                for (int i = 0; i < k; ++i) {
                    int dev = d;
                    if (i > 0) {
                        dev = __ffsll((long long)rest) - 1;
                        rest &= rest - 1;
                    }
                    const int cd = V.rowc[dev];
                    const bool is_static = cd == cA || cd == cB;
                    const int r = is_static ? -1 : __popcll(dyn_m & low_mask(cd));
                    const int slot = (r >= 0 && r < n_rows) ? r : -1;
                    double ssum;
                    if (tab && (is_static || slot >= 0)) {
                        ssum = V.shard[(cd * 2 + kslot) * V4_KT + i];
                    } else {
                        int lo, hi;
                        shard_range(nq, k, i, &lo, &hi);
                        PySum acc;
                        for (int q = lo; q < hi; ++q)
                            acc.add(slot >= 0 ? V.rows[slot * Bmax + q] : v4_qc(b, it, V, dev, q));
                        ssum = acc.result();
                    }
                    const double tot = V.sw[dev] + V.tr[dev] + ssum;
                    if (i == 0 || tot > worst) worst = tot;
                }
                const double overhead = w.shard_overhead_frac * here * (double)(k - 1);
                parallel = py_max0(full_total - worst - overhead);
            }
        }

        // sched_score (costs.py:210-231)
        const double tr_s = no_loc ? 0.0 : tr;
        const double colo_s = no_loc ? 0.0 : colo;
        const double prefix_s = no_pre ? 0.0 : prefix;
        const double par_s = no_shard ? 0.0 : parallel;
        const double S = -w.lambda_q * wait - w.lambda_s * sw * w.state_scale
                         - w.lambda_tr * tr_s * w.locality_scale
                         + w.lambda_c * colo_s * w.locality_scale
                         + w.lambda_p * prefix_s * w.prefix_scale + w.lambda_r * par_s;

        if (out.sched) out.sched[orow] = S;
        if (out.tail) out.tail[orow] = tail[j];
        if (out.completion) out.completion[orow] = wait + full_total;
        psi[d] = S + tail[j];

        // _marginal_shard_score (costs.py:249-279)
        if (bound > 1) {
            const double hi_v = here > bb ? here : bb;
            const double overhead = w.shard_overhead_frac * bb;
            const double tr_m = no_loc ? 0.0 : tr;
            const double split = no_loc ? 0.0 : der.split_penalty[v];
            for (int k = 1; k < bound; ++k) {
                const double reduction = bb / (double)k - hi_v / (double)(k + 1);
                psi[(long long)k * D + d] = w.lambda_r * (reduction - overhead) -
                                            w.lambda_q * wait - w.lambda_s * sw * w.state_scale -
                                            w.lambda_tr * (tr_m + split) * w.locality_scale;
            }
        }
    }
}
