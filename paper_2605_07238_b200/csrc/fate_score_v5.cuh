// fate_score_v5.cuh -- warp-per-item scoring kernel (production path).
//
// Included by fate_kernels.cu (inside its anonymous namespace).
//
// One warp owns one item = (scenario, stage v); lane t owns devices t and
// t+32 (DPL = 1 for D <= 32, 2 for D <= 64).  An item only ever synchronises
// its own warp; four items per 128-thread CTA run independently.
//
// Latency structure: every global load that does not depend on device state
// is issued up front -- the horizon-level metadata (bucket ranges, window-parent
// ranges, static tail rows, demand) and the "any located parent?" gather of
// each level -- so that its latency overlaps the device-state phase.  v's
// parent edges are fetched lane-parallel and broadcast with shuffles instead of
// a sequential dependent-load loop.
//
//   P0  per device: residency, free time, effective stage part
//       sp = max(0, P(v) - cached stage-group tokens) (costs.py:86-88), wait,
//       switch; transfer and colo from the broadcast parent list
//       (costs.py:107-125, 160-165); idle mask by ballot.
//   P1  row classes: equal (sp, speed) => bit-identical cache-aware
//       query_compute row (costs.py:70-94), found with __match_any_sync.
//       Under uniform speed and no query prefix groups the classes sp = P
//       (stateless row) and sp = 0 (full prefix hit) are static: their
//       Neumaier sums come from the prologue table row_sums.
//   P2  rows of the other (dynamic) classes in shared memory (<= RCAP), then
//       every Neumaier sum the reference takes: full batch (costs.py:257,
//       :404) and the shard ranges of the <= 2 shard counts used (:404-405).
//   P3  tail (costs.py:281-352) per level: no located parent edge => static
//       table row[displacement class]; else an ordered op list (warp scan;
//       signed values, a - b == a + (-b) exactly) walked branch-free by every
//       lane for its device slots (+0.0 for a skipped op is exact: the chain
//       starts at +0.0 and never becomes -0.0 in round-to-nearest).
//   P4  per device: colo, prefix overlap (= P - sp), parallel benefit, S,
//       tail, Psi(slot 0..bound-1), completion.

constexpr int V5_KT = 4;    // shard counts k <= V5_KT: shard sums tabulated per slot
constexpr int V5_RCAP = 8;  // dynamic classes with a shared-memory row
constexpr int V5_SLOTS = V5_RCAP + 2;  // table slots: 0 = static A, 1 = static B, 2+ = rows
constexpr int V5_PLV = 3;   // horizon levels whose metadata is prefetched into registers
constexpr int V5_KEY_MODEL = 1000;     // op key >= this: displacement op of model key-1000
constexpr int V5_KEY_SIGMA = 2000;     // op key >= this: override locality op, device key-2000

struct V5View {
    double* rows;     // [RCAP*Bmax]
    double* shard;    // [SLOTS*2*KT]
    double* aware;    // [SLOTS]
    double* sw;       // [D]
    double* tr;       // [D]
    double* opval;    // [ops_cap]
    int* opkey;       // [ops_cap]
    int* key;         // [D] effective stage part per device
    int* cslot;       // [D] table slot of the device's class (-1: direct)
    int* rowdev;      // [RCAP] representative device of each row slot
};

__host__ __device__ inline size_t v5_item_bytes(int D, int Bmax, int ops_cap) {
    size_t dbl = (size_t)V5_RCAP * Bmax + (size_t)V5_SLOTS * 2 * V5_KT + V5_SLOTS + 2 * (size_t)D +
                 ops_cap;
    size_t ints = (size_t)ops_cap + 2 * (size_t)D + V5_RCAP;
    return (dbl * 8 + ints * 4 + 15) & ~size_t(15);
}

__device__ inline V5View v5_view(unsigned char* base, int D, int Bmax, int ops_cap) {
    V5View v;
    double* dp = reinterpret_cast<double*>(base);
    v.rows = dp; dp += (size_t)V5_RCAP * Bmax;
    v.shard = dp; dp += (size_t)V5_SLOTS * 2 * V5_KT;
    v.aware = dp; dp += V5_SLOTS;
    v.sw = dp; dp += D;
    v.tr = dp; dp += D;
    v.opval = dp; dp += ops_cap;
    int* ip = reinterpret_cast<int*>(dp);
    v.opkey = ip; ip += ops_cap;
    v.key = ip; ip += D;
    v.cslot = ip; ip += D;
    v.rowdev = ip;
    return v;
}

struct V5Item {
    int q0, nq, m, Pv;
    long long dev_row0;
    int cap4;
    double pcoef, pscale, decode, cplx;
};

// cache-aware query_compute of query q on device dv (costs.py:70-94); the
// stage part is the device's effective sp
__device__ __forceinline__ double v5_qc(const fate_bank& b, const fate_state& st, const V5Item& it,
                                        const V5View& V, int dv, int q) {
    const long long sp = V.key[dv];
    long long qp = b.q_prompt[it.q0 + q];
    const int qg = b.q_group[it.q0 + q];
    if (qg != -1) {
        const long long drow = it.dev_row0 + dv;
        const long long cc = cached_tokens(st.kappa + drow * it.cap4, st.kappa_n[drow], qg, it.m);
        qp = qp - cc > 0 ? qp - cc : 0;
    }
    return qc_value(sp, qp, it.pcoef, it.pscale, it.decode, it.cplx, b.dev_speed[dv]);
}

template <int DPL, int MINB>
__global__ void __launch_bounds__(128, MINB) fate_score_v5_kernel(fate_bank b, fate_weights w,
                                                                  fate_windows win,
                                                                  fate_derived der, fate_state st,
                                                                  fate_work work, fate_out out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int D = b.n_devices, Bmax = b.max_queries, LV = win.levels, OPS = win.max_level_ops;
    const int wi = threadIdx.x >> 5, t = threadIdx.x & 31;
    const long long item = (long long)blockIdx.x * 4 + wi;
    if (item >= work.n_items) return;  // whole warps exit together
    V5View V = v5_view(smem_raw + v5_item_bytes(D, Bmax, OPS) * wi, D, Bmax, OPS);
    const unsigned FULL = 0xffffffffu;
    const bool no_loc = w.ablation & FATE_NO_LOCALITY;
    const bool no_pre = w.ablation & FATE_NO_PREFIX;
    const bool no_same = w.ablation & FATE_NO_SAME_MODEL;
    const bool no_shard = w.ablation & FATE_NO_SHARD;
    const int H = w.eff_horizon;
    const int M1 = b.n_models + 1;

    // ---- item header ------------------------------------------------------------------------
    const int s = work.scen[item];
    const int v = work.stage[item];
    const int inst = st.scen_inst[s];
    V5Item it;
    it.m = b.st_model[v];
    const int m = it.m;
    const int R = b.st_shard[v];
    const int gv = b.st_group[v];
    it.Pv = b.st_prompt[v];
    const uint64_t elig = b.st_elig[v];
    const bool cache_reuse = (b.st_flags[v] & FATE_STAGE_CACHE_REUSE) && gv != -1;
    const int pa0 = b.par_ptr[v], pa1 = b.par_ptr[v + 1];
    const double clock = st.scen_clock[s];
    it.q0 = b.inst_query_off[inst];
    it.nq = b.inst_n_queries[inst];
    const int nq = it.nq;
    const int32_t* loc_row = st.loc + st.scen_loc_off[s] - b.inst_stage_off[inst];
    it.dev_row0 = (long long)s * D;
    it.cap4 = st.kappa_cap * 4;

    // ---- prefetch: located-parent flag per horizon level and the static full tail --------
    int res0[DPL];
    bool live[DPL];
    double tail_full[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        live[j] = t + 32 * j < D;
        res0[j] = live[j] ? st.residency[it.dev_row0 + t + 32 * j] : -1;
        tail_full[j] = 0.0;
    }
    const bool do_tail = H > 1;
    unsigned walk_m = 0u;  // bit l: level l has a locality op (needs the op-list walk)
    if (do_tail) {
        const double* row = der.tail_sum + (size_t)v * M1;
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            const int r = res0[j];
            tail_full[j] = row[(r != -1 && r != m && r < b.n_models) ? 1 + r : 0];
        }
        if (!no_loc) {
            // a window parent above the scenario's highest located stage cannot be
            // located: levels whose parents all lie above it need no gather
            const int done_lvl = st.scen_done_level[s];
            for (int l = 0; l < LV; ++l) {
                const long long vl = (long long)v * LV + l;
                if (win.wpar_minlvl[vl] > done_lvl) continue;
                const long long w1 = win.wpar_ptr[vl + 1];
                bool located = false;
                for (long long i = win.wpar_ptr[vl] + t; i < w1; i += 32)
                    located |= loc_row[win.wpar_idx[i]] >= 0;
                if (__any_sync(FULL, located)) walk_m |= 1u << (l < 31 ? l : 31);
            }
        }
    }
    const double rsum = t < 6 ? der.row_sums[(size_t)v * 6 + t] : 0.0;  // static-class sums
    {
        const int ri = b.st_role[v];
        it.pcoef = m >= 0 ? b.model_prefill[m] : 1.0;
        const double dcoef = m >= 0 ? b.model_decode[m] : 0.0;
        it.decode = (double)b.st_out[v] * dcoef * b.role_decode[ri];
        it.pscale = b.role_prefill[ri];
        it.cplx = b.role_cplx[ri];
    }

    // ---- P0: device rows ----------------------------------------------------------------------
    int dv[DPL], cs[DPL], hit[DPL];
    bool ok[DPL];
    double fr[DPL], trv[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        dv[j] = t + 32 * j;
        ok[j] = live[j] && ((elig >> dv[j]) & 1ull);
        cs[j] = it.Pv;
        hit[j] = 0;
        fr[j] = 0.0;
        trv[j] = 0.0;
        if (live[j]) {
            const long long row = it.dev_row0 + dv[j];
            fr[j] = st.dev_free[row];
            if (cache_reuse) {
                const int c = cached_tokens(st.kappa + row * it.cap4, st.kappa_n[row], gv, m);
                cs[j] = it.Pv - c > 0 ? it.Pv - c : 0;
            }
            V.key[dv[j]] = cs[j];
            V.sw[dv[j]] = (m < 0 || res0[j] == m) ? 0.0 : b.model_switch[m] * w.switch_x;
        }
    }
    // v's parents: lane-parallel fetch, broadcast in ascending order
    for (int e0 = pa0; e0 < pa1; e0 += 32) {
        const int e = e0 + t;
        int L = -1;
        double sg = 0.0;
        if (e < pa1) {
            L = loc_row[b.par_idx[e]];
            sg = der.edge_sigma[e];
        }
        const int n = pa1 - e0 < 32 ? pa1 - e0 : 32;
        for (int i = 0; i < n; ++i) {
            const int Li = __shfl_sync(FULL, L, i);
            const double si = __shfl_sync(FULL, sg, i);
            if (Li < 0) continue;
#pragma unroll
            for (int j = 0; j < DPL; ++j) {
                hit[j] += Li == dv[j];
                if (live[j] && Li != dv[j]) trv[j] += b.beta[(size_t)Li * D + dv[j]] * si;
            }
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

    // ---- P1: row classes ------------------------------------------------------------------------
    int rep[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        unsigned same = (unsigned)(ok_m >> (32 * j));
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
    const int n_idle = __popcll(idle_m);
    int kb = 0, ki = 0;
    if (R > 1 && !no_shard) {
        kb = R < 1 + n_idle ? R : 1 + n_idle;
        ki = R < n_idle ? R : n_idle;
    }
    const bool kb_ok = kb >= 2 && kb <= V5_KT;
    const bool ki_ok = ki != kb && ki >= 2 && ki <= V5_KT;
    const int per = 1 + (kb_ok ? kb : 0) + (ki_ok ? ki : 0);
    // static classes: representatives with sp == P (A) and sp == 0 < P (B)
    unsigned long long am = 0ull, bm = 0ull;
    if ((b.flags & FATE_BANK_UNIFORM_SPEED) && !per_device_rows && kb <= 2 && ki <= 2) {
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            const bool r0 = ok[j] && rep[j] == dv[j];
            am |= (unsigned long long)__ballot_sync(FULL, r0 && cs[j] == it.Pv) << (32 * j);
            bm |= (unsigned long long)__ballot_sync(FULL, r0 && cs[j] == 0 && it.Pv > 0) << (32 * j);
        }
    }
    const unsigned long long dyn_m = rep_m & ~am & ~bm;  // representatives of dynamic classes
    const int n_dyn = __popcll(dyn_m);
    const int n_rows = n_dyn < V5_RCAP ? n_dyn : V5_RCAP;
    // table slot of each device's class: 0 = A, 1 = B, 2 + row slot, -1 = direct
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        if (!ok[j]) continue;
        const unsigned long long rb = 1ull << rep[j];
        int slot;
        if (am & rb) slot = 0;
        else if (bm & rb) slot = 1;
        else {
            const int r = __popcll(dyn_m & low_mask(rep[j]));
            slot = r < V5_RCAP ? 2 + r : -1;
            if (rep[j] == dv[j] && r < V5_RCAP) V.rowdev[r] = dv[j];
        }
        V.cslot[dv[j]] = slot;
    }
    if (t < 6) {
        // lane t holds row_sums[v][t]: class si = t / 3, entry e = t % 3 (full, shard 0, 1)
        const int si = t / 3, e = t - 3 * si;
        if (si == 0 ? am != 0ull : bm != 0ull) {
            if (e == 0) {
                V.aware[si] = rsum;
            } else {
                if (kb == 2) V.shard[(si * 2 + 0) * V5_KT + (e - 1)] = rsum;
                if (ki == 2 && ki != kb) V.shard[(si * 2 + 1) * V5_KT + (e - 1)] = rsum;
            }
        }
    }
    __syncwarp();

    // ---- P2: dynamic class rows and sums -------------------------------------------------
    for (int p = t; p < n_rows * nq; p += 32) {
        const int r = p / nq, q = p - r * nq;
        V.rows[r * Bmax + q] = v5_qc(b, st, it, V, V.rowdev[r], q);
    }
    __syncwarp();
    for (int p = t; p < n_rows * per; p += 32) {
        const int r = p / per;
        int j = p - r * per;
        const double* row = V.rows + r * Bmax;
        const int slot = 2 + r;
        PySum acc;
        if (j == 0) {
            for (int q = 0; q < nq; ++q) acc.add(row[q]);
            V.aware[slot] = acc.result();
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
            V.shard[(slot * 2 + kslot) * V5_KT + j] = acc.result();
        }
    }
    __syncwarp();

    // aware per device and base_best (costs.py:257-259); classes without a slot
    // (more than RCAP dynamic classes) are summed directly by their lanes
    double here[DPL];
    double bb = 0.0;
    {
        bool have = false;
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            here[j] = 0.0;
            if (!ok[j]) continue;
            const int slot = V.cslot[dv[j]];
            if (slot >= 0) {
                here[j] = V.aware[slot];
            } else {
                PySum acc;
                for (int q = 0; q < nq; ++q) acc.add(v5_qc(b, st, it, V, dv[j], q));
                here[j] = acc.result();
            }
            if (!have || here[j] < bb) bb = here[j];
            have = true;
        }
        // warp min over lanes with a value (min is order-free)
        double cand = have ? bb : __longlong_as_double(0x7ff0000000000000LL);  // +inf
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(FULL, cand, o);
            cand = y < cand ? y : cand;
        }
        bb = cand;
    }

    // ---- P3: tail ---------------------------------------------------------------------------------
    double tail[DPL];
    int dmc[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        tail[j] = 0.0;
        dmc[j] = (live[j] && res0[j] != -1 && res0[j] != m && res0[j] < b.n_models) ? res0[j] : -1;
    }
    if (do_tail && walk_m == 0u) {
        // no locality op anywhere in the horizon: the whole tail is static
#pragma unroll
        for (int j = 0; j < DPL; ++j) tail[j] = tail_full[j];
    } else if (do_tail) {
        for (int l = 0; l < LV; ++l) {
            const long long vl = (long long)v * LV + l;
            const long long lo = win.ptr[vl];
            const int n_b = (int)(win.ptr[vl + 1] - lo);
            if (n_b == 0) continue;
            const double dml = der.demand[vl];
            double aff[DPL];
            const bool wl = (walk_m >> (l < 31 ? l : 31)) & 1u;
            if (!wl) {
                // static level: its term is tabulated (fate_prepare_tail_static_kernel)
                const double* row = der.tail_static + vl * M1;
#pragma unroll
                for (int j = 0; j < DPL; ++j) tail[j] += row[1 + dmc[j]];
                continue;
            } else {
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
                        pre_op = !no_pre && gx != -1 && gx == gv;
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
                            V.opval[pos] = same_op ? bonus : -bonus;
                            V.opkey[pos] = same_op ? -1 : V5_KEY_MODEL + mx;
                            ++pos;
                        }
                        if (pre_op) {
                            const int Px = b.st_prompt[x];
                            const int shared = it.Pv < Px ? it.Pv : Px;
                            V.opval[pos] = w.lambda_p * w.kappa_prefix * (double)shared / 1000.0 *
                                           w.prefix_x * w.prefix_scale;
                            V.opkey[pos] = -1;
                            ++pos;
                        }
                        for (int e = b.par_ptr[x]; e < b.par_ptr[x + 1]; ++e) {
                            const int pp = b.par_idx[e];
                            if (pp == v) continue;
                            const int L = loc_row[pp];
                            if (L < 0) continue;
                            if (b.has_overrides) {
                                V.opval[pos] = der.edge_sigma[e];
                                V.opkey[pos] = V5_KEY_SIGMA + L;
                            } else {
                                V.opval[pos] = -der.edge_term[e];
                                V.opkey[pos] = L;
                            }
                            ++pos;
                        }
                    }
                }
                __syncwarp();
#pragma unroll
                for (int j = 0; j < DPL; ++j) aff[j] = 0.0;
                if (!b.has_overrides) {
                    int tgt[DPL];
#pragma unroll
                    for (int j = 0; j < DPL; ++j) tgt[j] = V5_KEY_MODEL + dmc[j];
#pragma unroll 4
                    for (int o = 0; o < base; ++o) {
                        const int k = V.opkey[o];
                        const double val = V.opval[o];
                        const bool model_op = k >= V5_KEY_MODEL;
#pragma unroll
                        for (int j = 0; j < DPL; ++j) {
                            const bool apply = model_op ? k == tgt[j] : k != dv[j];
                            aff[j] += apply ? val : 0.0;
                        }
                    }
                } else {
                    for (int o = 0; o < base; ++o) {
                        const int k = V.opkey[o];
                        const double val = V.opval[o];
#pragma unroll
                        for (int j = 0; j < DPL; ++j) {
                            if (k < V5_KEY_MODEL) {
                                if (k != dv[j]) aff[j] += val;
                            } else if (k < V5_KEY_SIGMA) {
                                if (k - V5_KEY_MODEL == dmc[j]) aff[j] += val;
                            } else if (k - V5_KEY_SIGMA != dv[j]) {
                                aff[j] -= w.lambda_tr *
                                          b.beta[(size_t)(k - V5_KEY_SIGMA) * D +
                                                 (live[j] ? dv[j] : 0)] *
                                          val * w.transfer_x * w.locality_scale;
                            }
                        }
                    }
                }
                __syncwarp();  // op buffer reused by the next level
            }
#pragma unroll
            for (int j = 0; j < DPL; ++j)
                tail[j] += w.gamma_pow[l + 1] * (aff[j] / (double)n_b + w.demand_coeff * dml);
        }
    }

    // ---- P4: per-device assembly ----------------------------------------------------------------
    const int n_elig = __popcll(elig);
    const int bound = no_shard ? 1 : (R < n_elig ? R : n_elig);
    double* psi = out.psi + work.psi_off[item];
    const double split = no_loc ? 0.0 : (bound > 1 ? der.split_penalty[v] : 0.0);
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
        // 0 / n == +0.0 exactly: divide only when a parent is co-located
        const double colo = (pa1 > pa0 && hit[j] > 0) ? (double)hit[j] / (double)(pa1 - pa0) : 0.0;

        // prefix_overlap_thousands (costs.py:127-145), integer-exact
        long long tokens = 0;
        if (cache_reuse) tokens += it.Pv - cs[j];  // min(cached, P) = P - sp
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
        const double prefix =
            w.kappa_prefix * (tokens == 0 ? 0.0 : (double)tokens / 1000.0) * w.prefix_x;

        // _parallel_benefit (costs.py:181-201)
        const double full_total = sw + tr + here[j];
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
                    const int slot = V.cslot[dev];
                    double ssum;
                    if (tab && slot >= 0) {
                        ssum = V.shard[(slot * 2 + kslot) * V5_KT + i];
                    } else {
                        int lo, hi;
                        shard_range(nq, k, i, &lo, &hi);
                        PySum acc;
                        for (int q = lo; q < hi; ++q)
                            acc.add(slot >= 2 ? V.rows[(slot - 2) * Bmax + q]
                                              : v5_qc(b, st, it, V, dev, q));
                        ssum = acc.result();
                    }
                    const double tot = V.sw[dev] + V.tr[dev] + ssum;
                    if (i == 0 || tot > worst) worst = tot;
                }
                const double overhead = w.shard_overhead_frac * here[j] * (double)(k - 1);
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
            const double hv = here[j] > bb ? here[j] : bb;
            const double overhead = w.shard_overhead_frac * bb;
            const double tr_m = no_loc ? 0.0 : tr;
            for (int k = 1; k < bound; ++k) {
                // x / 1 == x and x / 2 == x * 0.5 exactly (both correctly rounded x/2)
                const double q1 = k == 1 ? bb : bb / (double)k;
                const double q2 = k == 1 ? hv * 0.5 : hv / (double)(k + 1);
                const double reduction = q1 - q2;
                psi[(long long)k * D + d] = w.lambda_r * (reduction - overhead) -
                                            w.lambda_q * wait - w.lambda_s * sw * w.state_scale -
                                            w.lambda_tr * (tr_m + split) * w.locality_scale;
            }
        }
    }
}
