// fate_score_v2.cuh -- class-deduplicated, CTA-pooled scoring kernel.
//
// Included by fate_kernels.cu (inside its anonymous namespace).
//
// Why: in v1 every device lane recomputed its own query_compute row, its own
// Neumaier sums and its own horizon-tail chain, although for one (scenario,
// stage) item most devices produce bit-identical values (same cached-token
// amount, same displacing resident model, no located parent on the device).
// v2 computes each distinct value once, with bit-identical arithmetic:
//
//   row classes   devices with equal (cached stage-group tokens, speed) share
//                 the cache-aware query_compute row (costs.py:70-94), hence
//                 aware(d) (costs.py:257), the full-batch compute and every
//                 shard compute (costs.py:404-405); instances with query prefix
//                 groups fall back to one row per device;
//   tail tasks    per (item, level): devices whose level-l chain cannot skip an
//                 op (no located parent edge on that device) and that share the
//                 displacing resident model run the identical affinity chain
//                 (costs.py:307-348); such a class is walked once, "special"
//                 devices (a located parent on the device, or any located edge
//                 under transfer overrides) walk their own chain.
//
// The distinct work of all IPB items of a CTA is pooled and spread over all
// CTA threads (qc entries, Neumaier sums, tail chains), so the few distinct
// values do not leave lanes idle.  Phases, separated by __syncthreads:
//   P0 device state per lane (residency, wait, switch, transfer, cached tokens,
//      keys), idle mask, per-level located-device masks;
//   P1 class representatives (first equal key), tail-task owners;
//   P2 class / task numbering, pool offsets (thread 0);
//   P3 qc rows (pooled);
//   P4 row sums (aware + shard sums) and tail chains (pooled);
//   P5 per-device assembly of S, tail, Psi(slot 0..bound-1), completion.

constexpr int V2_KT = 4;  // shard counts k <= V2_KT use pooled shard sums

struct V2View {
    // per item
    int* hdr;                 // [32]
    unsigned long long* u64;  // [4 + 2*LV]: elig, idle_mask, rep_mask, -, lvl_mask[LV], owner_mask[LV]
    double* dh;               // [4]: clock, -, -, -
    int* key_cs;              // [D]
    int* rep;                 // [D]
    int* rowc;                // [D]
    int* md;                  // [D] displacing resident model or -1
    int* res;                 // [D]
    int* rowdev;              // [D]
    double* free_;            // [D]
    double* sw;               // [D]
    double* tr;               // [D]
    double* rows;             // [D*Bmax]
    double* aware_c;          // [D]
    double* shard;            // [D*2*V2_KT]
    double* taskres;          // [LV*D]
    int* tlo;                 // [LV] bucket lo (relative)
    int* tcnt;                // [LV]
    int* tbase;               // [LV] pool base of the (item, level) tasks
    unsigned char* owner;     // [LV*D] owner device of (level, d)
    unsigned char* tslot;     // [LV*D] task slot of (level, d)
    unsigned char* towner;    // [LV*D] owner device of (level, task)
};

enum {
    H_LIVE, H_S, H_V, H_INST, H_Q0, H_NQ, H_M, H_R, H_GV, H_PV, H_FLAGS, H_NROWS, H_NIDLE,
    H_KB, H_KI, H_NKS, H_QCBASE, H_SUMBASE, H_SUMPER, H_QG, H_COUNT
};
constexpr int V2_HDR = 32;

__host__ __device__ inline size_t v2_item_bytes(int D, int Bmax, int LV) {
    size_t dbl = 4 + 3 * (size_t)D + (size_t)D * Bmax + D + (size_t)D * 2 * V2_KT + (size_t)LV * D;
    size_t u64 = 4 + 2 * (size_t)LV;
    size_t ints = V2_HDR + 6 * (size_t)D + 3 * (size_t)LV;
    size_t bytes = 3 * (size_t)LV * D;
    size_t total = dbl * 8 + u64 * 8 + ints * 4 + bytes;
    return (total + 15) & ~size_t(15);
}

__device__ inline V2View v2_view(unsigned char* base, int D, int Bmax, int LV) {
    V2View v;
    double* dp = reinterpret_cast<double*>(base);
    v.dh = dp; dp += 4;
    v.free_ = dp; dp += D;
    v.sw = dp; dp += D;
    v.tr = dp; dp += D;
    v.rows = dp; dp += (size_t)D * Bmax;
    v.aware_c = dp; dp += D;
    v.shard = dp; dp += (size_t)D * 2 * V2_KT;
    v.taskres = dp; dp += (size_t)LV * D;
    unsigned long long* up = reinterpret_cast<unsigned long long*>(dp);
    v.u64 = up; up += 4 + 2 * LV;
    int* ip = reinterpret_cast<int*>(up);
    v.hdr = ip; ip += V2_HDR;
    v.key_cs = ip; ip += D;
    v.rep = ip; ip += D;
    v.rowc = ip; ip += D;
    v.md = ip; ip += D;
    v.res = ip; ip += D;
    v.rowdev = ip; ip += D;
    v.tlo = ip; ip += LV;
    v.tcnt = ip; ip += LV;
    v.tbase = ip; ip += LV;
    unsigned char* bp = reinterpret_cast<unsigned char*>(ip);
    v.owner = bp; bp += (size_t)LV * D;
    v.tslot = bp; bp += (size_t)LV * D;
    v.towner = bp;
    return v;
}

__device__ __forceinline__ unsigned long long low_mask(int d) {
    return d >= 64 ? ~0ull : ((1ull << d) - 1ull);
}

// Shard range of shard i of k over nq queries (_even_split, costs.py:419-428)
__device__ __forceinline__ void shard_range(int nq, int k, int i, int* lo, int* hi) {
    const int base = nq / k, extra = nq % k;
    *lo = i * base + (i < extra ? i : extra);
    *hi = *lo + base + (i < extra ? 1 : 0);
}

template <int G, int NT>
__global__ void __launch_bounds__(NT) fate_score_v2_kernel(fate_bank b, fate_weights w,
                                                           fate_windows win, fate_derived der,
                                                           fate_state st, fate_work work,
                                                           fate_out out) {
    constexpr int IPB = NT / G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int pool_tot[3];  // qc, sum, tail totals
    const int D = b.n_devices, Bmax = b.max_queries, LV = win.levels;
    const int li = threadIdx.x / G, t = threadIdx.x % G;
    const long long item = (long long)blockIdx.x * IPB + li;
    const bool live = item < work.n_items;
    const size_t item_bytes = v2_item_bytes(D, Bmax, LV);
    V2View V = v2_view(smem_raw + item_bytes * li, D, Bmax, LV);
    const bool no_loc = w.ablation & FATE_NO_LOCALITY;
    const bool no_pre = w.ablation & FATE_NO_PREFIX;
    const bool no_same = w.ablation & FATE_NO_SAME_MODEL;
    const bool no_shard = w.ablation & FATE_NO_SHARD;
    const int H = w.eff_horizon;

    // ---- item constants (every lane) -------------------------------------------
    int s = 0, v = 0, inst = 0, q0 = 0, nq = 0, m = -1, R = 1, gv = -1, Pv = 0;
    uint64_t elig = 0;
    double clock = 0.0;
    bool cache_reuse = false;
    const int32_t* loc_row = nullptr;
    if (live) {
        s = work.scen[item];
        v = work.stage[item];
        inst = st.scen_inst[s];
        q0 = b.inst_query_off[inst];
        nq = b.inst_n_queries[inst];
        m = b.st_model[v];
        R = b.st_shard[v];
        gv = b.st_group[v];
        Pv = b.st_prompt[v];
        elig = b.st_elig[v];
        clock = st.scen_clock[s];
        cache_reuse = (b.st_flags[v] & FATE_STAGE_CACHE_REUSE) && gv != -1;
        loc_row = st.loc + st.scen_loc_off[s] - b.inst_stage_off[inst];
    }
    const long long dev_row0 = (long long)s * D;
    const int cap4 = st.kappa_cap * 4;

    // ---- init accumulators ---------------------------------------------------------
    for (int i = t; i < 4 + 2 * LV; i += G) V.u64[i] = 0ull;
    if (t == 0) V.hdr[H_QG] = 0;
    __syncthreads();

    // ---- P0: device state, masks ----------------------------------------------------
    const int d = t;
    const bool dev_live = live && d < D;
    const bool dev_ok = dev_live && ((elig >> d) & 1ull);
    if (live) {
        // query prefix groups present? (row dedup needs none)
        for (int q = t; q < nq; q += G)
            if (b.q_group[q0 + q] != -1) V.hdr[H_QG] = 1;
    }
    if (dev_live) {
        const int r = st.residency[dev_row0 + d];
        const double fr = st.dev_free[dev_row0 + d];
        V.res[d] = r;
        V.free_[d] = fr;
        V.md[d] = (r != -1 && r != m) ? r : -1;
        int cs = 0;
        if (cache_reuse)
            cs = cached_tokens(st.kappa + (dev_row0 + d) * cap4, st.kappa_n[dev_row0 + d], gv, m);
        V.key_cs[d] = cs;
        if (dev_ok) {
            V.sw[d] = (m < 0 || r == m) ? 0.0 : b.model_switch[m] * w.switch_x;
            double tr = 0.0;
            for (int e = b.par_ptr[v]; e < b.par_ptr[v + 1]; ++e) {
                const int L = loc_row[b.par_idx[e]];
                if (L < 0 || L == d) continue;
                tr += b.beta[(size_t)L * D + d] * der.edge_sigma[e];
            }
            V.tr[d] = tr * w.transfer_x;
            if (fr <= clock + 1e-12) atomicOr(&V.u64[1], 1ull << d);
        }
    }
    // located-device mask per level (tail chains may skip ops of these devices)
    if (live && H > 1 && !no_loc) {
        for (int l = 0; l < LV; ++l) {
            const long long lo = win.ptr[(long long)v * LV + l];
            const long long hi = win.ptr[(long long)v * LV + l + 1];
            unsigned long long mask = 0ull;
            for (long long i = lo + t; i < hi; i += G) {
                const int x = win.idx[i];
                for (int e = b.par_ptr[x]; e < b.par_ptr[x + 1]; ++e) {
                    const int p = b.par_idx[e];
                    if (p == v) continue;
                    const int L = loc_row[p];
                    if (L >= 0) mask |= 1ull << L;
                }
            }
            if (mask) atomicOr(&V.u64[4 + l], mask);
        }
    }
    __syncthreads();

    // ---- P1: class representatives, tail owners -----------------------------------
    const bool per_device_rows = live && V.hdr[H_QG] != 0;
    if (dev_ok) {
        int rp = d;
        if (!per_device_rows) {
            const int key = V.key_cs[d];
            const double sp = b.dev_speed[d];
            for (int e = 0; e < d; ++e) {
                if (((elig >> e) & 1ull) && V.key_cs[e] == key && b.dev_speed[e] == sp) {
                    rp = e;
                    break;
                }
            }
        }
        V.rep[d] = rp;
        if (rp == d) atomicOr(&V.u64[2], 1ull << d);
        for (int l = 0; l < LV; ++l) {
            const unsigned long long lm = V.u64[4 + l];
            const bool any_loc = lm != 0ull;
            const bool special = !no_loc && any_loc && (b.has_overrides || ((lm >> d) & 1ull));
            int ow = d;
            if (!special) {
                const int mk = V.md[d];
                for (int e = 0; e < d; ++e) {
                    if (!((elig >> e) & 1ull)) continue;
                    const bool sp_e = !no_loc && any_loc && (b.has_overrides || ((lm >> e) & 1ull));
                    if (!sp_e && V.md[e] == mk) {
                        ow = e;
                        break;
                    }
                }
            }
            V.owner[l * D + d] = (unsigned char)ow;
            if (ow == d) atomicOr(&V.u64[4 + LV + l], 1ull << d);
        }
    }
    __syncthreads();

    // ---- P2: numbering and pool offsets ------------------------------------------
    if (dev_ok) {
        const unsigned long long rm = V.u64[2];
        const int rp = V.rep[d];
        const int c = __popcll(rm & low_mask(rp));
        V.rowc[d] = c;
        if (rp == d) V.rowdev[c] = d;
        for (int l = 0; l < LV; ++l) {
            const unsigned long long om = V.u64[4 + LV + l];
            const int ow = V.owner[l * D + d];
            const int k = __popcll(om & low_mask(ow));
            V.tslot[l * D + d] = (unsigned char)k;
            if (ow == d) V.towner[l * D + k] = (unsigned char)d;
        }
    }
    if (threadIdx.x == 0) {
        int qc_tot = 0, sum_tot = 0, tail_tot = 0;
        unsigned char* base0 = smem_raw;
        for (int it = 0; it < IPB; ++it) {
            V2View I = v2_view(base0 + item_bytes * it, D, Bmax, LV);
            const long long gitem = (long long)blockIdx.x * IPB + it;
            const bool lv = gitem < work.n_items;
            int nrows = 0, n_idle = 0, kb = 0, ki = 0, per = 0, nqi = 0;
            if (lv) {
                const int vi = work.stage[gitem];
                const int si = work.scen[gitem];
                nqi = b.inst_n_queries[st.scen_inst[si]];
                nrows = __popcll(I.u64[2]);
                n_idle = __popcll(I.u64[1]);
                const int Ri = b.st_shard[vi];
                if (Ri > 1 && !no_shard) {
                    kb = Ri < 1 + n_idle ? Ri : 1 + n_idle;
                    ki = Ri < n_idle ? Ri : n_idle;
                }
                per = 1;
                if (kb >= 2 && kb <= V2_KT) per += kb;
                if (ki != kb && ki >= 2 && ki <= V2_KT) per += ki;
                for (int l = 0; l < LV; ++l) {
                    const long long lo = win.ptr[(long long)vi * LV + l];
                    const long long hi = win.ptr[(long long)vi * LV + l + 1];
                    const int cnt = (hi > lo && H > 1) ? __popcll(I.u64[4 + LV + l]) : 0;
                    I.tcnt[l] = cnt;
                    I.tbase[l] = tail_tot;
                    tail_tot += cnt;
                }
            }
            I.hdr[H_LIVE] = lv;
            I.hdr[H_NQ] = nqi;
            I.hdr[H_NROWS] = nrows;
            I.hdr[H_NIDLE] = n_idle;
            I.hdr[H_KB] = kb;
            I.hdr[H_KI] = ki;
            I.hdr[H_SUMPER] = per;
            I.hdr[H_QCBASE] = qc_tot;
            I.hdr[H_SUMBASE] = sum_tot;
            qc_tot += nrows * nqi;
            sum_tot += nrows * per;
        }
        pool_tot[0] = qc_tot;
        pool_tot[1] = sum_tot;
        pool_tot[2] = tail_tot;
    }
    __syncthreads();

    // ---- P3: pooled query_compute rows --------------------------------------------
    {
        const int total = pool_tot[0];
        for (int p = threadIdx.x; p < total; p += NT) {
            int it = 0;
            while (it + 1 < IPB) {
                V2View N = v2_view(smem_raw + item_bytes * (it + 1), D, Bmax, LV);
                if (N.hdr[H_QCBASE] > p || !N.hdr[H_LIVE]) break;
                ++it;
            }
            V2View I = v2_view(smem_raw + item_bytes * it, D, Bmax, LV);
            const long long gitem = (long long)blockIdx.x * IPB + it;
            const int local = p - I.hdr[H_QCBASE];
            const int nqi = I.hdr[H_NQ];
            const int c = local / nqi, q = local - c * nqi;
            const int dv = I.rowdev[c];
            const int vi = work.stage[gitem], si = work.scen[gitem];
            const int insti = st.scen_inst[si];
            const int qq = b.inst_query_off[insti] + q;
            const int mi = b.st_model[vi], ri = b.st_role[vi], gvi = b.st_group[vi];
            const double pcoef = mi >= 0 ? b.model_prefill[mi] : 1.0;
            const double dcoef = mi >= 0 ? b.model_decode[mi] : 0.0;
            const double decode = (double)b.st_out[vi] * dcoef * b.role_decode[ri];
            long long sp = b.st_prompt[vi], qp = b.q_prompt[qq];
            const long long drow = (long long)si * D + dv;
            if ((b.st_flags[vi] & FATE_STAGE_CACHE_REUSE) && gvi != -1) {
                const long long cc = I.key_cs[dv];
                sp = sp - cc > 0 ? sp - cc : 0;
            }
            const int qg = b.q_group[qq];
            if (qg != -1) {
                const long long cc = cached_tokens(st.kappa + drow * cap4, st.kappa_n[drow], qg, mi);
                qp = qp - cc > 0 ? qp - cc : 0;
            }
            I.rows[c * Bmax + q] = qc_value(sp, qp, pcoef, b.role_prefill[ri], decode,
                                            b.role_cplx[ri], b.dev_speed[dv]);
        }
    }
    __syncthreads();

    // ---- P4: pooled row sums and tail chains ----------------------------------------
    {
        const int n_sum = pool_tot[1];
        const int total = n_sum + pool_tot[2];
        for (int p = threadIdx.x; p < total; p += NT) {
            if (p < n_sum) {
                int it = 0;
                while (it + 1 < IPB) {
                    V2View N = v2_view(smem_raw + item_bytes * (it + 1), D, Bmax, LV);
                    if (N.hdr[H_SUMBASE] > p || !N.hdr[H_LIVE]) break;
                    ++it;
                }
                V2View I = v2_view(smem_raw + item_bytes * it, D, Bmax, LV);
                const int local = p - I.hdr[H_SUMBASE];
                const int per = I.hdr[H_SUMPER];
                const int c = local / per;
                int j = local - c * per;
                const int nqi = I.hdr[H_NQ];
                const double* row = I.rows + c * Bmax;
                PySum acc;
                if (j == 0) {
                    for (int q = 0; q < nqi; ++q) acc.add(row[q]);
                    I.aware_c[c] = acc.result();
                } else {
                    j -= 1;
                    const int kb = I.hdr[H_KB], ki = I.hdr[H_KI];
                    int kslot = 0, k = kb;
                    if (!(kb >= 2 && kb <= V2_KT)) { kslot = 1; k = ki; }
                    else if (j >= kb) { j -= kb; kslot = 1; k = ki; }
                    int lo, hi;
                    shard_range(nqi, k, j, &lo, &hi);
                    for (int q = lo; q < hi; ++q) acc.add(row[q]);
                    I.shard[(c * 2 + kslot) * V2_KT + j] = acc.result();
                }
            } else {
                // tail chain task: find (item, level, slot)
                const int tp = p - n_sum;
                int it = 0, l = 0;
                for (it = 0; it < IPB; ++it) {
                    V2View I = v2_view(smem_raw + item_bytes * it, D, Bmax, LV);
                    if (!I.hdr[H_LIVE]) continue;
                    bool found = false;
                    for (l = 0; l < LV; ++l) {
                        if (tp >= I.tbase[l] && tp < I.tbase[l] + I.tcnt[l]) { found = true; break; }
                    }
                    if (found) break;
                }
                V2View I = v2_view(smem_raw + item_bytes * it, D, Bmax, LV);
                const int k = tp - I.tbase[l];
                const int od = I.towner[l * D + k];
                const long long gitem = (long long)blockIdx.x * IPB + it;
                const int vi = work.stage[gitem], si = work.scen[gitem];
                const int insti = st.scen_inst[si];
                const int32_t* lrow = st.loc + st.scen_loc_off[si] - b.inst_stage_off[insti];
                const int mv = b.st_model[vi], gvv = b.st_group[vi], Pvv = b.st_prompt[vi];
                const int res_d = I.res[od];
                const bool displaces = res_d != -1 && res_d != mv;
                const bool walk_loc = !no_loc && I.u64[4 + l] != 0ull;
                const long long lo = win.ptr[(long long)vi * LV + l];
                const long long hi = win.ptr[(long long)vi * LV + l + 1];
                double aff = 0.0;
                for (long long i = lo; i < hi; ++i) {
                    const int x = win.idx[i];
                    const int mx = b.st_model[x];
                    if (!no_same && mx != -1) {
                        if (mx == mv) {
                            aff += w.lambda_s * b.model_switch[mx] * w.switch_x * w.state_scale;
                        } else if (displaces && mx == res_d) {
                            aff -= w.lambda_s * b.model_switch[mx] * w.switch_x * w.state_scale;
                        }
                    }
                    const int gx = b.st_group[x];
                    if (!no_pre && gx != -1 && gx == gvv) {
                        const int Px = b.st_prompt[x];
                        const int shared = Pvv < Px ? Pvv : Px;
                        aff += w.lambda_p * w.kappa_prefix * (double)shared / 1000.0 * w.prefix_x *
                               w.prefix_scale;
                    }
                    if (walk_loc) {
                        for (int e = b.par_ptr[x]; e < b.par_ptr[x + 1]; ++e) {
                            const int pp = b.par_idx[e];
                            if (pp == vi) continue;
                            const int Lp = lrow[pp];
                            if (Lp < 0 || Lp == od) continue;
                            if (b.has_overrides) {
                                aff -= w.lambda_tr * b.beta[(size_t)Lp * D + od] *
                                       der.edge_sigma[e] * w.transfer_x * w.locality_scale;
                            } else {
                                aff -= der.edge_term[e];
                            }
                        }
                    }
                }
                I.taskres[l * D + k] = aff;
            }
        }
    }
    __syncthreads();

    // ---- P5: per-device assembly ------------------------------------------------------
    if (!dev_live) return;
    const int n_elig = __popcll(elig);
    const int bound = no_shard ? 1 : (R < n_elig ? R : n_elig);
    const long long orow = item * D + d;
    double* psi = out.psi + work.psi_off[item];
    if (!dev_ok) {
        const double qnan = __longlong_as_double(0x7ff8000000000000LL);
        for (int k = 0; k < bound; ++k) psi[(long long)k * D + d] = qnan;
        if (out.sched) out.sched[orow] = qnan;
        if (out.tail) out.tail[orow] = qnan;
        if (out.completion) out.completion[orow] = qnan;
        return;
    }
    const double free_d = V.free_[d];
    const double wait = py_max0(free_d - clock);
    const double sw = V.sw[d];
    const double tr = V.tr[d];
    const int c_d = V.rowc[d];
    const double here = V.aware_c[c_d];

    // colo (costs.py:160-165)
    const int pa0 = b.par_ptr[v], pa1 = b.par_ptr[v + 1];
    double colo = 0.0;
    if (pa1 > pa0) {
        int hit = 0;
        for (int e = pa0; e < pa1; ++e) hit += loc_row[b.par_idx[e]] == d;
        colo = (double)hit / (double)(pa1 - pa0);
    }
    // prefix_overlap_thousands (costs.py:127-145), integer-exact
    long long tokens = 0;
    if (cache_reuse) {
        const long long c = V.key_cs[d];
        tokens += c < Pv ? c : Pv;
    }
    if (V.hdr[H_QG]) {
        const int32_t* kap = st.kappa + (dev_row0 + d) * cap4;
        const int kn = st.kappa_n[dev_row0 + d];
        for (int q = 0; q < nq; ++q) {
            const int qg = b.q_group[q0 + q];
            if (qg == -1) continue;
            const long long c = cached_tokens(kap, kn, qg, m);
            const long long qp = b.q_prompt[q0 + q];
            tokens += c < qp ? c : qp;
        }
    }
    const double prefix = w.kappa_prefix * ((double)tokens / 1000.0) * w.prefix_x;

    // _parallel_benefit (costs.py:181-201)
    const double full_total = sw + tr + here;
    double parallel = 0.0;
    if (R > 1 && !no_shard) {
        const unsigned long long idle_m = V.u64[1];
        const bool self_idle = (idle_m >> d) & 1ull;
        const int n_idle = V.hdr[H_NIDLE];
        const int others = n_idle - (self_idle ? 1 : 0);
        const int k = R < 1 + others ? R : 1 + others;
        if (k > 1) {
            const int kb = V.hdr[H_KB];
            const bool pooled = k <= V2_KT;
            const int kslot = (k == kb && kb >= 2 && kb <= V2_KT) ? 0 : 1;
            unsigned long long rest = idle_m & ~(1ull << d);
            double worst = 0.0;
            for (int i = 0; i < k; ++i) {
                int dev = d;
                if (i > 0) {
                    dev = __ffsll((long long)rest) - 1;
                    rest &= rest - 1;
                }
                const int cd = V.rowc[dev];
                double ssum;
                if (pooled) {
                    ssum = V.shard[(cd * 2 + kslot) * V2_KT + i];
                } else {
                    int lo, hi;
                    shard_range(nq, k, i, &lo, &hi);
                    PySum acc;
                    for (int q = lo; q < hi; ++q) acc.add(V.rows[cd * Bmax + q]);
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
                     - w.lambda_tr * tr_s * w.locality_scale + w.lambda_c * colo_s * w.locality_scale
                     + w.lambda_p * prefix_s * w.prefix_scale + w.lambda_r * par_s;

    // tail_value (costs.py:281-352): level sums from the pooled chains
    double tail = 0.0;
    if (H > 1) {
        for (int l = 1; l < H; ++l) {
            const long long lo = win.ptr[(long long)v * LV + (l - 1)];
            const long long hi = win.ptr[(long long)v * LV + l];
            if (hi == lo) continue;
            const double aff = V.taskres[(l - 1) * D + V.tslot[(l - 1) * D + d]];
            const double dem = der.demand[(long long)v * LV + (l - 1)];
            tail += w.gamma_pow[l] * (aff / (double)(hi - lo) + w.demand_coeff * dem);
        }
    }

    if (out.sched) out.sched[orow] = S;
    if (out.tail) out.tail[orow] = tail;
    if (out.completion) out.completion[orow] = wait + full_total;
    psi[d] = S + tail;

    // _marginal_shard_score (costs.py:249-279)
    if (bound > 1) {
        double bb = V.aware_c[0];
        for (int c = 1; c < V.hdr[H_NROWS]; ++c) bb = V.aware_c[c] < bb ? V.aware_c[c] : bb;
        const double hi_v = here > bb ? here : bb;
        const double overhead = w.shard_overhead_frac * bb;
        const double tr_m = no_loc ? 0.0 : tr;
        const double split = no_loc ? 0.0 : der.split_penalty[v];
        for (int k = 1; k < bound; ++k) {
            const double reduction = bb / (double)k - hi_v / (double)(k + 1);
            psi[(long long)k * D + d] = w.lambda_r * (reduction - overhead) - w.lambda_q * wait -
                                        w.lambda_s * sw * w.state_scale -
                                        w.lambda_tr * (tr_m + split) * w.locality_scale;
        }
    }
}
