// fate_score_v3.cuh -- item-local, class-deduplicated scoring kernel with a
// static tail table and compact per-level op lists.
//
// Included by fate_kernels.cu (inside its anonymous namespace).
//
// Item = (scenario, stage v) owned by a group of G threads (G = 32 for D <= 32,
// 64 otherwise), thread d <-> device d.  The group synchronises with
// __syncwarp (G = 32) or a named barrier (G = 64); items never wait for each
// other.  Per item:
//
//   P0  lane d: device row (residency, free time, cached stage-group tokens),
//       wait, switch, transfer and colo counts (costs.py:107-125, 157-165).
//   P1  row classes: devices with equal (cached tokens, speed) share the
//       cache-aware query_compute row bit for bit (costs.py:70-94) -- one
//       representative per class (instances with query prefix groups: one
//       row per device).
//   P2  the group computes each class row once, then the Neumaier sums the
//       reference takes over it: full batch (aware, costs.py:257 / :404) and
//       the shard ranges of the <= 2 shard counts the item uses (:404-405).
//   P3  tail (costs.py:281-352), level by level:
//         * no located parent edge in the level (always in frontier mode, or
//           no_locality): the affinity chain depends only on (v, l, the
//           device's displacing resident model), so it is read from the static
//           table tail_static[v][l][class] built by the prologue;
//         * otherwise the group compacts the level into an ordered op list
//           (signed values: a - b == a + (-b) exactly in IEEE 754) and every
//           lane walks it with its own skip / displacement conditions.
//   P4  lane d assembles colo, prefix overlap, parallel benefit, S, tail,
//       Psi(slot 0..bound-1) and completion.

constexpr int V3_KT = 4;          // shard counts k <= V3_KT use the group's shard sums
constexpr int V3_COND_ALWAYS = -1;  // op applies to every lane
// cond <= -2: displacement op of model (-2 - cond); applies iff lane's class == model
// 0 <= cond < 64: locality op of located device cond; applies iff lane != cond
// cond >= 1000: locality op under transfer overrides; value holds sigma,
//               lane computes lambda_tr*beta[L][d]*sigma*transfer_x*locality_scale

struct V3View {
    double* rows;       // [D*Bmax]
    double* aware_c;    // [D]
    double* shard;      // [D*2*V3_KT]
    double* sw;         // [D]
    double* tr;         // [D]
    double* opval;      // [ops_cap]
    int* opcond;        // [ops_cap]
    int* key;           // [D]
    int* rowc;          // [D]
    int* rowdev;        // [D]
    int* scratch;       // [G + 8]
    unsigned long long* masks;  // [4]: idle, rep, qgroups, -
};

__host__ __device__ inline size_t v3_item_bytes(int D, int Bmax, int G, int ops_cap) {
    size_t dbl = (size_t)D * Bmax + D + (size_t)D * 2 * V3_KT + 2 * (size_t)D + ops_cap;
    size_t u64 = 4;
    size_t ints = (size_t)ops_cap + 3 * (size_t)D + G + 8;
    return ((dbl + u64) * 8 + ints * 4 + 15) & ~size_t(15);
}

__device__ inline V3View v3_view(unsigned char* base, int D, int Bmax, int G, int ops_cap) {
    V3View v;
    double* dp = reinterpret_cast<double*>(base);
    v.rows = dp; dp += (size_t)D * Bmax;
    v.aware_c = dp; dp += D;
    v.shard = dp; dp += (size_t)D * 2 * V3_KT;
    v.sw = dp; dp += D;
    v.tr = dp; dp += D;
    v.opval = dp; dp += ops_cap;
    unsigned long long* up = reinterpret_cast<unsigned long long*>(dp);
    v.masks = up; up += 4;
    int* ip = reinterpret_cast<int*>(up);
    v.opcond = ip; ip += ops_cap;
    v.key = ip; ip += D;
    v.rowc = ip; ip += D;
    v.rowdev = ip; ip += D;
    v.scratch = ip;
    return v;
}

template <int G>
__device__ __forceinline__ void group_sync(int li) {
    if (G == 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + li), "r"(G) : "memory");
    }
}

// 64-bit ballot over the item group (G = 32: one warp; G = 64: two warps
// through shared scratch).  Every lane of the group receives the mask.
template <int G>
__device__ __forceinline__ unsigned long long group_ballot(bool pred, int t, int li,
                                                           unsigned long long* slot) {
    const unsigned int b = __ballot_sync(0xffffffffu, pred);
    if (G == 32) return (unsigned long long)b;
    if ((t & 31) == 0) reinterpret_cast<unsigned int*>(slot)[t >> 5] = b;
    group_sync<G>(li);
    const unsigned long long m = *reinterpret_cast<volatile unsigned long long*>(slot);
    group_sync<G>(li);
    return m;
}

// Exclusive prefix sum of `val` over the group; returns the exclusive prefix,
// *total gets the group sum.
template <int G>
__device__ __forceinline__ int group_scan(int val, int t, int li, int* scratch, int* total) {
    int x = val;
    const int lane = t & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (G == 32) {
        *total = __shfl_sync(0xffffffffu, x, 31);
        return x - val;
    }
    if (lane == 31) scratch[t >> 5] = x;
    group_sync<G>(li);
    const int w0 = scratch[0], w1 = scratch[1];
    group_sync<G>(li);
    *total = w0 + w1;
    return x - val + ((t >> 5) ? w0 : 0);
}

// Prologue: static tail chains (no locality op applied) per (stage, level,
// displacement class): class 0 = not displacing, class 1+m = displaces with
// resident model m (costs.py:307-331).
__global__ void fate_prepare_tail_static_kernel(fate_bank b, fate_weights w, fate_windows win,
                                                double* tail_static) {
    const int M1 = b.n_models + 1;
    const int LV = win.levels;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)b.n_stages * LV * M1) return;
    const int c = (int)(t % M1);
    const long long vl = t / M1;
    const int v = (int)(vl / LV);
    const bool no_same = w.ablation & FATE_NO_SAME_MODEL;
    const bool no_pre = w.ablation & FATE_NO_PREFIX;
    const int mv = b.st_model[v], gv = b.st_group[v], Pv = b.st_prompt[v];
    const int res = c - 1;  // -1: no displacement
    double aff = 0.0;
    for (long long i = win.ptr[vl]; i < win.ptr[vl + 1]; ++i) {
        const int x = win.idx[i];
        const int mx = b.st_model[x];
        if (!no_same && mx != -1) {
            if (mx == mv) {
                aff += w.lambda_s * b.model_switch[mx] * w.switch_x * w.state_scale;
            } else if (res != -1 && mx == res) {
                aff -= w.lambda_s * b.model_switch[mx] * w.switch_x * w.state_scale;
            }
        }
        const int gx = b.st_group[x];
        if (!no_pre && gx != -1 && gx == gv) {
            const int Px = b.st_prompt[x];
            const int shared = Pv < Px ? Pv : Px;
            aff += w.lambda_p * w.kappa_prefix * (double)shared / 1000.0 * w.prefix_x *
                   w.prefix_scale;
        }
    }
    tail_static[t] = aff;
}

// Prologue: full tail per (stage, displacement class) from the static level
// chains and the demand table, accumulated level by level in the reference
// order (costs.py:296-351).
__global__ void fate_prepare_tail_sum_kernel(fate_bank b, fate_weights w, fate_windows win,
                                             fate_derived der) {
    const int M1 = b.n_models + 1;
    const int LV = win.levels;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)b.n_stages * M1) return;
    const int c = (int)(t % M1);
    const long long v = t / M1;
    double total = 0.0;
    for (int l = 0; l < LV; ++l) {
        const long long vl = v * LV + l;
        const long long n = win.ptr[vl + 1] - win.ptr[vl];
        if (n == 0) continue;
        const double aff = der.tail_static[vl * M1 + c];
        total += w.gamma_pow[l + 1] * (aff / (double)n + w.demand_coeff * der.demand[vl]);
    }
    der.tail_sum[t] = total;
}

template <int G>
__global__ void __launch_bounds__(128) fate_score_v3_kernel(fate_bank b, fate_weights w,
                                                            fate_windows win, fate_derived der,
                                                                                                                        fate_state st, fate_work work,
                                                            fate_out out) {
    constexpr int IPB = 128 / G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int D = b.n_devices, Bmax = b.max_queries, LV = win.levels, OPS = win.max_level_ops;
    const int li = threadIdx.x / G, t = threadIdx.x % G;
    const long long item = (long long)blockIdx.x * IPB + li;
    if (item >= work.n_items) return;  // whole groups exit together
    V3View V = v3_view(smem_raw + v3_item_bytes(D, Bmax, G, OPS) * li, D, Bmax, G, OPS);
    const bool no_loc = w.ablation & FATE_NO_LOCALITY;
    const bool no_pre = w.ablation & FATE_NO_PREFIX;
    const bool no_same = w.ablation & FATE_NO_SAME_MODEL;
    const bool no_shard = w.ablation & FATE_NO_SHARD;
    const int H = w.eff_horizon;
    const int M1 = b.n_models + 1;

    const int s = work.scen[item];
    const int v = work.stage[item];
    const int inst = st.scen_inst[s];
    const int q0 = b.inst_query_off[inst];
    const int nq = b.inst_n_queries[inst];
    const int m = b.st_model[v];
    const int R = b.st_shard[v];
    const int gv = b.st_group[v];
    const int Pv = b.st_prompt[v];
    const uint64_t elig = b.st_elig[v];
    const double clock = st.scen_clock[s];
    const bool cache_reuse = (b.st_flags[v] & FATE_STAGE_CACHE_REUSE) && gv != -1;
    const int32_t* loc_row = st.loc + st.scen_loc_off[s] - b.inst_stage_off[inst];
    const long long dev_row0 = (long long)s * D;
    const int cap4 = st.kappa_cap * 4;
    const int pa0 = b.par_ptr[v], pa1 = b.par_ptr[v + 1];

    // ---- P0: device row ------------------------------------------------------------
    const int d = t;
    const bool dev_live = d < D;
    const bool dev_ok = dev_live && ((elig >> d) & 1ull);
    int res = -1, cs = 0, hit = 0;
    double fr = 0.0;
    if (dev_live) {
        res = st.residency[dev_row0 + d];
        fr = st.dev_free[dev_row0 + d];
        if (cache_reuse)
            cs = cached_tokens(st.kappa + (dev_row0 + d) * cap4, st.kappa_n[dev_row0 + d], gv, m);
        V.key[d] = cs;
    }
    if (dev_ok) {
        V.sw[d] = (m < 0 || res == m) ? 0.0 : b.model_switch[m] * w.switch_x;
        double tr = 0.0;
        for (int e = pa0; e < pa1; ++e) {
            const int L = loc_row[b.par_idx[e]];
            hit += L == d;
            if (L < 0 || L == d) continue;
            tr += b.beta[(size_t)L * D + d] * der.edge_sigma[e];
        }
        V.tr[d] = tr * w.transfer_x;
    }
    bool qg_any = false;
    for (int q = t; q < nq; q += G) qg_any |= b.q_group[q0 + q] != -1;
    const bool per_device_rows = group_ballot<G>(qg_any, t, li, &V.masks[2]) != 0ull;
    const unsigned long long idle_m =
        group_ballot<G>(dev_ok && fr <= clock + 1e-12, t, li, &V.masks[0]);
    group_sync<G>(li);

    // ---- P1: row classes ----------------------------------------------------------------
    int rp = d;
    if (dev_ok && !per_device_rows) {
        const double sp = b.dev_speed[d];
        for (int e = 0; e < d; ++e) {
            if (((elig >> e) & 1ull) && V.key[e] == cs && b.dev_speed[e] == sp) {
                rp = e;
                break;
            }
        }
    }
    const unsigned long long rep_m = group_ballot<G>(dev_ok && rp == d, t, li, &V.masks[1]);
    const int n_rows = __popcll(rep_m);
    const int c_d = __popcll(rep_m & low_mask(rp));
    if (dev_ok && rp == d) V.rowdev[c_d] = d;
    if (dev_ok) V.rowc[d] = c_d;
    group_sync<G>(li);

    // ---- P2: class rows and their Neumaier sums ------------------------------------------
    {
        const int ri = b.st_role[v];
        const double pcoef = m >= 0 ? b.model_prefill[m] : 1.0;
        const double dcoef = m >= 0 ? b.model_decode[m] : 0.0;
        const double decode = (double)b.st_out[v] * dcoef * b.role_decode[ri];
        const double pscale = b.role_prefill[ri], cplx = b.role_cplx[ri];
        for (int p = t; p < n_rows * nq; p += G) {
            const int c = p / nq, q = p - c * nq;
            const int dv = V.rowdev[c];
            long long sp = Pv, qp = b.q_prompt[q0 + q];
            if (cache_reuse) {
                const long long cc = V.key[dv];
                sp = sp - cc > 0 ? sp - cc : 0;
            }
            const int qg = b.q_group[q0 + q];
            if (qg != -1) {
                const long long drow = dev_row0 + dv;
                const long long cc = cached_tokens(st.kappa + drow * cap4, st.kappa_n[drow], qg, m);
                qp = qp - cc > 0 ? qp - cc : 0;
            }
            V.rows[c * Bmax + q] = qc_value(sp, qp, pcoef, pscale, decode, cplx, b.dev_speed[dv]);
        }
    }
    const int n_idle = __popcll(idle_m);
    int kb = 0, ki = 0;
    if (R > 1 && !no_shard) {
        kb = R < 1 + n_idle ? R : 1 + n_idle;
        ki = R < n_idle ? R : n_idle;
    }
    const bool kb_ok = kb >= 2 && kb <= V3_KT;
    const bool ki_ok = ki != kb && ki >= 2 && ki <= V3_KT;
    const int per = 1 + (kb_ok ? kb : 0) + (ki_ok ? ki : 0);
    group_sync<G>(li);
    for (int p = t; p < n_rows * per; p += G) {
        const int c = p / per;
        int j = p - c * per;
        const double* row = V.rows + c * Bmax;
        PySum acc;
        if (j == 0) {
            for (int q = 0; q < nq; ++q) acc.add(row[q]);
            V.aware_c[c] = acc.result();
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
            V.shard[(c * 2 + kslot) * V3_KT + j] = acc.result();
        }
    }
    group_sync<G>(li);

    // ---- P3: tail ----------------------------------------------------------------------
    double tail = 0.0;
    const int mdc = (dev_live && res != -1 && res != m && res < b.n_models) ? 1 + res : 0;
    if (H > 1) {
        for (int l = 0; l < LV; ++l) {
            const long long lo = win.ptr[(long long)v * LV + l];
            const long long hi = win.ptr[(long long)v * LV + l + 1];
            if (hi == lo) continue;
            const int n_b = (int)(hi - lo);
            // count located parent edges of this lane's bucket items
            int located = 0;
            if (!no_loc) {
                for (int j = t; j < n_b; j += G) {
                    const int x = win.idx[lo + j];
                    for (int e = b.par_ptr[x]; e < b.par_ptr[x + 1]; ++e) {
                        const int pp = b.par_idx[e];
                        if (pp != v && loc_row[pp] >= 0) ++located;
                    }
                }
            }
            const bool walk = group_ballot<G>(located > 0, t, li, &V.masks[3]) != 0ull;
            double aff;
            if (!walk) {
                aff = der.tail_static[((long long)v * LV + l) * M1 + mdc];
            } else {
                // compact ordered op list, G bucket items per round
                int base = 0;
                for (int j0 = 0; j0 < n_b; j0 += G) {
                    const int j = j0 + t;
                    int x = -1, mx = -1, cnt = 0;
                    bool same_op = false, disp_op = false, pre_op = false;
                    if (j < n_b) {
                        x = win.idx[lo + j];
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
                            if (pp != v && loc_row[pp] >= 0) ++cnt;
                        }
                    }
                    int total;
                    int pos = base + group_scan<G>(cnt, t, li, V.scratch, &total);
                    if (j < n_b) {
                        if (same_op || disp_op) {
                            const double bonus =
                                w.lambda_s * b.model_switch[mx] * w.switch_x * w.state_scale;
                            V.opval[pos] = same_op ? bonus : -bonus;
                            V.opcond[pos] = same_op ? V3_COND_ALWAYS : -2 - mx;
                            ++pos;
                        }
                        if (pre_op) {
                            const int Px = b.st_prompt[x];
                            const int shared = Pv < Px ? Pv : Px;
                            V.opval[pos] = w.lambda_p * w.kappa_prefix * (double)shared / 1000.0 *
                                           w.prefix_x * w.prefix_scale;
                            V.opcond[pos] = V3_COND_ALWAYS;
                            ++pos;
                        }
                        for (int e = b.par_ptr[x]; e < b.par_ptr[x + 1]; ++e) {
                            const int pp = b.par_idx[e];
                            if (pp == v) continue;
                            const int L = loc_row[pp];
                            if (L < 0) continue;
                            if (b.has_overrides) {
                                V.opval[pos] = der.edge_sigma[e];
                                V.opcond[pos] = 1000 + L;
                            } else {
                                V.opval[pos] = -der.edge_term[e];
                                V.opcond[pos] = L;
                            }
                            ++pos;
                        }
                    }
                    base += total;
                }
                group_sync<G>(li);
                aff = 0.0;
                const int dm = mdc - 1;  // displacing model or -1
                for (int o = 0; o < base; ++o) {
                    const int cond = V.opcond[o];
                    const double val = V.opval[o];
                    if (cond == V3_COND_ALWAYS) {
                        aff += val;
                    } else if (cond <= -2) {
                        if (-2 - cond == dm) aff += val;
                    } else if (cond < 1000) {
                        if (cond != d) aff += val;
                    } else {
                        const int L = cond - 1000;
                        if (L != d)
                            aff -= w.lambda_tr * b.beta[(size_t)L * D + d] * val * w.transfer_x *
                                   w.locality_scale;
                    }
                }
                group_sync<G>(li);  // op buffer reused by the next level
            }
            const double dem = der.demand[(long long)v * LV + l];
            tail += w.gamma_pow[l + 1] * (aff / (double)n_b + w.demand_coeff * dem);
        }
    }

    // ---- P4: per-device assembly ----------------------------------------------------------
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
    const double wait = py_max0(fr - clock);
    const double sw = V.sw[d];
    const double tr = V.tr[d];
    const double here = V.aware_c[c_d];
    const double colo = pa1 > pa0 ? (double)hit / (double)(pa1 - pa0) : 0.0;

    // prefix_overlap_thousands (costs.py:127-145), integer-exact
    long long tokens = 0;
    if (cache_reuse) tokens += cs < Pv ? cs : Pv;
    if (per_device_rows) {
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
        const bool self_idle = (idle_m >> d) & 1ull;
        const int others = n_idle - (self_idle ? 1 : 0);
        const int k = R < 1 + others ? R : 1 + others;
        if (k > 1) {
            const int kslot = (k == kb && kb_ok) ? 0 : 1;
            const bool pooled = kslot == 0 || (k == ki && ki_ok);
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
                    ssum = V.shard[(cd * 2 + kslot) * V3_KT + i];
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

    if (out.sched) out.sched[orow] = S;
    if (out.tail) out.tail[orow] = tail;
    if (out.completion) out.completion[orow] = wait + full_total;
    psi[d] = S + tail;

    // _marginal_shard_score (costs.py:249-279)
    if (bound > 1) {
        double bb = V.aware_c[0];
        for (int c = 1; c < n_rows; ++c) bb = V.aware_c[c] < bb ? V.aware_c[c] : bb;
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
