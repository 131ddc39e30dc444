// fate_kernels.cu -- B200 (sm_100a) FATE candidate scorer + its C ABI.
//
// Replaces the reference's per-candidate Python scorer
//   wfsched.planner.build_problem -> CostModel.plan_score
//   (/root/reference/pkg/src/wfsched/planner.py:75-98, costs.py:70-416)
// with one launch that scores every (scenario, frontier stage, slot, device)
// candidate of a batch.  See DESIGN.md for the layout and roofline.
//
// Exactness contract: every Psi bit equals CPython 3.12 running the
// reference.  IEEE fp64 only, the reference's association order, no FMA
// contraction (this TU is compiled with --fmad=false; the build checks the
// PTX has no fma.rn.f64), CPython's Neumaier builtin sum() reproduced where
// the reference sums floats (costs.py:100, :104, :257, :404-405), plain
// sequential += where the reference loops.  Parallelism is used only across
// candidates, for gathers, and for order-free reductions (min/max/counts).
//
// Work decomposition (v1): one "item" = (scenario, stage v) owns TPI threads
// (TPI = D rounded up to a warp), one thread per device d.  Items are packed
// IPB per CTA.  Per item:
//   A. all TPI threads fill the cache-aware query_compute table qc[d][q]
//      in shared memory (costs.py:70-94);
//   B. thread d: aware(d) = Neumaier sum of its row (= full-batch compute,
//      costs.py:257 and :404), switch(d), transfer(d) (costs.py:107-125),
//      idle flag (costs.py:190);
//   C. one thread: base_best = min over eligible aware (costs.py:259) and the
//      sorted idle-device list (costs.py:187-191);
//   D. thread d: wait, colo, prefix overlap, parallel benefit (using other
//      devices' qc rows for the split shards), S, tail over the horizon window,
//      Psi(slot 0), Psi(slot k>=1), completion.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fate.h"
#include "fate_internal.h"

namespace {

thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_status(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
        return static_cast<int>(e);
    }
    return 0;
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------

// CPython 3.12 builtin sum() over floats (Python/bltinmodule.c): the start
// value is int 0, so the first term enters as 0 + x; Neumaier compensation
// afterwards; the compensation is added only when nonzero and finite.
struct PySum {
    double s, c;
    int n;
    __device__ __forceinline__ PySum() : s(0.0), c(0.0), n(0) {}
    __device__ __forceinline__ void add(double x) {
        if (n == 0) {
            s = 0.0 + x;
        } else {
            double t = s + x;
            if (fabs(s) >= fabs(x)) c += (s - t) + x;
            else c += (x - t) + s;
            s = t;
        }
        ++n;
    }
    __device__ __forceinline__ double result() const {
        if (n == 0) return 0.0;
        return (c != 0.0 && isfinite(c)) ? s + c : s;
    }
};

__device__ __forceinline__ double py_max0(double x) { return x > 0.0 ? x : 0.0; }

__device__ __forceinline__ unsigned long long low_mask(int d) {
    return d >= 64 ? ~0ull : ((1ull << d) - 1ull);
}

// Shard i of k over nq queries (_even_split, costs.py:419-428): contiguous,
// sizes nq/k + (i < nq%k)
__device__ __forceinline__ void shard_range(int nq, int k, int i, int* lo, int* hi) {
    const int base = nq / k, extra = nq % k;
    *lo = i * base + (i < extra ? i : extra);
    *hi = *lo + base + (i < extra ? 1 : 0);
}

// state.cached_tokens (state.py:110-123): group -1 = None, model -1 = None
__device__ __forceinline__ int cached_tokens(const int32_t* __restrict__ kap, int n, int group,
                                             int model) {
    if (group == -1) return 0;
    for (int k = 0; k < n; ++k) {
        const int4 e = reinterpret_cast<const int4*>(kap)[k];
        if (e.x == group) return (model != -1 && e.z != model) ? 0 : e.y;
    }
    return 0;
}

// query_compute numerator/denominator order (costs.py:92-94)
__device__ __forceinline__ double qc_value(long long stage_part, long long query_part,
                                           double pcoef, double pscale, double decode,
                                           double cplx, double speed) {
    double prefill = (double)(stage_part + query_part) / 1000.0 * pcoef * pscale;
    const double x = (prefill + decode) * cplx;
    return speed == 1.0 ? x : x / speed;  // x / 1.0 == x exactly
}

struct ItemSmem {
    double* qc;       // [D * Bmax]
    double* aware;    // [D]
    double* swc;      // [D]
    double* trc;      // [D]
    int* idle;        // [D] sorted eligible idle devices
    int* misc;        // [4]: n_idle
    double* bb;       // [1]
};

__host__ __device__ __forceinline__ size_t item_smem_bytes(int D, int Bmax) {
    size_t doubles = (size_t)D * Bmax + 3 * (size_t)D + 1;
    size_t ints = (size_t)D + 4;
    return doubles * sizeof(double) + ((ints * sizeof(int) + 15) & ~size_t(15));
}

// ---------------------------------------------------------------------------
// prologue: static per-(bank, weights) tables
// ---------------------------------------------------------------------------

// One thread per stage g: mean_base (costs.py:102-105), split penalty
// (costs.py:268-273) and per-parent-edge sigma / tail locality term at the
// default beta (costs.py:123, :341-348).
__global__ void fate_prepare_stage_kernel(fate_bank b, fate_weights w, fate_derived out) {
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= b.n_stages) return;
    const int D = b.n_devices;
    const int inst = b.st_inst[g];
    const int q0 = b.inst_query_off[inst], nq = b.inst_n_queries[inst];
    const int m = b.st_model[g], r = b.st_role[g];
    const double pcoef = m >= 0 ? b.model_prefill[m] : 1.0;
    const double dcoef = m >= 0 ? b.model_decode[m] : 0.0;
    const double pscale = b.role_prefill[r], cplx = b.role_cplx[r];
    const double decode = (double)b.st_out[g] * dcoef * b.role_decode[r];
    const uint64_t elig = b.st_elig[g];
    const int orow = b.st_override[g];

    // base_cost over the devices of _mean_base (sorted eligible, or all in
    // topology order when the eligibility set is empty)
    PySum tot;
    int n = 0;
    for (int i = 0; i < D; ++i) {
        int d;
        if (elig != 0) {
            d = i;
            if (!((elig >> d) & 1ull)) continue;
        } else {
            d = b.dev_topo_order[i];
        }
        double base;
        if (orow >= 0 && ((b.override_mask[orow] >> d) & 1ull)) {
            base = b.override_cost[(size_t)orow * D + d];
        } else {
            PySum acc;
            for (int q = 0; q < nq; ++q)
                acc.add(qc_value(b.st_prompt[g], b.q_prompt[q0 + q], pcoef, pscale, decode, cplx,
                                 b.dev_speed[d]));
            base = acc.result();
        }
        tot.add(base);
        ++n;
    }
    out.mean_base[g] = tot.result() / (double)n;

    // Neumaier sums of the stateless row (stage part P) and of the full-hit row
    // (stage part 0) under uniform speed: full batch and the two k=2 shards
    // (costs.py:257, :404-405)
    if (out.row_sums) {
        const int half = nq / 2 + (nq % 2);
#pragma unroll
        for (int which = 0; which < 2; ++which) {
            const long long sp = which == 0 ? b.st_prompt[g] : 0;
            PySum all, s0, s1;
            for (int q = 0; q < nq; ++q) {
                const double x = qc_value(sp, b.q_prompt[q0 + q], pcoef, pscale, decode, cplx,
                                          b.dev_speed[0]);
                all.add(x);
                if (q < half) s0.add(x);
                else s1.add(x);
            }
            out.row_sums[(size_t)g * 6 + 3 * which + 0] = all.result();
            out.row_sums[(size_t)g * 6 + 3 * which + 1] = s0.result();
            out.row_sums[(size_t)g * 6 + 3 * which + 2] = s1.result();
        }
    }
    if (out.inst_qgroups && g == b.inst_stage_off[inst]) {
        int any = 0;
        for (int q = 0; q < nq; ++q) any |= b.q_group[q0 + q] != -1;
        out.inst_qgroups[inst] = any;
    }

    double split = 0.0;
    for (int e = b.ch_ptr[g]; e < b.ch_ptr[g + 1]; ++e) {
        const int c = b.ch_idx[e];
        const double sigma = (double)b.st_out[g] * b.role_comm[b.st_role[c]] / 1000.0;
        split += 0.5 * b.beta_default * sigma * w.transfer_x;
    }
    out.split_penalty[g] = split;

    const double comm = b.role_comm[r];
    for (int e = b.par_ptr[g]; e < b.par_ptr[g + 1]; ++e) {
        const int p = b.par_idx[e];
        const double sigma = (double)b.st_out[p] * comm / 1000.0;
        out.edge_sigma[e] = sigma;
        out.edge_term[e] = w.lambda_tr * b.beta_default * sigma * w.transfer_x * w.locality_scale;
    }
}

// demand(v, l) = max over bucket of mean_base (costs.py:303); first maximum
__global__ void fate_prepare_demand_kernel(fate_bank b, fate_windows win, fate_derived out) {
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int L = win.levels;
    if (t >= (long long)b.n_stages * L) return;
    const long long lo = win.ptr[t], hi = win.ptr[t + 1];
    double dem = 0.0;
    for (long long i = lo; i < hi; ++i) {
        const double mb = out.mean_base[win.idx[i]];
        if (i == lo || mb > dem) dem = mb;
    }
    out.demand[t] = dem;
}

// ---------------------------------------------------------------------------
// main scoring kernel
// ---------------------------------------------------------------------------

template <int TPI>
__global__ void __launch_bounds__(128) fate_score_kernel(fate_bank b, fate_weights w,
                                                         fate_windows win, fate_derived der,
                                                         fate_state st, fate_work work,
                                                         fate_out out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int IPB = 128 / TPI;
    const int D = b.n_devices;
    const int Bmax = b.max_queries;
    const int lane_item = threadIdx.x / TPI;  // item slot in this CTA
    const int t = threadIdx.x % TPI;          // thread within the item (= device in B/D)
    const long long item = (long long)blockIdx.x * IPB + lane_item;
    const bool live = item < work.n_items;

    const size_t per_item = item_smem_bytes(D, Bmax);
    unsigned char* base = smem_raw + per_item * lane_item;
    ItemSmem sm;
    sm.qc = reinterpret_cast<double*>(base);
    sm.aware = sm.qc + (size_t)D * Bmax;
    sm.swc = sm.aware + D;
    sm.trc = sm.swc + D;
    sm.bb = sm.trc + D;
    sm.idle = reinterpret_cast<int*>(sm.bb + 1);
    sm.misc = sm.idle + D;

    // ---- item constants ------------------------------------------------------
    int s = 0, v = 0, inst = 0, q0 = 0, nq = 0, m = -1, r = 0, R = 1, gv = -1, Pv = 0, Ov = 0;
    uint64_t elig = 0;
    double clock = 0.0, pcoef = 1.0, pscale = 1.0, decode = 0.0, cplx = 1.0, comm_v = 1.0;
    bool cache_reuse = false;
    const int32_t* loc_row = nullptr;
    if (live) {
        s = work.scen[item];
        v = work.stage[item];
        inst = st.scen_inst[s];
        q0 = b.inst_query_off[inst];
        nq = b.inst_n_queries[inst];
        m = b.st_model[v];
        r = b.st_role[v];
        R = b.st_shard[v];
        gv = b.st_group[v];
        Pv = b.st_prompt[v];
        Ov = b.st_out[v];
        elig = b.st_elig[v];
        clock = st.scen_clock[s];
        pcoef = m >= 0 ? b.model_prefill[m] : 1.0;
        const double dcoef = m >= 0 ? b.model_decode[m] : 0.0;
        pscale = b.role_prefill[r];
        cplx = b.role_cplx[r];
        comm_v = b.role_comm[r];
        decode = (double)Ov * dcoef * b.role_decode[r];
        cache_reuse = (b.st_flags[v] & FATE_STAGE_CACHE_REUSE) && gv != -1;
        loc_row = st.loc + st.scen_loc_off[s] - b.inst_stage_off[inst];
    }
    const int cap4 = st.kappa_cap * 4;
    const long long dev_row0 = (long long)s * D;

    // ---- A: cache-aware query_compute table ----------------------------------
    if (live) {
        for (int p = t; p < D * nq; p += TPI) {
            const int d = p / nq, q = p - d * nq;
            if (!((elig >> d) & 1ull)) continue;
            const int32_t* kap = st.kappa + (dev_row0 + d) * cap4;
            const int kn = st.kappa_n[dev_row0 + d];
            long long sp = Pv, qp = b.q_prompt[q0 + q];
            if (cache_reuse) {
                const long long c = cached_tokens(kap, kn, gv, m);
                sp = sp - c > 0 ? sp - c : 0;
            }
            const int qg = b.q_group[q0 + q];
            if (qg != -1) {
                const long long c = cached_tokens(kap, kn, qg, m);
                qp = qp - c > 0 ? qp - c : 0;
            }
            sm.qc[d * Bmax + q] = qc_value(sp, qp, pcoef, pscale, decode, cplx, b.dev_speed[d]);
        }
    }
    __syncthreads();

    // ---- B: per-device sums, switch, transfer --------------------------------
    const int d = t;
    const bool dev_ok = live && d < D && ((elig >> d) & 1ull);
    if (dev_ok) {
        PySum acc;
        for (int q = 0; q < nq; ++q) acc.add(sm.qc[d * Bmax + q]);
        sm.aware[d] = acc.result();
        const int res = st.residency[dev_row0 + d];
        sm.swc[d] = (m < 0 || res == m) ? 0.0 : b.model_switch[m] * w.switch_x;
        double tr = 0.0;
        for (int e = b.par_ptr[v]; e < b.par_ptr[v + 1]; ++e) {
            const int L = loc_row[b.par_idx[e]];
            if (L < 0 || L == d) continue;
            tr += b.beta[(size_t)L * D + d] * der.edge_sigma[e];
        }
        sm.trc[d] = tr * w.transfer_x;
    }
    __syncthreads();

    // ---- C: base_best and the sorted idle list --------------------------------
    if (live && t == 0) {
        double bb = 0.0;
        bool first = true;
        int n_idle = 0;
        const double limit = clock + 1e-12;
        for (int e = 0; e < D; ++e) {
            if (!((elig >> e) & 1ull)) continue;
            const double a = sm.aware[e];
            if (first || a < bb) bb = a;
            first = false;
            if (st.dev_free[dev_row0 + e] <= limit) sm.idle[n_idle++] = e;
        }
        sm.bb[0] = bb;
        sm.misc[0] = n_idle;
    }
    __syncthreads();

    if (!(live && d < D)) return;  // no barriers below
    const int n_elig = __popcll(elig);
    const int bound = (w.ablation & FATE_NO_SHARD) ? 1 : (R < n_elig ? R : n_elig);
    if (!dev_ok) {
        // ineligible device: no candidate; NaN marks the hole in the dense rows
        const double qnan = __longlong_as_double(0x7ff8000000000000LL);
        double* psi = out.psi + work.psi_off[item];
        for (int k = 0; k < bound; ++k) psi[(long long)k * D + d] = qnan;
        const long long orow = item * D + d;
        if (out.sched) out.sched[orow] = qnan;
        if (out.tail) out.tail[orow] = qnan;
        if (out.completion) out.completion[orow] = qnan;
        return;
    }

    // ---- D: per-candidate terms ------------------------------------------------
    const double free_d = st.dev_free[dev_row0 + d];
    const double wait = py_max0(free_d - clock);
    const double sw = sm.swc[d];
    const double tr = sm.trc[d];
    const double here = sm.aware[d];
    const bool no_loc = w.ablation & FATE_NO_LOCALITY;
    const bool no_pre = w.ablation & FATE_NO_PREFIX;
    const bool no_shard = w.ablation & FATE_NO_SHARD;

    // colo (costs.py:160-165): located-on-d parents over ALL parents
    const int pa0 = b.par_ptr[v], pa1 = b.par_ptr[v + 1];
    double colo = 0.0;
    if (pa1 > pa0) {
        int hit = 0;
        for (int e = pa0; e < pa1; ++e) hit += loc_row[b.par_idx[e]] == d;
        colo = (double)hit / (double)(pa1 - pa0);
    }

    // prefix_overlap_thousands (costs.py:127-145): integer-exact token sum
    const int32_t* kap = st.kappa + (dev_row0 + d) * cap4;
    const int kn = st.kappa_n[dev_row0 + d];
    long long tokens = 0;
    if (cache_reuse) {
        const long long c = cached_tokens(kap, kn, gv, m);
        tokens += c < Pv ? c : Pv;
    }
    for (int q = 0; q < nq; ++q) {
        const int qg = b.q_group[q0 + q];
        if (qg == -1) continue;
        const long long c = cached_tokens(kap, kn, qg, m);
        const long long qp = b.q_prompt[q0 + q];
        tokens += c < qp ? c : qp;
    }
    const double prefix = w.kappa_prefix * ((double)tokens / 1000.0) * w.prefix_x;

    // _parallel_benefit (costs.py:181-201) with _even_split (costs.py:419-428)
    const double full_total = sw + tr + here;
    double parallel = 0.0;
    if (R > 1 && !no_shard) {
        const int n_idle = sm.misc[0];
        const bool self_idle = free_d <= clock + 1e-12;
        const int others = n_idle - (self_idle ? 1 : 0);
        const int k = R < 1 + others ? R : 1 + others;
        if (k > 1) {
            double worst = 0.0;
            int start = 0, j = 0;
            for (int i = 0; i < k; ++i) {
                int dev = d;
                if (i > 0) {
                    while (sm.idle[j] == d) ++j;
                    dev = sm.idle[j++];
                }
                const int size = nq / k + (i < nq % k ? 1 : 0);
                PySum acc;
                for (int q = start; q < start + size; ++q) acc.add(sm.qc[dev * Bmax + q]);
                const double tot = sm.swc[dev] + sm.trc[dev] + acc.result();
                if (i == 0 || tot > worst) worst = tot;
                start += size;
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

    // tail_value (costs.py:281-352)
    double tail = 0.0;
    const int H = w.eff_horizon;
    if (H > 1) {
        const int res = st.residency[dev_row0 + d];
        const bool displaces = res != -1 && res != m;
        const bool no_same = w.ablation & FATE_NO_SAME_MODEL;
        const int L = win.levels;
        for (int l = 1; l < H; ++l) {
            const long long lo = win.ptr[(long long)v * L + (l - 1)];
            const long long hi = win.ptr[(long long)v * L + l];
            if (hi == lo) continue;
            double aff = 0.0;
            for (long long i = lo; i < hi; ++i) {
                const int x = win.idx[i];
                const int mx = b.st_model[x];
                if (!no_same && mx != -1) {
                    if (mx == m) {
                        aff += w.lambda_s * b.model_switch[mx] * w.switch_x * w.state_scale;
                    } else if (displaces && mx == res) {
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
                if (!no_loc) {
                    for (int e = b.par_ptr[x]; e < b.par_ptr[x + 1]; ++e) {
                        const int p = b.par_idx[e];
                        if (p == v) continue;
                        const int Lp = loc_row[p];
                        if (Lp < 0 || Lp == d) continue;
                        if (b.has_overrides) {
                            aff -= w.lambda_tr * b.beta[(size_t)Lp * D + d] * der.edge_sigma[e] *
                                   w.transfer_x * w.locality_scale;
                        } else {
                            aff -= der.edge_term[e];
                        }
                    }
                }
            }
            const double dem = der.demand[(long long)v * L + (l - 1)];
            tail += w.gamma_pow[l] * (aff / (double)(hi - lo) + w.demand_coeff * dem);
        }
    }

    const long long orow = item * D + d;
    if (out.sched) out.sched[orow] = S;
    if (out.tail) out.tail[orow] = tail;
    if (out.completion) out.completion[orow] = wait + full_total;

    double* psi = out.psi + work.psi_off[item];
    psi[d] = S + tail;

    // _marginal_shard_score (costs.py:249-279), slots 1..bound-1
    if (bound > 1) {
        const double bb = sm.bb[0];
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

#include "fate_score_v3.cuh"
#include "fate_score_v4.cuh"
#include "fate_score_v5.cuh"
#include "fate_score_v6.cuh"

template <int DPL, bool OVR, int MINB>
int launch_v6_mb(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
                 const fate_derived* der, const fate_state* st, const fate_work* work,
                 const fate_out* out, cudaStream_t s) {
    if (!der->stage_rec || (win->levels > 0 && (!der->tmpl_ptr || !der->tmpl)))
        return fail(FATE_ENOTREADY, "v6 kernel needs stage records and op templates");
    const V6Layout lay = v6_layout(bank->n_devices, bank->max_queries, win->max_level_ops);
    const size_t smem = (size_t)lay.item_bytes * 4;
    if (smem > 220 * 1024) return fail(FATE_ETOOBIG, "v6 shared-memory footprint too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fate_score_v6_kernel<DPL, OVR, MINB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // persistent grid: every resident CTA slot once (capped by the item count)
    static thread_local size_t occ_smem = ~size_t(0);
    static thread_local int occ_dev = -1, o = 0;
    static thread_local const void* occ_fn = nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    const void* fn = (const void*)fate_score_v6_kernel<DPL, OVR, MINB>;
    if (occ_smem != smem || occ_dev != dev || occ_fn != fn) {
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fate_score_v6_kernel<DPL, OVR, MINB>,
                                                      128, smem);
        o = std::max(1, sms * std::max(1, per));
        occ_smem = smem;
        occ_dev = dev;
        occ_fn = fn;
    }
    // items per ticket: 2 for one device slot per lane, 1 for two (heavier
    // items: finer tail balance beats fewer atomics; measured on B200)
    static int fetch_env = -2;
    if (fetch_env == -2) {
        const char* e = getenv("FATE_V6_FETCH");
        fetch_env = e ? std::max(1, std::min(64, atoi(e))) : -1;
    }
    const int fetch = fetch_env > 0 ? fetch_env : (DPL == 1 ? V6_FETCH : 1);
    if (work->n_items > 0x7fffffffLL - 4 * 128 * 64)
        return fail(FATE_ETOOBIG, "v6: too many items for the 32-bit ticket counter");
    const long long want = (work->n_items + 3) / 4;
    const unsigned blocks = (unsigned)std::min<long long>(o, want);
    static std::atomic<int> slot{0};
    const int qs = slot.fetch_add(1) % V6_QSLOTS;
    fate_score_v6_kernel<DPL, OVR, MINB><<<blocks, 128, smem, s>>>(*bank, *w, *win, *der, *st,
                                                                    *work, *out, lay, qs, fetch);
    return 0;
}

template <int DPL, int MINB>
int launch_v5_mb(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
                 const fate_derived* der, const fate_state* st, const fate_work* work,
                 const fate_out* out, cudaStream_t s) {
    const size_t smem = v5_item_bytes(bank->n_devices, bank->max_queries, win->max_level_ops) * 4;
    if (smem > 220 * 1024) return fail(FATE_ETOOBIG, "v5 shared-memory footprint too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fate_score_v5_kernel<DPL, MINB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned blocks = (unsigned)((work->n_items + 3) / 4);
    fate_score_v5_kernel<DPL, MINB><<<blocks, 128, smem, s>>>(*bank, *w, *win, *der, *st, *work,
                                                               *out);
    return 0;
}

template <int DPL, int MINB>
int launch_v4_mb(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
                 const fate_derived* der, const fate_state* st, const fate_work* work,
                 const fate_out* out, cudaStream_t s) {
    const size_t smem = v4_item_bytes(bank->n_devices, bank->max_queries, win->max_level_ops) * 4;
    if (smem > 220 * 1024) return fail(FATE_ETOOBIG, "v4 shared-memory footprint too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fate_score_v4_kernel<DPL, MINB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned blocks = (unsigned)((work->n_items + 3) / 4);
    fate_score_v4_kernel<DPL, MINB><<<blocks, 128, smem, s>>>(*bank, *w, *win, *der, *st, *work,
                                                               *out);
    return 0;
}

// register budget: CTAs per SM the register allocation must allow.  Measured
// on B200 (profiles/): 8 for one device slot per lane (<= 64 registers); for
// two, 6 (<= 80) for v4/v5 and 7 (<= 72, no spills) for v6.  FATE_MINB =
// 1 | 6 | 7 | 8 overrides for A/B runs.
int v4_minb(int dpl) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FATE_MINB");
        v = e ? atoi(e) : 0;
    }
    return v ? v : (dpl == 1 ? 8 : 6);
}

template <int DPL>
int launch_v5(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
              const fate_derived* der, const fate_state* st, const fate_work* work,
              const fate_out* out, cudaStream_t s) {
    switch (v4_minb(DPL)) {
        case 1: return launch_v5_mb<DPL, 1>(bank, w, win, der, st, work, out, s);
        case 6: return launch_v5_mb<DPL, 6>(bank, w, win, der, st, work, out, s);
        default: return launch_v5_mb<DPL, 8>(bank, w, win, der, st, work, out, s);
    }
}

template <int DPL>
int launch_v6(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
              const fate_derived* der, const fate_state* st, const fate_work* work,
              const fate_out* out, cudaStream_t s) {
    const bool ovr = bank->has_overrides != 0;
    const char* e = getenv("FATE_MINB");
    switch (e ? atoi(e) : (DPL == 1 ? 8 : 7)) {
        case 1:
            return ovr ? launch_v6_mb<DPL, true, 1>(bank, w, win, der, st, work, out, s)
                       : launch_v6_mb<DPL, false, 1>(bank, w, win, der, st, work, out, s);
        case 7:
            return ovr ? launch_v6_mb<DPL, true, 7>(bank, w, win, der, st, work, out, s)
                       : launch_v6_mb<DPL, false, 7>(bank, w, win, der, st, work, out, s);
        case 6:
            return ovr ? launch_v6_mb<DPL, true, 6>(bank, w, win, der, st, work, out, s)
                       : launch_v6_mb<DPL, false, 6>(bank, w, win, der, st, work, out, s);
        default:
            return ovr ? launch_v6_mb<DPL, true, 8>(bank, w, win, der, st, work, out, s)
                       : launch_v6_mb<DPL, false, 8>(bank, w, win, der, st, work, out, s);
    }
}

template <int DPL>
int launch_v4(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
              const fate_derived* der, const fate_state* st, const fate_work* work,
              const fate_out* out, cudaStream_t s) {
    switch (v4_minb(DPL)) {
        case 6: return launch_v4_mb<DPL, 6>(bank, w, win, der, st, work, out, s);
        case 8: return launch_v4_mb<DPL, 8>(bank, w, win, der, st, work, out, s);
        default: return launch_v4_mb<DPL, 1>(bank, w, win, der, st, work, out, s);
    }
}

template <int G>
int launch_v3(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
              const fate_derived* der, const fate_state* st, const fate_work* work,
              const fate_out* out, cudaStream_t s) {
    constexpr int IPB = 128 / G;
    const size_t smem = v3_item_bytes(bank->n_devices, bank->max_queries, G, win->max_level_ops) * IPB;
    if (smem > 220 * 1024) return fail(FATE_ETOOBIG, "v3 shared-memory footprint too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fate_score_v3_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    const unsigned blocks = (unsigned)((work->n_items + IPB - 1) / IPB);
    fate_score_v3_kernel<G><<<blocks, 128, smem, s>>>(*bank, *w, *win, *der, *st, *work, *out);
    return 0;
}

// Kernel generation (A/B benchmarking only): FATE_SCORE_KERNEL=v1|v3|v4|v5,
// default v6 (which needs the stage records and op templates; without them
// the library falls back to v5, the previous production kernel).
int kernel_gen() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("FATE_SCORE_KERNEL");
        v = (e && strcmp(e, "v1") == 0)   ? 1
            : (e && strcmp(e, "v3") == 0) ? 3
            : (e && strcmp(e, "v4") == 0) ? 4
            : (e && strcmp(e, "v5") == 0) ? 5
                                          : 6;
    }
    return v;
}

int check_bank(const fate_bank* b) {
    if (!b) return fail(FATE_EINVAL, "bank is NULL");
    if (b->n_devices < 1 || b->n_devices > FATE_MAX_DEVICES)
        return fail(FATE_ETOOBIG, "n_devices outside 1..64");
    if (b->max_queries < 0 || b->max_queries > FATE_MAX_QUERIES)
        return fail(FATE_ETOOBIG, "batch size exceeds FATE_MAX_QUERIES");
    if (b->n_stages < 0 || b->n_edges < 0) return fail(FATE_EINVAL, "negative sizes");
    return 0;
}

int check_weights(const fate_weights* w, const fate_windows* win) {
    if (!w || !win) return fail(FATE_EINVAL, "weights/windows is NULL");
    if (w->eff_horizon < 0 || w->eff_horizon >= FATE_MAX_HORIZON)
        return fail(FATE_ETOOBIG, "horizon exceeds FATE_MAX_HORIZON-1");
    const int levels = w->eff_horizon > 1 ? w->eff_horizon - 1 : 0;
    if (win->levels != levels) return fail(FATE_EINVAL, "windows built for another horizon");
    return 0;
}

// Wire format -> SoA (fate_pipeline.cpp): blocks [0, n_s) scatter one scenario
// record each (layout in fate.h), the next n_ib blocks 128 items each, the rest
// widen 512 int8 loc entries each.
__global__ void fate_unpack_kernel(const unsigned char* __restrict__ rec, size_t rb, int s0,
                                   int n_s, int D, int cap, const fate_item* __restrict__ items,
                                   int i0, int n_i, int n_ib, const int8_t* __restrict__ loc8,
                                   long long l0, long long l1, fate_state dst, int32_t* w_scen,
                                   int32_t* w_stage, int64_t* w_psi_off) {
    if ((int)blockIdx.x >= n_s + n_ib) {
        const long long base = l0 + ((long long)blockIdx.x - n_s - n_ib) * 512;
        int32_t* out = const_cast<int32_t*>(dst.loc);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const long long i = base + k * 128 + threadIdx.x;
            if (i < l1) out[i] = loc8[i];
        }
        return;
    }
    if ((int)blockIdx.x < n_s) {
        const int s = s0 + blockIdx.x;
        const unsigned char* r = rec + rb * s;
        if (threadIdx.x == 0) {
            const_cast<double*>(dst.scen_clock)[s] = *reinterpret_cast<const double*>(r);
            const_cast<int64_t*>(dst.scen_loc_off)[s] = *reinterpret_cast<const int64_t*>(r + 8);
            const_cast<int32_t*>(dst.scen_inst)[s] = *reinterpret_cast<const int32_t*>(r + 16);
            const_cast<int32_t*>(dst.scen_done_level)[s] = *reinterpret_cast<const int32_t*>(r + 20);
        }
        const int32_t* res = reinterpret_cast<const int32_t*>(r + 32);
        const int32_t* kn = res + D;
        const double* fr = reinterpret_cast<const double*>(r + 32 + 8 * D);
        const int4* kap = reinterpret_cast<const int4*>(r + 32 + 16 * D);
        const size_t row = (size_t)s * D;
        for (int d = threadIdx.x; d < D; d += blockDim.x) {
            const_cast<int32_t*>(dst.residency)[row + d] = res[d];
            const_cast<int32_t*>(dst.kappa_n)[row + d] = kn[d];
            const_cast<double*>(dst.dev_free)[row + d] = fr[d];
        }
        int4* kdst = reinterpret_cast<int4*>(const_cast<int32_t*>(dst.kappa)) + row * cap;
        for (int k = threadIdx.x; k < D * cap; k += blockDim.x) kdst[k] = kap[k];
    } else {
        const int i = i0 + ((int)blockIdx.x - n_s) * blockDim.x + threadIdx.x;
        if (i >= i0 + n_i) return;
        const fate_item x = items[i];
        w_scen[i] = x.scen;
        w_stage[i] = x.stage;
        w_psi_off[i] = x.psi_off;
    }
}

}  // namespace

int fate_internal_fail(int code, const std::string& msg) { return fail(code, msg); }

long long fate_internal_launches() { return g_launches.load(); }

void fate_internal_count_launches(long long n) { g_launches += n; }

int fate_internal_unpack(const void* rec, size_t rec_bytes, int s0, int s1, int D, int cap,
                         const fate_item* items, int i0, int i1, const int8_t* loc8, int64_t l0,
                         int64_t l1, const fate_state* dst, int32_t* w_scen, int32_t* w_stage,
                         int64_t* w_psi_off, cudaStream_t s) {
    const int n_s = s1 - s0, n_i = i1 - i0;
    const int n_ib = (n_i + 127) / 128;
    const long long n_lb = (l1 - l0 + 511) / 512;
    const unsigned blocks = (unsigned)(n_s + n_ib + n_lb);
    if (blocks == 0) return 0;
    fate_unpack_kernel<<<blocks, 128, 0, s>>>(static_cast<const unsigned char*>(rec), rec_bytes,
                                               s0, n_s, D, cap, items, i0, n_i, n_ib, loc8, l0,
                                               l1, *dst, w_scen, w_stage, w_psi_off);
    g_launches++;
    return cuda_status("fate_unpack_kernel");
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" {

int fate_abi_version(void) { return FATE_ABI_VERSION; }

const char* fate_last_error(void) { return g_last_error.c_str(); }

int64_t fate_launch_count(void) { return g_launches.load(); }

int fate_prepare(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
                 const fate_derived* out, void* stream) {
    int rc = check_bank(bank);
    if (rc) return rc;
    rc = check_weights(w, win);
    if (rc) return rc;
    if (!out) return fail(FATE_EINVAL, "derived is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    {
        // the v6 quotient tables, once per device (stream-ordered before any
        // scoring launch that follows this prologue)
        static std::atomic<unsigned long long> done{0};
        int dev = 0;
        cudaGetDevice(&dev);
        const unsigned long long bit = 1ull << (dev & 63);
        if (!(done.load() & bit)) {
            fate_v6_tables_kernel<<<(V6_DIVTAB + 127) / 128, 128, 0, s>>>();
            g_launches++;
            if ((rc = cuda_status("fate_v6_tables_kernel"))) return rc;
            // one-time: make the tables visible to scoring launches on any stream
            if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_status("fate_v6_tables_kernel");
            done.fetch_or(bit);
        }
    }
    if (bank->n_stages > 0) {
        const int threads = 128;
        const int blocks = (bank->n_stages + threads - 1) / threads;
        fate_prepare_stage_kernel<<<blocks, threads, 0, s>>>(*bank, *w, *out);
        g_launches++;
        if ((rc = cuda_status("fate_prepare_stage_kernel"))) return rc;
        if (out->stage_rec) {
            if (!out->split_penalty || !out->inst_qgroups)
                return fail(FATE_EINVAL, "stage records need split_penalty and inst_qgroups");
            fate_prepare_stagerec_kernel<<<blocks, threads, 0, s>>>(*bank, *w, *out);
            g_launches++;
            if ((rc = cuda_status("fate_prepare_stagerec_kernel"))) return rc;
        }
        const long long n = (long long)bank->n_stages * win->levels;
        if (n > 0) {
            fate_prepare_demand_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(
                *bank, *win, *out);
            g_launches++;
            if ((rc = cuda_status("fate_prepare_demand_kernel"))) return rc;
            if (out->tmpl && out->tmpl_ptr) {
                fate_template_fill_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0,
                                            s>>>(*bank, *w, *win, *out);
                g_launches++;
                if ((rc = cuda_status("fate_template_fill_kernel"))) return rc;
            }
            if (out->tail_static) {
                const long long nt = n * (bank->n_models + 1);
                fate_prepare_tail_static_kernel<<<(unsigned)((nt + threads - 1) / threads), threads, 0,
                                                  s>>>(*bank, *w, *win, out->tail_static);
                g_launches++;
                if ((rc = cuda_status("fate_prepare_tail_static_kernel"))) return rc;
                if (out->tail_sum) {
                    const long long ns = (long long)bank->n_stages * (bank->n_models + 1);
                    fate_prepare_tail_sum_kernel<<<(unsigned)((ns + threads - 1) / threads),
                                                   threads, 0, s>>>(*bank, *w, *win, *out);
                    g_launches++;
                    if ((rc = cuda_status("fate_prepare_tail_sum_kernel"))) return rc;
                }
            }
        }
    }
    return 0;
}

int fate_template_count(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
                        const fate_derived* der, int64_t* counts, void* stream) {
    int rc = check_bank(bank);
    if (rc) return rc;
    rc = check_weights(w, win);
    if (rc) return rc;
    if (!der || !counts) return fail(FATE_EINVAL, "derived/counts is NULL");
    const long long n = (long long)bank->n_stages * win->levels;
    if (n == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    fate_template_count_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(
        *bank, *w, *win, *der, reinterpret_cast<long long*>(counts));
    g_launches++;
    return cuda_status("fate_template_count_kernel");
}

int fate_score(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
               const fate_derived* der, const fate_state* st, const fate_work* work,
               const fate_out* out, void* stream) {
    int rc = check_bank(bank);
    if (rc) return rc;
    rc = check_weights(w, win);
    if (rc) return rc;
    if (!der || !st || !work || !out || !out->psi)
        return fail(FATE_EINVAL, "NULL derived/state/work/out");
    if (st->kappa_cap < 1 || st->kappa_cap > FATE_MAX_KAPPA)
        return fail(FATE_ETOOBIG, "kappa_cap outside 1..FATE_MAX_KAPPA");
    if (work->n_items <= 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int D = bank->n_devices;
    const size_t per_item = item_smem_bytes(D, bank->max_queries);
    const bool v6_ready = der->stage_rec && (win->levels == 0 || (der->tmpl_ptr && der->tmpl));
    if (kernel_gen() == 6 && v6_ready) {
        rc = D <= 32 ? launch_v6<1>(bank, w, win, der, st, work, out, s)
                     : launch_v6<2>(bank, w, win, der, st, work, out, s);
        if (rc) return rc;
    } else if (kernel_gen() >= 5) {
        rc = D <= 32 ? launch_v5<1>(bank, w, win, der, st, work, out, s)
                     : launch_v5<2>(bank, w, win, der, st, work, out, s);
        if (rc) return rc;
    } else if (kernel_gen() == 4) {
        rc = D <= 32 ? launch_v4<1>(bank, w, win, der, st, work, out, s)
                     : launch_v4<2>(bank, w, win, der, st, work, out, s);
        if (rc) return rc;
    } else if (kernel_gen() == 3) {
        rc = D <= 32 ? launch_v3<32>(bank, w, win, der, st, work, out, s)
                     : launch_v3<64>(bank, w, win, der, st, work, out, s);
        if (rc) return rc;
    } else if (D <= 32) {
        constexpr int TPI = 32, IPB = 128 / TPI;
        const size_t smem = per_item * IPB;
        if (smem > 48 * 1024) {
            cudaFuncSetAttribute(fate_score_kernel<TPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        }
        const unsigned blocks = (unsigned)((work->n_items + IPB - 1) / IPB);
        fate_score_kernel<TPI><<<blocks, TPI * IPB, smem, s>>>(*bank, *w, *win, *der, *st, *work,
                                                               *out);
    } else {
        constexpr int TPI = 64, IPB = 128 / TPI;
        const size_t smem = per_item * IPB;
        if (smem > 48 * 1024) {
            cudaFuncSetAttribute(fate_score_kernel<TPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        }
        const unsigned blocks = (unsigned)((work->n_items + IPB - 1) / IPB);
        fate_score_kernel<TPI><<<blocks, TPI * IPB, smem, s>>>(*bank, *w, *win, *der, *st, *work,
                                                               *out);
    }
    g_launches++;
    return cuda_status("fate_score_kernel");
}

}  // extern "C"
