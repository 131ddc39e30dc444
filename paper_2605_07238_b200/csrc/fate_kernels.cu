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
// Work decomposition: one "item" = (scenario, stage v) is scored by one warp
// (fate_score_v6.cuh, the production kernel; fate_score_v5.cuh is the previous
// generation, compiled only into -DFATE_AB experiment builds).  This file holds the shared device helpers, the
// prologue kernels of fate_prepare (mean_base, demand, split penalty, edge
// terms, static tail tables, stage records, op templates), the wire-format
// unpack kernel of the host pipeline, and the C ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "fate.h"
#include "fate_internal.h"

namespace {

thread_local std::string g_last_error;
// queue slot for the next v6 launch of this thread (-1: rotate over the
// direct-launch slots); set by the host pipeline around its scoring launches
thread_local int g_queue_slot_override = -1;
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

#include "fate_prologue.cuh"
#ifdef FATE_AB
#include "fate_score_v5.cuh"
#endif
#include "fate_score_v6.cuh"

// A/B knobs.  The production library (built without FATE_AB) runs exactly
// one kernel generation with the measured launch shape; a build with
// -DFATE_AB (FATE_BUILD_AB=1 python -m paper_2605_07238_b200.build) adds the
// previous generation v5 and reads the environment overrides below, for
// experiments only.
#ifdef FATE_AB
int ab_env(const char* name, int dflt, int lo, int hi) {
    const char* e = getenv(name);
    return e ? std::max(lo, std::min(hi, atoi(e))) : dflt;
}
#endif

template <int DPL, bool OVR, bool SL, int MINB, bool QG, bool UNIT = false>
int launch_v6_mb(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
                 const fate_derived* der, const fate_state* st, const fate_work* work,
                 const fate_out* out, cudaStream_t s) {
    if (!der->stage_rec || (win->levels > 0 && (!der->tmpl_ptr || !der->tmpl)))
        return fail(FATE_ENOTREADY, "v6 kernel needs stage records and op templates");
#ifdef FATE_AB
    static const int opcap_env = ab_env("FATE_V6_OPCAP", 0, 32, 4096) & ~3;
    const int opcap = opcap_env > 0 ? opcap_env : v6_opcap_default<DPL>();
#else
    const int opcap = v6_opcap_default<DPL>();
#endif
    constexpr bool maskw = !OVR && DPL == 2;
    V6Layout lay =
        SL ? v6_layout_static<DPL>(win->max_level_ops, bank->n_models, maskw, opcap)
           : v6_layout(bank->n_devices, bank->max_queries, win->max_level_ops, bank->n_models,
                       maskw, opcap);
#ifdef FATE_AB
    static const int diag_env = ab_env("FATE_V6_DIAG", 0, 0, 15);
    lay.diag = diag_env;
#endif
    const size_t smem = (size_t)lay.item_bytes * 4;
    if (smem > 220 * 1024) return fail(FATE_ETOOBIG, "v6 shared-memory footprint too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fate_score_v6_kernel<DPL, OVR, SL, MINB, QG, UNIT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // persistent grid: every resident CTA slot once (capped by the item count)
    static thread_local size_t occ_smem = ~size_t(0);
    static thread_local int occ_dev = -1, o = 0;
    static thread_local const void* occ_fn = nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    const void* fn = (const void*)fate_score_v6_kernel<DPL, OVR, SL, MINB, QG, UNIT>;
    if (occ_smem != smem || occ_dev != dev || occ_fn != fn) {
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fate_score_v6_kernel<DPL, OVR, SL, MINB, QG, UNIT>,
                                                      128, smem);
        o = std::max(1, sms * std::max(1, per));
        occ_smem = smem;
        occ_dev = dev;
        occ_fn = fn;
    }
    if (work->n_items > 0x7fffffffLL - 4 * 128 * 64)
        return fail(FATE_ETOOBIG, "v6: too many items for the 32-bit ticket counter");
    const long long want = (work->n_items + 3) / 4;
    const unsigned blocks = (unsigned)std::min<long long>(o, want);
    // items per ticket, one device slot per lane: 3 on batches of >= 8 items
    // per warp, 2 on >= 3, else 1; two slots: 1 (heavier items, or small
    // shards -- 2 items per warp at config 5's 8-way shard: finer tail
    // balance beats fewer atomics).  Measured on B200 at the current
    // register budgets (A/B: 0 = guided sizes).
    const long long per_warp = work->n_items / (4LL * blocks);
    const int fetch_dflt = DPL != 1 ? 1 : per_warp >= 8 ? 3 : per_warp >= 3 ? 2 : 1;
#ifdef FATE_AB
    static const int fetch_env = ab_env("FATE_V6_FETCH", -1, 0, 64);
    const int fetch = fetch_env >= 0 ? fetch_env : fetch_dflt;
#else
    const int fetch = fetch_dflt;
#endif
    // static first share on batches of >= 3 items per warp: each warp first
    // scores a contiguous run of its share (no atomics, one scenario's rows
    // stay in L1), then pulls tickets.  3/4 of the share for one device slot
    // (config-5 items cost alike), 1/2 for two (config-4 items vary with
    // their walked levels).  Measured on B200: C5 -3 %, C4 -1.5 %, 4-way C5
    // shard -6 %; larger static shares made C4 up to 25 % slower, the whole
    // share made both slower.
    const long long first_take = per_warp < 3 ? 0 : DPL == 1 ? per_warp * 3 / 4 : per_warp / 2;
    const int fetch_arg = fetch | (int)(std::min<long long>(first_take, 255) << 8);
    static std::atomic<int> slot{0};
    const int qs = g_queue_slot_override >= 0 ? g_queue_slot_override
                                              : slot.fetch_add(1) % V6_QDIRECT;
    fate_score_v6_kernel<DPL, OVR, SL, MINB, QG, UNIT><<<blocks, 128, smem, s>>>(*bank, *w, *win, *der, *st,
                                                                    *work, *out, lay, qs, fetch_arg);
    return 0;
}

#ifdef FATE_AB
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

template <int DPL>
int launch_v5(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
              const fate_derived* der, const fate_state* st, const fate_work* work,
              const fate_out* out, cudaStream_t s) {
    switch (ab_env("FATE_MINB", DPL == 1 ? 8 : 6, 1, 16)) {
        case 1: return launch_v5_mb<DPL, 1>(bank, w, win, der, st, work, out, s);
        case 6: return launch_v5_mb<DPL, 6>(bank, w, win, der, st, work, out, s);
        default: return launch_v5_mb<DPL, 8>(bank, w, win, der, st, work, out, s);
    }
}
#endif

// The UNIT instantiation's precondition (fate_score_v6.cuh v6_item): no
// ablation and every multiplicative identity weight exactly 1.0 (and, checked
// at the call, D == 64 for two device slots).
inline bool v6_unit_weights(const fate_weights* w) {
    return w->ablation == 0 && w->lambda_q == 1.0 && w->lambda_s == 1.0 &&
           w->lambda_tr == 1.0 && w->state_scale == 1.0 && w->locality_scale == 1.0 &&
           w->prefix_scale == 1.0 && w->transfer_x == 1.0 && w->prefix_x == 1.0 &&
           w->kappa_prefix == 1.0;
}

// Lean instantiation (QG = false) when the bank declares that no query has a
// prefix group (FATE_BANK_NO_QGROUPS) and every device has the same speed
// (FATE_BANK_UNIFORM_SPEED) -- both verified by fate_prepare -- and the
// topology has no transfer override: the per-device query-group and
// per-speed class paths compile out (configs 4/5: 12 % less code, C4 -6.6 %,
// C5 -1.7 % on B200 -- the D = 64 kernel was instruction-fetch bound).
template <int DPL, bool SL, int MINB>
int launch_v6_q(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
                const fate_derived* der, const fate_state* st, const fate_work* work,
                const fate_out* out, cudaStream_t s) {
    if (bank->has_overrides != 0)
        return launch_v6_mb<DPL, true, SL, MINB, true>(bank, w, win, der, st, work, out, s);
    if ((bank->flags & FATE_BANK_NO_QGROUPS) && (bank->flags & FATE_BANK_UNIFORM_SPEED)) {
#ifndef FATE_V6_NOUNIT
        if (v6_unit_weights(w) && (DPL == 1 || bank->n_devices == 64))
            return launch_v6_mb<DPL, false, SL, MINB, false, true>(bank, w, win, der, st, work,
                                                                   out, s);
#endif
        return launch_v6_mb<DPL, false, SL, MINB, false>(bank, w, win, der, st, work, out, s);
    }
    return launch_v6_mb<DPL, false, SL, MINB, true>(bank, w, win, der, st, work, out, s);
}

// Register budget (CTAs per SM), measured on B200: 10 for one device slot per
// lane (48 registers: the extra warps hide more latency than the spills
// cost; 8/9/12 were slower), 8 for two (64 registers; 1 % ahead of 7 x 72
// registers once the chunked op buffer let 8 CTAs fit in shared memory).
template <int DPL, bool SL>
int launch_v6_sl(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
                 const fate_derived* der, const fate_state* st, const fate_work* work,
                 const fate_out* out, cudaStream_t s) {
#ifndef FATE_V6_MINB1
#define FATE_V6_MINB1 10
#endif
#ifndef FATE_V6_MINB2
#define FATE_V6_MINB2 8
#endif
    constexpr int MINB = DPL == 1 ? FATE_V6_MINB1 : FATE_V6_MINB2;
#ifdef FATE_AB
    switch (ab_env("FATE_MINB", MINB, 1, 16)) {
        case 7: return launch_v6_q<DPL, SL, 7>(bank, w, win, der, st, work, out, s);
        case 8: return launch_v6_q<DPL, SL, 8>(bank, w, win, der, st, work, out, s);
        case 10: return launch_v6_q<DPL, SL, 10>(bank, w, win, der, st, work, out, s);
        case 12: return launch_v6_q<DPL, SL, 12>(bank, w, win, der, st, work, out, s);
        case 16: return launch_v6_q<DPL, SL, 16>(bank, w, win, der, st, work, out, s);
        default: break;
    }
#endif
    return launch_v6_q<DPL, SL, MINB>(bank, w, win, der, st, work, out, s);
}

// Static shared-memory layout when the query batch fits it (V6Static<DPL>;
// measured: C4 -4.5 %); larger batches use the runtime layout.
template <int DPL>
int launch_v6(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
              const fate_derived* der, const fate_state* st, const fate_work* work,
              const fate_out* out, cudaStream_t s) {
#ifdef FATE_AB
    static const bool dyn = getenv("FATE_V6_DYNLAYOUT") != nullptr;
#else
    constexpr bool dyn = false;
#endif
    if (!dyn && bank->max_queries <= V6Static<DPL>::B)
        return launch_v6_sl<DPL, true>(bank, w, win, der, st, work, out, s);
    return launch_v6_sl<DPL, false>(bank, w, win, der, st, work, out, s);
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
    const double* f = &w->lambda_q;  // the 17 leading doubles of ScoreWeights
    for (int i = 0; i < 17; ++i)
        if (!std::isfinite(f[i])) return fail(FATE_EINVAL, "non-finite ScoreWeights field");
    for (int l = 0; l < FATE_MAX_HORIZON && l < w->eff_horizon + 1; ++l)
        if (!std::isfinite(w->gamma_pow[l])) return fail(FATE_EINVAL, "non-finite gamma ** l");
    if (w->eff_horizon < 0 || w->eff_horizon >= FATE_MAX_HORIZON)
        return fail(FATE_ETOOBIG, "horizon exceeds FATE_MAX_HORIZON-1");
    const int levels = w->eff_horizon > 1 ? w->eff_horizon - 1 : 0;
    if (win->levels != levels) return fail(FATE_EINVAL, "windows built for another horizon");
    return 0;
}

// realized_duration (costs.py:383-416) of arbitrary shard tasks on one
// scenario state, one thread per task: switch_cost (costs.py:107-111),
// transfer_cost (costs.py:113-125, beta table), and the CPython-sum of the
// cache-aware query_compute (costs.py:70-94) over the task's queries in their
// order -- the executor's issue-time pricing (executor.py:231-233).
__global__ void fate_realized_kernel(fate_bank b, fate_weights w, fate_state st, int scen, int n,
                                     const fate_task* __restrict__ tasks,
                                     const int32_t* __restrict__ tq, double* __restrict__ timing) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const fate_task t = tasks[i];
    const int v = t.stage, d = t.device, D = b.n_devices;
    const int inst = b.st_inst[v];
    const int m = b.st_model[v], r = b.st_role[v];
    const long long row = (long long)scen * D + d;
    const double sw = (m < 0 || st.residency[row] == m) ? 0.0 : b.model_switch[m] * w.switch_x;
    const int32_t* loc_row = st.loc + st.scen_loc_off[scen] - b.inst_stage_off[inst];
    const double comm = b.role_comm[r];
    double tr = 0.0;
    for (int e = b.par_ptr[v]; e < b.par_ptr[v + 1]; ++e) {
        const int u = b.par_idx[e];
        const int L = loc_row[u];
        if (L < 0 || L == d) continue;
        const double sigma = (double)b.st_out[u] * comm / 1000.0;
        tr += b.beta[(size_t)L * D + d] * sigma;
    }
    tr = tr * w.transfer_x;
    const double pcoef = m >= 0 ? b.model_prefill[m] : 1.0;
    const double dcoef = m >= 0 ? b.model_decode[m] : 0.0;
    const double decode = (double)b.st_out[v] * dcoef * b.role_decode[r];
    const int32_t* kap = st.kappa + row * st.kappa_cap * 4;
    const int kn = st.kappa_n[row];
    long long sp = b.st_prompt[v];
    const int gv = b.st_group[v];
    if ((b.st_flags[v] & FATE_STAGE_CACHE_REUSE) && gv != -1) {
        const long long c = cached_tokens(kap, kn, gv, m);
        sp = sp - c > 0 ? sp - c : 0;
    }
    const int q0 = b.inst_query_off[inst];
    PySum acc;
    for (int k = t.q0; k < t.q0 + t.nq; ++k) {
        const int q = q0 + tq[k];
        long long qp = b.q_prompt[q];
        if (b.q_group[q] != -1) {
            const long long c = cached_tokens(kap, kn, b.q_group[q], m);
            qp = qp - c > 0 ? qp - c : 0;
        }
        acc.add(qc_value(sp, qp, pcoef, b.role_prefill[r], decode, b.role_cplx[r],
                         b.dev_speed[d]));
    }
    timing[3 * i + 0] = sw;
    timing[3 * i + 1] = tr;
    timing[3 * i + 2] = acc.result();
}

// fate_prepare's verification of what the bank declares (the lean kernel
// instantiation relies on both): FATE_BANK_NO_QGROUPS => every q_group is -1
// (status bit 1), FATE_BANK_UNIFORM_SPEED => every dev_speed equals device
// 0's (bit 2).
__global__ void fate_validate_bank_kernel(fate_bank b, int* status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int stride = gridDim.x * blockDim.x;
    if (b.flags & FATE_BANK_NO_QGROUPS)
        for (int q = i; q < b.n_queries; q += stride)
            if (b.q_group[q] != -1) atomicOr(status, 1);
    if (b.flags & FATE_BANK_UNIFORM_SPEED)
        for (int d = i; d < b.n_devices; d += stride)
            if (b.dev_speed[d] != b.dev_speed[0]) atomicOr(status, 2);
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

namespace {
std::atomic<unsigned long long> g_queue_used[(V6_QSLOTS - V6_QDIRECT + 63) / 64];
}

int fate_internal_reserve_queue_slot() {
    for (int k = 0; k < V6_QSLOTS - V6_QDIRECT; ++k) {
        const unsigned long long bit = 1ull << (k & 63);
        if (!(g_queue_used[k / 64].fetch_or(bit) & bit)) return V6_QDIRECT + k;
    }
    return -1;  // all reserved: the caller's launches rotate like direct ones
}

void fate_internal_release_queue_slot(int slot) {
    if (slot < V6_QDIRECT || slot >= V6_QSLOTS) return;
    const int k = slot - V6_QDIRECT;
    g_queue_used[k / 64].fetch_and(~(1ull << (k & 63)));
}

void fate_internal_set_queue_slot(int slot) { g_queue_slot_override = slot; }

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

namespace {
int prepare(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
            const fate_derived* out, cudaStream_t s);
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
    nvtxRangePushA("fate_prepare");
    rc = prepare(bank, w, win, out, s);
    nvtxRangePop();
    return rc;
}

}  // extern "C"

namespace {

int prepare(const fate_bank* bank, const fate_weights* w, const fate_windows* win,
            const fate_derived* out, cudaStream_t s) {
    int rc = 0;
    // verification status of the declared bank flags and the op values,
    // read back once at the end (fate_prepare runs once per (bank, weights))
    int* status = nullptr;
    cudaError_t ce = cudaMallocAsync(reinterpret_cast<void**>(&status), sizeof(int), s);
    if (ce != cudaSuccess) return cuda_status("fate_prepare: status buffer");
    cudaMemsetAsync(status, 0, sizeof(int), s);
    struct Free {
        int* p;
        cudaStream_t s;
        ~Free() { cudaFreeAsync(p, s); }
    } free_status{status, s};
    fate_validate_bank_kernel<<<1, 128, 0, s>>>(*bank, status);
    g_launches++;
    if ((rc = cuda_status("fate_validate_bank_kernel"))) return rc;
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
        if (out->tok_vals && out->tok_sums) {
            if (!out->inst_qgroups) return fail(FATE_EINVAL, "token classes need inst_qgroups");
            fate_prepare_tok_kernel<<<blocks, threads, 0, s>>>(*bank, *out);
            g_launches++;
            if ((rc = cuda_status("fate_prepare_tok_kernel"))) return rc;
        }
        if (out->stage_rec) {
            if (!out->split_penalty || !out->inst_qgroups)
                return fail(FATE_EINVAL, "stage records need split_penalty and inst_qgroups");
            fate_prepare_stagerec_kernel<<<blocks, threads, 0, s>>>(*bank, *w, *win, *out);
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
                                            s>>>(*bank, *w, *win, *out, status);
                g_launches++;
                if ((rc = cuda_status("fate_template_fill_kernel"))) return rc;
            }
            if (out->tail_static) {
                const long long nt = n * (bank->n_models + 1);
                fate_prepare_tail_static_kernel<<<(unsigned)((nt + threads - 1) / threads), threads, 0,
                                                  s>>>(*bank, *w, *win, *out, out->tail_static);
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
    int h = 0;
    if ((ce = cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (ce = cudaStreamSynchronize(s)) != cudaSuccess)
        return cuda_status("fate_prepare: status read-back");
    if (h & 1)
        return fail(FATE_EINVAL, "bank declares FATE_BANK_NO_QGROUPS but a query has a prefix group");
    if (h & 2)
        return fail(FATE_EINVAL, "bank declares FATE_BANK_UNIFORM_SPEED but device speeds differ");
    if (h & FATE_PREP_NONFINITE)
        return fail(FATE_EINVAL, "non-finite tail op value (weights x catalog): the exact walk "
                                 "needs finite op values");
    return 0;
}

}  // namespace

extern "C" {

int fate_realized(const fate_bank* bank, const fate_weights* w, const fate_state* st,
                  int32_t scen, int32_t n_tasks, const fate_task* tasks,
                  const int32_t* task_queries, double* timing, void* stream) {
    int rc = check_bank(bank);
    if (rc) return rc;
    if (!w || !st || (n_tasks > 0 && (!tasks || !task_queries || !timing)))
        return fail(FATE_EINVAL, "fate_realized: NULL argument");
    if (scen < 0 || scen >= st->n_scenarios || n_tasks < 0)
        return fail(FATE_EINVAL, "fate_realized: scenario or task count out of range");
    if (n_tasks == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    fate_realized_kernel<<<(n_tasks + 127) / 128, 128, 0, s>>>(*bank, *w, *st, scen, n_tasks,
                                                                tasks, task_queries, timing);
    g_launches++;
    return cuda_status("fate_realized_kernel");
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
#ifdef FATE_AB
    // A/B build only: FATE_SCORE_KERNEL=v5 runs the previous generation
    static const bool v5 = getenv("FATE_SCORE_KERNEL") && !strcmp(getenv("FATE_SCORE_KERNEL"), "v5");
    if (v5) {
        rc = D <= 32 ? launch_v5<1>(bank, w, win, der, st, work, out, s)
                     : launch_v5<2>(bank, w, win, der, st, work, out, s);
        if (rc) return rc;
        g_launches++;
        return cuda_status("fate_score_kernel");
    }
#endif
    rc = D <= 32 ? launch_v6<1>(bank, w, win, der, st, work, out, s)
                 : launch_v6<2>(bank, w, win, der, st, work, out, s);
    if (rc) return rc;
    g_launches++;
    return cuda_status("fate_score_kernel");
}

}  // extern "C"
