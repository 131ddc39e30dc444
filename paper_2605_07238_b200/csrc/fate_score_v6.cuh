// fate_score_v6.cuh -- warp-per-item scoring kernel, generation 6 (production).
//
// Included by fate_kernels.cu (inside its anonymous namespace), after v5.
//
// Same work decomposition and exactness argument as v5 (one warp per item =
// (scenario, stage v); lane t owns devices t and t+32), with the per-item
// instruction count and the dependent-load depth cut:
//
//  * stage record: every static per-stage scalar the item needs (model,
//    shard bound, group, prompt, parent range, query range, instance offset,
//    eligibility, bound, cost coefficients, switch value, split penalty,
//    instance query-group flag) is one 112-byte record built by the prologue
//    (fate_prepare_stagerec_kernel) and read with seven uniform 16-byte loads,
//    instead of ~20 scalar loads two and three levels deep;
//  * transfer without overrides: beta(L, d) == beta_default for every L != d
//    when the topology has no transfer override (OVR = false), so v's parent
//    walk multiplies by the constant instead of gathering beta rows;
//  * tail op lists from static templates: per (v, level) the prologue lays out
//    the reference's op sequence (costs.py:307-348: per descendant x, its
//    model op, its prefix op, then one entry per parent edge of x other than
//    v).  Model/prefix entries are final; an edge entry carries its parent
//    index and is kept iff that parent is located in the scenario -- so a
//    level's op list is built with one coalesced 16-byte load and one loc
//    gather per 32 entries plus a ballot compaction, no nested parent loops;
//  * op walk with conditional adds in inline PTX.  With two device slots per
//    lane and no overrides each buffered op carries the 64-bit mask of the
//    devices it applies to, and an (op, slot) is one bit test and one
//    predicated DADD (a branch around add.rn.f64, which ptxas keeps as
//    @P DADD); a skipped op leaves the chain untouched.  One slot per lane
//    walks op keys (three predicate-combining setp) with the exact 0/1-factor
//    FMA (skipping = adding +0.0, exact because the chain starts at +0.0 and
//    never becomes -0.0 in round-to-nearest).  Both are v5's chain bit for
//    bit;
//  * op lists compacted and walked in chunks through a small per-warp buffer
//    (order preserved), so shared memory does not grow with the longest
//    template and the L1 carve-out stays large;
//  * shared-memory layout offsets computed once on the host (V6Layout); the
//    warp's slice base comes from a lane-0 shuffle (a uniform register) and
//    the lane id from %laneid, so neither is rematerialised from threadIdx
//    under the register budget.

constexpr int V6_KT = 4;               // shard counts k <= V6_KT: shard sums tabulated
// dynamic classes with a shared-memory row (further classes are computed in
// place).  4, not 8: the smaller per-warp slice moves config 5 to the 132 KB
// carve-out (C5 -1.5 %, C4 -1 % on B200)
constexpr int V6_RCAP = 4;
constexpr int V6_NTOK = 3;             // tabulated partial-hit classes per stage
constexpr int V6_ROW0 = 2 + V6_NTOK;   // first dynamic-row slot
// table slots: 0 = static A (sp = P), 1 = static B (sp = 0), 2..4 = tabulated
// partial hits (sp = P - t), V6_ROW0+ = dynamic rows
constexpr int V6_SLOTS = V6_RCAP + V6_ROW0;
static_assert(V6_SLOTS <= 127, "class slots are stored as int8");
constexpr int V6_KEY_ALWAYS = 999;     // op applied on every device (same-model, prefix)
constexpr int V6_KEY_MODEL = 1000;     // op key >= this: displacement op of model key-1000
constexpr int V6_KEY_SIGMA = 2000;     // OVR edge op: key-2000 = location, val = sigma
constexpr int V6_KEY_NOOP = 0x7ffffff0;  // padding op: matches no device (val +0.0)

// stage record flags
constexpr int V6_CACHE_REUSE = 1;  // cache_reuse and a stage group
constexpr int V6_QGROUPS = 2;      // the instance has queries with prefix groups

struct __align__(16) V6Stage {
    int m, R, gv, Pv;              // model (-1 None), shard bound R(v), group (-1), prompt
    int pa0, pa1, q0, nq;          // parent CSR range, query range
    int stage_off, flags, bound, n_elig;  // instance's first stage, V6_*, slots, |A(v)|
    unsigned long long elig;       // eligible-device mask
    int role, minlvl;              // role row; lowest window-parent level of any horizon
                                   // level (INT_MAX: no window parent)
    double pcoef, pscale;          // prefill coeff (1.0 without model), role prefill scale
    double decode, cplx;           // out * decode coeff * decode scale, role complexity
    double swv, split;             // switch cost if switching, slot>=1 split penalty
};
static_assert(sizeof(V6Stage) == 112, "V6Stage layout");

struct __align__(16) V6Op {
    double val;  // op value (edge entry: -edge_term, or sigma under OVR)
    int pp;      // edge entry: parent stage (global index); -1 = static op
    int key;     // static op key (V6_KEY_ALWAYS / V6_KEY_MODEL + mx)
};
static_assert(sizeof(V6Op) == 16, "V6Op layout");

// Byte offsets of one item's shared-memory slice (host-computed).
struct V6Layout {
    int item_bytes;
    int rows, shard, aware, sw, tr, opval, opmask, key, cslot, rowdev, mmask;
    int ops_cap;  // op-buffer entries (multiple of 8, >= 32)
    int diag;     // -DFATE_AB experiment builds only (FATE_V6_DIAG): 1 = skip the
                  // tail walk, 2 = skip the per-device assembly, 4 = compact the op
                  // lists but skip their walk, 8 = no location gather in the
                  // compaction (timing probes; results are then wrong)
};

// Op buffer: a level's op list is compacted and walked in chunks of at most
// `cap` entries (order preserved), so the shared-memory footprint does not
// grow with the longest op template.  A small buffer leaves more of the SM's
// unified L1/shared array to the L1 cache (the carve-out is sized by the
// resident CTAs' shared memory).  Entry: 8-byte value + 8-byte device mask
// (two device slots per lane, no overrides) or 4-byte key (otherwise).
// Measured on B200: 64 entries (config 5: the resident slices fit the
// 164 KB carve-out, 2 % faster than 128 entries; config 4 at 8 CTAs per SM:
// 1.5 % faster than 96 or 128 entries -- the larger L1 outweighs the extra
// chunk flushes on its long templates).
template <int DPL>
constexpr int v6_opcap_default() { return 64; }
inline int v6_ops_cap(int max_level_ops, int cap) {
    // a multiple of 8: the two-slot walk pads a chunk to 8 ops
    cap &= ~7;
    const int ops8 = ((max_level_ops > 0 ? max_level_ops : 1) + 7) & ~7;
    return ops8 < 32 ? 32 : (ops8 > cap ? cap : ops8);
}

// Static per-warp layouts for the common shapes: every field at a
// compile-time offset from the warp's slice base, so the many shared-memory
// accesses use immediate offsets and the compiler's rematerialisation under
// the register budget is a base re-derivation, not a reload of runtime
// offsets.  Sized per device-slot count for query batches <= 16 (larger
// batches use the runtime layout).  The op buffers (size set by the longest
// op template) follow the struct.
template <int DMX, int BMX>
struct __align__(16) V6SmemT {
    double rows[V6_RCAP * BMX];
    double shard[V6_SLOTS * 2 * V6_KT];
    double aware[(V6_SLOTS + 1) & ~1];
    double sw[DMX];
    double tr[DMX];
    int key[DMX];
    int8_t cslot[DMX];  // class slot per device: -1 .. V6_SLOTS - 1
    int rowdev[V6_RCAP];
};
template <int DPL>
struct V6Static {
    static constexpr int B = 16;  // largest query batch (configs 1-5 use 16 / 32)
    using T = V6SmemT<32 * DPL, B>;
};

template <int DPL>
inline V6Layout v6_layout_static(int max_level_ops, int n_models, bool maskw, int cap) {
    using S = typename V6Static<DPL>::T;
    V6Layout L{};
    const int ops4 = v6_ops_cap(max_level_ops, cap);
    L.ops_cap = ops4;
    L.rows = (int)offsetof(S, rows);
    L.shard = (int)offsetof(S, shard);
    L.aware = (int)offsetof(S, aware);
    L.sw = (int)offsetof(S, sw);
    L.tr = (int)offsetof(S, tr);
    L.key = (int)offsetof(S, key);
    L.cslot = (int)offsetof(S, cslot);
    L.rowdev = (int)offsetof(S, rowdev);
    L.opval = (int)((sizeof(S) + 15) & ~size_t(15));
    L.opmask = L.opval + 8 * ops4;
    L.mmask = L.opmask + (maskw ? 8 : 4) * ops4;
    L.item_bytes = (L.mmask + (maskw ? 8 * n_models : 0) + 15) & ~15;
    return L;
}

inline V6Layout v6_layout(int D, int Bmax, int max_level_ops, int n_models, bool maskw,
                          int cap) {
    V6Layout L{};
    int o = 0;
    const auto take = [&](int n, int sz) {
        const int at = o;
        o += n * sz;
        o = (o + 15) & ~15;
        return at;
    };
    L.rows = take(V6_RCAP * Bmax, 8);
    L.shard = take(V6_SLOTS * 2 * V6_KT, 8);
    L.aware = take(V6_SLOTS, 8);
    L.sw = take(D, 8);
    L.tr = take(D, 8);
    const int ops4 = v6_ops_cap(max_level_ops, cap);  // walked 4 (8) at a time
    L.ops_cap = ops4;
    L.opval = take(ops4, 8);
    L.opmask = take(ops4, maskw ? 8 : 4);
    L.mmask = take(maskw ? n_models : 0, 8);
    L.key = take(D, 4);
    L.cslot = take(D, 1);
    L.rowdev = take(V6_RCAP, 4);
    L.item_bytes = o;
    return L;
}

// ---------------------------------------------------------------------------
// prologue
// ---------------------------------------------------------------------------

// One thread per stage: the stage record (after fate_prepare_stage_kernel,
// which produced split_penalty and inst_qgroups).
__global__ void fate_prepare_stagerec_kernel(fate_bank b, fate_weights w, fate_windows win,
                                             fate_derived der) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= b.n_stages) return;
    V6Stage r;
    const int inst = b.st_inst[g];
    r.m = b.st_model[g];
    r.R = b.st_shard[g];
    r.gv = b.st_group[g];
    r.Pv = b.st_prompt[g];
    r.pa0 = b.par_ptr[g];
    r.pa1 = b.par_ptr[g + 1];
    r.q0 = b.inst_query_off[inst];
    r.nq = b.inst_n_queries[inst];
    r.stage_off = b.inst_stage_off[inst];
    r.flags = (((b.st_flags[g] & FATE_STAGE_CACHE_REUSE) && r.gv != -1) ? V6_CACHE_REUSE : 0) |
              (der.inst_qgroups[inst] ? V6_QGROUPS : 0);
    r.elig = b.st_elig[g];
    r.n_elig = __popcll(r.elig);
    r.bound = (w.ablation & FATE_NO_SHARD) ? 1 : (r.R < r.n_elig ? r.R : r.n_elig);
    r.role = b.st_role[g];
    r.minlvl = 0x7fffffff;
    for (int l = 0; l < win.levels; ++l) {
        const int x = win.wpar_minlvl[(long long)g * win.levels + l];
        r.minlvl = x < r.minlvl ? x : r.minlvl;
    }
    const int ri = r.role;
    r.pcoef = r.m >= 0 ? b.model_prefill[r.m] : 1.0;
    const double dcoef = r.m >= 0 ? b.model_decode[r.m] : 0.0;
    r.decode = (double)b.st_out[g] * dcoef * b.role_decode[ri];
    r.pscale = b.role_prefill[ri];
    r.cplx = b.role_cplx[ri];
    r.swv = r.m >= 0 ? b.model_switch[r.m] * w.switch_x : 0.0;
    r.split = der.split_penalty[g];
    reinterpret_cast<V6Stage*>(der.stage_rec)[g] = r;
}

// Thread per (stage v, level l): length of the op template of the level
// (model op + prefix op + parent edges other than v, per descendant).
__device__ __forceinline__ long long v6_template_walk(const fate_bank& b, const fate_weights& w,
                                                      const fate_windows& win,
                                                      const fate_derived& der, long long vl,
                                                      V6Op* out) {
    const int LV = win.levels;
    const int v = (int)(vl / LV);
    const bool no_loc = w.ablation & FATE_NO_LOCALITY;
    const bool no_pre = w.ablation & FATE_NO_PREFIX;
    const bool no_same = w.ablation & FATE_NO_SAME_MODEL;
    const int mv = b.st_model[v], gv = b.st_group[v], Pv = b.st_prompt[v];
    long long n = 0;
    for (long long i = win.ptr[vl]; i < win.ptr[vl + 1]; ++i) {
        const int x = win.idx[i];
        const int mx = b.st_model[x];
        if (!no_same && mx != -1) {
            if (out) {
                const double bonus = w.lambda_s * b.model_switch[mx] * w.switch_x * w.state_scale;
                const bool same = mx == mv;
                out[n] = V6Op{same ? bonus : -bonus, -1, same ? V6_KEY_ALWAYS : V6_KEY_MODEL + mx};
            }
            ++n;
        }
        const int gx = b.st_group[x];
        if (!no_pre && gx != -1 && gx == gv) {
            if (out) {
                const int Px = b.st_prompt[x];
                const int shared = Pv < Px ? Pv : Px;
                out[n] = V6Op{w.lambda_p * w.kappa_prefix * (double)shared / 1000.0 * w.prefix_x *
                                  w.prefix_scale,
                              -1, V6_KEY_ALWAYS};
            }
            ++n;
        }
        if (!no_loc) {
            for (int e = b.par_ptr[x]; e < b.par_ptr[x + 1]; ++e) {
                const int pp = b.par_idx[e];
                if (pp == v) continue;
                if (out)
                    out[n] = V6Op{b.has_overrides ? der.edge_sigma[e] : -der.edge_term[e], pp, 0};
                ++n;
            }
        }
    }
    return n;
}

__global__ void fate_template_count_kernel(fate_bank b, fate_weights w, fate_windows win,
                                           fate_derived der, long long* counts) {
    const long long vl = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (vl >= (long long)b.n_stages * win.levels) return;
    counts[vl] = v6_template_walk(b, w, win, der, vl, nullptr);
}

// status bit FATE_PREP_NONFINITE: an op value is not finite.  The walk applies
// a skipped op as fma(v, +0.0, a), which equals a only for finite v (the
// reference never evaluates a skipped op), so such a bank is rejected.
constexpr int FATE_PREP_NONFINITE = 4;

__global__ void fate_template_fill_kernel(fate_bank b, fate_weights w, fate_windows win,
                                          fate_derived der, int* status) {
    const long long vl = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (vl >= (long long)b.n_stages * win.levels) return;
    V6Op* out = reinterpret_cast<V6Op*>(der.tmpl) + der.tmpl_ptr[vl];
    const long long n = v6_template_walk(b, w, win, der, vl, out);
    for (long long i = 0; i < n; ++i)
        if (!isfinite(out[i].val)) {
            atomicOr(status, FATE_PREP_NONFINITE);
            break;
        }
}

// ---------------------------------------------------------------------------
// exact quotient tables (universal constants, one copy per device)
// ---------------------------------------------------------------------------
// n / 1000.0 for integer token counts n < V6_DIVTAB (prefix overlap,
// costs.py:145; query_compute's prefill tokens, costs.py:92) and h / n for
// the colocated-parent fraction with n <= V6_COLO_N (costs.py:163).  Filled
// by fate_v6_tables_kernel with the same IEEE division the kernel would
// execute, so a lookup returns the identical double; larger operands divide.
constexpr int V6_DIVTAB = 4096;
constexpr int V6_COLO_N = 64;
__device__ double g_v6_div1000[V6_DIVTAB];
__device__ double g_v6_colo[(V6_COLO_N + 1) * (V6_COLO_N + 2) / 2];

__global__ void fate_v6_tables_kernel() {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < V6_DIVTAB) g_v6_div1000[i] = (double)i / 1000.0;
    if (i <= V6_COLO_N) {
        const int n = i;
        for (int h = 0; h <= n; ++h)
            g_v6_colo[n * (n + 1) / 2 + h] = n > 0 ? (double)h / (double)n : 0.0;
    }
}

// IEEE division kept out of line: for operands the tables and shortcuts do not
// cover (rare), so each call site costs a call instead of an inlined
// division sequence (the kernel is instruction-cache bound on D = 64 banks).
__device__ __noinline__ double v6_div(double a, double b) { return a / b; }

__device__ __forceinline__ double v6_div1000(long long n) {
    return (n >= 0 && n < V6_DIVTAB) ? __ldg(&g_v6_div1000[n]) : v6_div((double)n, 1000.0);
}

// query_compute numerator/denominator order (costs.py:92-94), tabulated /1000
__device__ __forceinline__ double v6_qc_value(long long stage_part, long long query_part,
                                              double pcoef, double pscale, double decode,
                                              double cplx, double speed) {
    const double prefill = v6_div1000(stage_part + query_part) * pcoef * pscale;
    const double x = (prefill + decode) * cplx;
    return speed == 1.0 ? x : v6_div(x, speed);  // x / 1.0 == x exactly
}

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------

// The walk's conditional add.  `@p add.rn.f64` in PTX is if-converted by
// ptxas into an unconditional DADD plus a two-word FSEL (4 SASS per op and
// device slot); a branch around the add is compiled to a predicated DADD
// instead (LOP3 -> P, @!P DADD: 2 SASS per op and slot, against 3 for the
// exact 0/1-factor FMA of the previous generation).  A skipped op leaves the
// accumulator untouched, exactly as the reference, which never evaluates it.

// aff_j += val for every device slot j that the op applies to:
//   key <  1000: applies unless key == device (key 999 = every device)
//   key >= 1000: applies iff key == tgt_j (= 1000 + displaced resident model)
template <int DPL>
__device__ __forceinline__ void v6_apply(double (&aff)[DPL], double val, int k, const int (&d)[DPL],
                                         const int (&tgt)[DPL]) {
    if (DPL == 1) {
        // one device slot: the exact 0/1-factor FMA (fma(v, 1, a) = RN(v + a),
        // fma(v, 0, a) = a for finite v and a chain that is never -0.0) -- on
        // the one-slot kernel the predicated form measured 2 % slower (C5)
        asm("{\n\t// fate-fma01\n\t.reg .pred q, p;\n\t.reg .b32 h;\n\t.reg .f64 f;\n\t"
            "setp.lt.s32 q, %2, 1000;\n\t"
            "setp.ne.and.s32 p, %2, %3, q;\n\t"
            "setp.eq.or.s32 p, %2, %4, p;\n\t"
            "selp.b32 h, 0x3ff00000, 0, p;\n\t"
            "mov.b64 f, {0, h};\n\t"
            "fma.rn.f64 %0, %1, f, %0;\n\t}"
            : "+d"(aff[0])
            : "d"(val), "r"(k), "r"(d[0]), "r"(tgt[0]));
    } else {
        asm volatile("{\n\t.reg .pred q, p, r;\n\t"
                     "setp.lt.s32 q, %3, 1000;\n\t"
                     "setp.ne.and.s32 p, %3, %4, q;\n\t"
                     "setp.eq.or.s32 p, %3, %6, p;\n\t"
                     "setp.ne.and.s32 r, %3, %5, q;\n\t"
                     "setp.eq.or.s32 r, %3, %7, r;\n\t"
                     "@!p bra V6A%=;\n\t"
                     "add.rn.f64 %0, %0, %2;\n\t"
                     "V6A%=:\n\t"
                     "@!r bra V6B%=;\n\t"
                     "add.rn.f64 %1, %1, %2;\n\t"
                     "V6B%=:\n\t}"
                     : "+d"(aff[0]), "+d"(aff[DPL - 1])
                     : "d"(val), "r"(k), "r"(d[0]), "r"(d[DPL - 1]), "r"(tgt[0]),
                       "r"(tgt[DPL - 1]));
    }
}

// Masked op of the non-override walk: the op applies to device t (t + 32)
// iff bit t of lo (hi) is set -- one bit test (LOP3 with a predicate output)
// and one predicated DADD per device slot.
template <int DPL>
__device__ __forceinline__ void v6_apply_m(double (&aff)[DPL], double val, unsigned lo,
                                           unsigned hi, unsigned lanebit) {
    if (DPL == 1) {
        asm("{\n\t.reg .pred p;\n\t.reg .b32 x;\n\t"
            "and.b32 x, %2, %3;\n\t"
            "setp.ne.b32 p, x, 0;\n\t"
            "@p add.rn.f64 %0, %0, %1;\n\t}"
            : "+d"(aff[0])
            : "d"(val), "r"(lo), "r"(lanebit));
    } else {
        asm volatile("{\n\t.reg .pred p, r;\n\t.reg .b32 x, y;\n\t"
                     "and.b32 x, %3, %5;\n\t"
                     "and.b32 y, %4, %5;\n\t"
                     "setp.eq.b32 p, x, 0;\n\t"
                     "setp.eq.b32 r, y, 0;\n\t"
                     "@p bra V6M%=;\n\t"
                     "add.rn.f64 %0, %0, %2;\n\t"
                     "V6M%=:\n\t"
                     "@r bra V6N%=;\n\t"
                     "add.rn.f64 %1, %1, %2;\n\t"
                     "V6N%=:\n\t}"
                     : "+d"(aff[0]), "+d"(aff[DPL - 1])
                     : "d"(val), "r"(lo), "r"(hi), "r"(lanebit));
    }
}

// state.cached_tokens (state.py:110-123) for the stage group, with the first
// two entries loaded speculatively next to the entry count (one dependent load
// level less on the critical path; entries past the count are never used)
__device__ __forceinline__ int v6_cached_tokens(const int32_t* __restrict__ kap,
                                                const int32_t* __restrict__ kn_p, int cap,
                                                int group, int model) {
    if (group == -1) return 0;
    const int4* e = reinterpret_cast<const int4*>(kap);
    const int n = __ldg(kn_p);
    const int4 e0 = __ldg(e);
    const int4 e1 = cap > 1 ? __ldg(e + 1) : e0;
    if (n > 0 && e0.x == group) return (model != -1 && e0.z != model) ? 0 : e0.y;
    if (n > 1 && e1.x == group) return (model != -1 && e1.z != model) ? 0 : e1.y;
#pragma unroll 1
    for (int k = 2; k < n; ++k) {
        const int4 x = __ldg(e + k);
        if (x.x == group) return (model != -1 && x.z != model) ? 0 : x.y;
    }
    return 0;
}

struct V6Item {
    int q0, nq, m, Pv;
    long long dev_row0;
    int cap4;
    double pcoef, pscale, decode, cplx;
};

// cache-aware query_compute of query q on device dv (costs.py:70-94) with the
// device's effective stage part sp
// (QG = false: the bank has no query prefix groups, FATE_BANK_NO_QGROUPS)
template <bool QG>
__device__ __forceinline__ double v6_qc(const fate_bank& b, const fate_state& st,
                                        const V6Item& it, const int* key, int dv, int q) {
    const long long sp = key[dv];
    long long qp = b.q_prompt[it.q0 + q];
    const int qg = QG ? b.q_group[it.q0 + q] : -1;
    if (qg != -1) {
        const long long drow = it.dev_row0 + dv;
        const long long cc = cached_tokens(st.kappa + drow * it.cap4, st.kappa_n[drow], qg, it.m);
        qp = qp - cc > 0 ? qp - cc : 0;
    }
    return v6_qc_value(sp, qp, it.pcoef, it.pscale, it.decode, it.cplx, b.dev_speed[dv]);
}

// ---------------------------------------------------------------------------
// scoring kernel
// ---------------------------------------------------------------------------

// One item (scenario, stage v) by one warp; sb = the warp's shared-memory slice
// (static layout V6Static<DPL>::T when SL, else the runtime layout `lay`).
// UNIT: the weights' multiplicative identities are compile-time constants
// (and, with two device slots, the bank fills all 64) -- no ablation, and lambda_q = lambda_s = lambda_tr = state_scale =
// locality_scale = prefix_scale = transfer_x = prefix_x = kappa_prefix = 1.0
// (checked on the host, v6_unit_weights).  x * 1.0 == x and (-1.0) * x == -x
// bit for bit (signed zeros included), so dropping those products is exact;
// the kernel then carries no ablation branches or selects.
template <int DPL, bool OVR, bool SL, bool QG, bool UNIT>
__device__ __forceinline__ void v6_item(const fate_bank& b, const fate_weights& w,
                                        const fate_windows& win, const fate_derived& der,
                                        const fate_state& st, const fate_work& work,
                                        const fate_out& out, const V6Layout& lay,
                                        const long long item, unsigned char* sb) {
    int t;
    asm("mov.u32 %0, %%laneid;" : "=r"(t));
    using SMEM = typename V6Static<DPL>::T;
    SMEM* const ss = reinterpret_cast<SMEM*>(sb);
    double* const s_rows = SL ? ss->rows : reinterpret_cast<double*>(sb + lay.rows);
    double* const s_shard = SL ? ss->shard : reinterpret_cast<double*>(sb + lay.shard);
    double* const s_aware = SL ? ss->aware : reinterpret_cast<double*>(sb + lay.aware);
    double* const s_sw = SL ? ss->sw : reinterpret_cast<double*>(sb + lay.sw);
    double* const s_tr = SL ? ss->tr : reinterpret_cast<double*>(sb + lay.tr);
    double* const s_opval = reinterpret_cast<double*>(sb + lay.opval);
    uint2* const s_opmask = reinterpret_cast<uint2*>(sb + lay.opmask);
    int* const s_opkey = reinterpret_cast<int*>(sb + lay.opmask);  // key walks: 4-byte keys
    unsigned* const s_mm = reinterpret_cast<unsigned*>(sb + lay.mmask);
    int* const s_key = SL ? ss->key : reinterpret_cast<int*>(sb + lay.key);
    int8_t* const s_cslot = SL ? ss->cslot : reinterpret_cast<int8_t*>(sb + lay.cslot);
    int* const s_rowdev = SL ? ss->rowdev : reinterpret_cast<int*>(sb + lay.rowdev);

    const unsigned FULL = 0xffffffffu;
    // two-slot UNIT banks fill every device slot (D == 64): all lanes live
    // (measured: C4 -2.8 %; the one-slot kernel is 1 % faster without it)
    constexpr bool FULLD = UNIT && DPL == 2;
    const int D = FULLD ? 64 : b.n_devices, LV = win.levels;
    const int Bmax = SL ? V6Static<DPL>::B : b.max_queries;  // row stride of s_rows
    const bool no_loc = !UNIT && (w.ablation & FATE_NO_LOCALITY);
    const bool no_shard = !UNIT && (w.ablation & FATE_NO_SHARD);
    const double lam_q = UNIT ? 1.0 : w.lambda_q, lam_s = UNIT ? 1.0 : w.lambda_s;
    const double lam_tr = UNIT ? 1.0 : w.lambda_tr, st_sc = UNIT ? 1.0 : w.state_scale;
    const double loc_sc = UNIT ? 1.0 : w.locality_scale, pre_sc = UNIT ? 1.0 : w.prefix_scale;
    const double tr_x = UNIT ? 1.0 : w.transfer_x, pre_x = UNIT ? 1.0 : w.prefix_x;
    const double kap_p = UNIT ? 1.0 : w.kappa_prefix;
    const int H = w.eff_horizon;
    const int M1 = b.n_models + 1;

    // ---- item header: work entry, stage record, scenario scalars ----------------------------
    const int s = work.scen[item];
    const int v = work.stage[item];
    const V6Stage* srec = reinterpret_cast<const V6Stage*>(der.stage_rec) + v;
    const int4 h0 = __ldg(reinterpret_cast<const int4*>(srec) + 0);
    const int4 h1 = __ldg(reinterpret_cast<const int4*>(srec) + 1);
    const int4 h2 = __ldg(reinterpret_cast<const int4*>(srec) + 2);
    const longlong2 h3 = __ldg(reinterpret_cast<const longlong2*>(srec) + 3);
    const double2 c0 = __ldg(reinterpret_cast<const double2*>(srec) + 4);
    const double2 c1 = __ldg(reinterpret_cast<const double2*>(srec) + 5);
    const double2 c2 = __ldg(reinterpret_cast<const double2*>(srec) + 6);
    const double clock = st.scen_clock[s];
    const long long loc_off = st.scen_loc_off[s];
    const int done_lvl = st.scen_done_level[s];

    V6Item it;
    it.m = h0.x;
    const int m = it.m, R = h0.y, gv = h0.z;
    it.Pv = h0.w;
    const int pa0 = h1.x, pa1 = h1.y;
    it.q0 = h1.z;
    it.nq = h1.w;
    const int nq = it.nq;
    const int32_t* loc_row = st.loc + loc_off - h2.x;
    const int sflags = h2.y;
    const int bound = h2.z;
    const uint64_t elig = (uint64_t)h3.x;
    const bool cache_reuse = sflags & V6_CACHE_REUSE;
    const bool per_device_rows = QG && (sflags & V6_QGROUPS);
    it.pcoef = c0.x;
    it.pscale = c0.y;
    it.decode = c1.x;
    it.cplx = c1.y;
    const double swv = c2.x;
    it.dev_row0 = (long long)s * D;
    it.cap4 = st.kappa_cap * 4;

    // ---- device rows that everything below needs ----------------------------------------------
    int res0[DPL], dv[DPL];
    bool live[DPL];
    double fr[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        dv[j] = t + 32 * j;
        live[j] = FULLD || dv[j] < D;
        res0[j] = live[j] ? st.residency[it.dev_row0 + dv[j]] : -1;
        fr[j] = live[j] ? st.dev_free[it.dev_row0 + dv[j]] : 0.0;
    }

    // ---- prefetch: located-parent flag per horizon level and the static full tail --------
    const bool do_tail = H > 1;
    unsigned walk_m = 0u;  // bit l: level l has a locality op (needs the op-list walk)
    double tail_full[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) tail_full[j] = 0.0;
    if (do_tail) {
        const double* row = der.tail_sum + (size_t)v * M1;
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            const int r = res0[j];
            tail_full[j] = row[(r != -1 && r != m && r < b.n_models) ? 1 + r : 0];
        }
        if (!no_loc && (int)(h3.y >> 32) <= done_lvl) {
            // a window parent above the scenario's highest located stage cannot be
            // located: levels whose parents all lie above it need no gather (the
            // stage record's minimum over the levels skips the whole loop)
            // A level whose lowest window parent is at or below that level is
            // walked without first checking that a parent is actually located:
            // with no located parent the walk over its op template is the
            // static chain itself (same ops, same order), so the outcome is
            // identical either way and the extra gather pass is saved.
            #pragma unroll 1
            for (int l = 0; l < LV; ++l) {
                const long long vl = (long long)v * LV + l;
                if (win.wpar_minlvl[vl] <= done_lvl) walk_m |= 1u << (l < 31 ? l : 31);
            }
        }
    }
    // static-class sums: lanes 0-5 row_sums (A, B), lanes 6-14 tok_sums (T0..T2)
    const double rsum = t < 6    ? der.row_sums[(size_t)v * 6 + t]
                        : t < 15 ? (der.tok_sums ? der.tok_sums[(size_t)v * 9 + t - 6] : 0.0)
                                 : 0.0;
    const int4 tokv = der.tok_vals ? __ldg(reinterpret_cast<const int4*>(der.tok_vals) + v)
                                   : make_int4(0, 0, 0, 0);

    // ---- P0: per-device stage part, switch; v's parents --------------------------------------
    int cs[DPL], hit[DPL];
    bool ok[DPL];
    double trv[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        ok[j] = live[j] && ((elig >> dv[j]) & 1ull);
        cs[j] = it.Pv;
        hit[j] = 0;
        trv[j] = 0.0;
        if (live[j]) {
            if (cache_reuse) {
                const long long row = it.dev_row0 + dv[j];
                const int c = v6_cached_tokens(st.kappa + row * it.cap4, st.kappa_n + row,
                                               st.kappa_cap, gv, m);
                cs[j] = it.Pv - c > 0 ? it.Pv - c : 0;
            }
            s_key[dv[j]] = cs[j];
            s_sw[dv[j]] = res0[j] == m ? 0.0 : swv;
        }
    }
    // v's parents: lane-parallel fetch, broadcast in ascending order
    // (transfer_cost, costs.py:113-125; colo counts, costs.py:160-165).
    // Under unit weights without overrides the prologue's edge term
    // lambda_tr * beta * sigma * transfer_x * locality_scale is beta * sigma
    // bit for bit (x * 1.0 == x), so the product is read, not recomputed.
    constexpr bool TERM = UNIT && !OVR;
    #pragma unroll 1
    for (int e0 = pa0; e0 < pa1; e0 += 32) {
        const int e = e0 + t;
        int L = -1;
        double sg = 0.0;
        if (e < pa1) {
            L = loc_row[b.par_idx[e]];
            sg = TERM ? der.edge_term[e] : der.edge_sigma[e];
        }
        const int n = pa1 - e0 < 32 ? pa1 - e0 : 32;
        #pragma unroll 1
        for (int i = 0; i < n; ++i) {
            const int Li = __shfl_sync(FULL, L, i);
            const double si = __shfl_sync(FULL, sg, i);
            if (Li < 0) continue;
#pragma unroll
            for (int j = 0; j < DPL; ++j) {
                hit[j] += Li == dv[j];
                if (OVR) {
                    if (live[j] && Li != dv[j])
                        trv[j] += b.beta[(size_t)Li * D + dv[j]] * si;
                } else {
                    if (live[j] && Li != dv[j]) trv[j] += TERM ? si : b.beta_default * si;
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < DPL; ++j)
        if (live[j]) s_tr[dv[j]] = trv[j] * tr_x;
    unsigned long long idle_m = 0ull, ok_m = 0ull;
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        idle_m |= (unsigned long long)__ballot_sync(FULL, ok[j] && fr[j] <= clock + 1e-12) << (32 * j);
        ok_m |= (unsigned long long)__ballot_sync(FULL, ok[j]) << (32 * j);
    }
    __syncwarp();

    // ---- P1: row classes ------------------------------------------------------------------------
    // Devices with equal (sp, speed) share a bit-identical cache-aware row.
    // Under uniform speed without query prefix groups a row depends on sp
    // alone, so each device finds its *static* class by value -- sp == P (A),
    // sp == 0 < P (B), sp == P - t for a tabulated partial-hit count t (T0..T2)
    // -- and only the remaining (dynamic) devices group by __match_any_sync.
    int kb = 0, ki = 0, per = 0, n_rows = 0;
    bool kb_ok = false, ki_ok = false;
    unsigned long long dyn_m = 0ull;
    // the lean instantiation (QG = false) is only launched for uniform-speed banks
    const bool uniform = !QG || (b.flags & FATE_BANK_UNIFORM_SPEED);
    const int n_idle = __popcll(idle_m);
    if (R > 1 && !no_shard) {
        kb = R < 1 + n_idle ? R : 1 + n_idle;
        ki = R < n_idle ? R : n_idle;
    }
    kb_ok = kb >= 2 && kb <= V6_KT;
    ki_ok = ki != kb && ki >= 2 && ki <= V6_KT;
    per = 1 + (kb_ok ? kb : 0) + (ki_ok ? ki : 0);
    const bool stat_ok = uniform && !per_device_rows && kb <= 2 && ki <= 2;
    int rep[DPL];
    bool dyn[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        int sl = -2;  // dynamic
        if (stat_ok) {
            const int c = cs[j], tt = it.Pv - c;
            sl = c == it.Pv                                      ? 0
                 : (c == 0 && it.Pv > 0)                         ? 1
                 : (c > 0 && c < it.Pv && tokv.w > 0 && tt == tokv.x) ? 2
                 : (c > 0 && c < it.Pv && tokv.w > 1 && tt == tokv.y) ? 3
                 : (c > 0 && c < it.Pv && tokv.w > 2 && tt == tokv.z) ? 4
                                                                 : -2;
        }
        if (ok[j] && sl >= 0) s_cslot[dv[j]] = (int8_t)sl;  // static class: slot known now
        dyn[j] = ok[j] && sl == -2;
        unsigned same = __ballot_sync(FULL, dyn[j]);
        if (!per_device_rows) {
            same &= __match_any_sync(FULL, cs[j]);
            if (!uniform) {
                const unsigned long long spd =
                    __double_as_longlong(b.dev_speed[live[j] ? dv[j] : 0]);
                same &= __match_any_sync(FULL, spd);
            }
        } else {
            same &= 1u << t;
        }
        rep[j] = dyn[j] ? 32 * j + __ffs(same) - 1 : -1;
    }
    if (DPL == 2 && !per_device_rows) {
        // a slot-1 dynamic class may already exist among slot-0 devices
        const unsigned reps0 = __ballot_sync(FULL, dyn[0] && rep[0] == dv[0]);
        if (dyn[DPL - 1]) {
            unsigned rr = reps0;
            const double sp = b.dev_speed[dv[DPL - 1]];
            #pragma unroll 1
            while (rr) {
                const int e = __ffs(rr) - 1;
                rr &= rr - 1;
                if (s_key[e] == cs[DPL - 1] && (uniform || b.dev_speed[e] == sp)) {
                    rep[DPL - 1] = e;
                    break;
                }
            }
        }
    }
    // representatives of dynamic classes
#pragma unroll
    for (int j = 0; j < DPL; ++j)
        dyn_m |= (unsigned long long)__ballot_sync(FULL, dyn[j] && rep[j] == dv[j]) << (32 * j);
    const int n_dyn = __popcll(dyn_m);
    n_rows = n_dyn < V6_RCAP ? n_dyn : V6_RCAP;
    // table slot of each device's class: 0 = A, 1 = B, 2..4 = T0..T2,
    // V6_ROW0 + row slot, -1 = direct
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        if (!dyn[j]) continue;
        const int r = __popcll(dyn_m & low_mask(rep[j]));
        if (rep[j] == dv[j] && r < V6_RCAP) s_rowdev[r] = dv[j];
        s_cslot[dv[j]] = (int8_t)(r < V6_RCAP ? V6_ROW0 + r : -1);
    }
    if (stat_ok && t < 15) {
        // lane t holds the sums of static class si = t / 3 (A, B, T0, T1, T2),
        // entry e = t % 3 (full, k=2 shard 0, shard 1); written whether or not
        // a device uses the class
        const int si = t / 3, e = t - 3 * si;
        if (e == 0) {
            s_aware[si] = rsum;
        } else {
            if (kb == 2) s_shard[(si * 2 + 0) * V6_KT + (e - 1)] = rsum;
            if (ki == 2 && ki != kb) s_shard[(si * 2 + 1) * V6_KT + (e - 1)] = rsum;
        }
    }
    __syncwarp();

    // ---- P2: dynamic class rows and sums -------------------------------------------------
    #pragma unroll 1
    for (int p = t; p < n_rows * nq; p += 32) {
        const int r = p / nq, q = p - r * nq;
        s_rows[r * Bmax + q] = v6_qc<QG>(b, st, it, s_key, s_rowdev[r], q);
    }
    __syncwarp();
    #pragma unroll 1
    for (int p = t; p < n_rows * per; p += 32) {
        const int r = p / per;
        int j = p - r * per;
        const double* row = s_rows + r * Bmax;
        const int slot = V6_ROW0 + r;
        PySum acc;
        if (j == 0) {
            #pragma unroll 1
            for (int q = 0; q < nq; ++q) acc.add(row[q]);
            s_aware[slot] = acc.result();
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
            #pragma unroll 1
            for (int q = lo; q < hi; ++q) acc.add(row[q]);
            s_shard[(slot * 2 + kslot) * V6_KT + j] = acc.result();
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
            const int slot = s_cslot[dv[j]];
            if (slot >= 0) {
                here[j] = s_aware[slot];
            } else {
                PySum acc;
                #pragma unroll 1
                for (int q = 0; q < nq; ++q) acc.add(v6_qc<QG>(b, st, it, s_key, dv[j], q));
                here[j] = acc.result();
            }
            if (!have || here[j] < bb) bb = here[j];
            have = true;
        }
        // warp min over lanes with a value (min is order-free)
        double cand = have ? bb : __longlong_as_double(0x7ff0000000000000LL);  // +inf
        const unsigned long long cb = (unsigned long long)__double_as_longlong(cand);
        // (one device slot per lane: C5 -1 %; the two-slot kernel keeps the
        // butterfly, +0.5 % with the reductions)
        if (DPL == 1 && !__any_sync(FULL, (cb >> 63) != 0ull)) {
            // no negative value and no -0.0: the bit patterns of non-negative
            // doubles order like the values (and +inf above all finite ones),
            // so the minimum is two 32-bit warp reductions, high word first
            const unsigned hi = (unsigned)(cb >> 32);
            const unsigned mhi = __reduce_min_sync(FULL, hi);
            const unsigned mlo = __reduce_min_sync(FULL, hi == mhi ? (unsigned)cb : 0xffffffffu);
            bb = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
        } else {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double y = __shfl_xor_sync(FULL, cand, o);
                cand = y < cand ? y : cand;
            }
            bb = cand;
        }
    }

    // ---- P3: tail ---------------------------------------------------------------------------------
    double tail[DPL];
    int dmc[DPL], tgt[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        tail[j] = 0.0;
        dmc[j] = (live[j] && res0[j] != -1 && res0[j] != m && res0[j] < b.n_models) ? res0[j] : -1;
        tgt[j] = dmc[j] >= 0 ? V6_KEY_MODEL + dmc[j] : -2;
    }
#ifdef FATE_AB
    if (lay.diag & 1) walk_m = 0u;
#endif
    if (do_tail && walk_m == 0u) {
        // no locality op anywhere in the horizon: the whole tail is static
#pragma unroll
        for (int j = 0; j < DPL; ++j) tail[j] = tail_full[j];
    } else if (do_tail) {
        const V6Op* tmpl = reinterpret_cast<const V6Op*>(der.tmpl);
        const unsigned lanebit = 1u << t;
        // device masks per op for two device slots per lane; one slot keeps
        // the op keys (three predicate ops per op, no per-item mask table)
        constexpr bool MASKW = !OVR && DPL == 2;
        if (MASKW) {
            // s_mm[2x + j]: devices t + 32j whose displaced resident model is x
            for (int i = t; i < 2 * b.n_models; i += 32) s_mm[i] = 0u;
            __syncwarp();
#pragma unroll
            for (int j = 0; j < DPL; ++j) {
                const unsigned grp = __match_any_sync(FULL, dmc[j]);
                if (dmc[j] >= 0) s_mm[2 * dmc[j] + j] = grp;
            }
            __syncwarp();
        }
        #pragma unroll 1
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
                // op list from the level's template: static entries always, edge
                // entries iff their parent is located (order preserved), compacted
                // and walked in chunks of at most lay.ops_cap entries.  Without
                // overrides each entry carries the 64-bit mask of the devices it
                // applies to (edge: all but the parent's location; displacement of
                // model x: the devices whose displaced resident is x; otherwise
                // all), so a device's predicate is one bit test.
                const long long t0 = der.tmpl_ptr[vl], t1 = der.tmpl_ptr[vl + 1];
#pragma unroll
                for (int j = 0; j < DPL; ++j) aff[j] = 0.0;
                long long j0 = t0;
                // two device slots: 32-bit level-relative indices and
                // branch-free entries (an edge's location gather is
                // predicated, the static masks are selected)
                const V6Op* const lvt = tmpl + t0;
                const int cnt = (int)(t1 - t0);
                int k0 = 0;
                unsigned lt_mask;
                asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt_mask));
                #pragma unroll 1
                while (MASKW ? k0 < cnt : j0 < t1) {
                    // compact template blocks until the buffer could overflow
                    int base = 0;
                    if (MASKW) {
                        #pragma unroll 1
                        do {
                            const int k = k0 + t;
                            bool keep = false;
                            double val = 0.0;
                            unsigned mlo = 0u, mhi = 0u;
                            if (k < cnt) {
                                const int4 raw = __ldg(reinterpret_cast<const int4*>(lvt + k));
                                val = __hiloint2double(raw.y, raw.x);
                                const bool edge = raw.z >= 0;
#ifdef FATE_AB
                                const int L = !edge ? -1
                                              : (lay.diag & 8) ? (raw.z & 1) - 1 + (raw.z & 2)
                                                               : loc_row[raw.z];
#else
                                const int L = edge ? loc_row[raw.z] : -1;
#endif
                                const int mx = raw.w - V6_KEY_MODEL;
                                const bool disp = !edge && raw.w != V6_KEY_ALWAYS;
                                unsigned slo = ~0u, shi = ~0u;
                                if (disp) {
                                    const bool known = mx < b.n_models;
                                    slo = known ? s_mm[2 * mx] : 0u;
                                    shi = known ? s_mm[2 * mx + 1] : 0u;
                                }
                                const unsigned nb = ~(1u << (L & 31));
                                mlo = edge ? (L < 32 ? nb : ~0u) : slo;
                                mhi = edge ? (L >= 32 ? nb : ~0u) : shi;
                                keep = !edge || L >= 0;
                            }
                            const unsigned bal = __ballot_sync(FULL, keep);
                            if (keep) {
                                const int pos = base + __popc(bal & lt_mask);
                                s_opval[pos] = val;
                                s_opmask[pos] = make_uint2(mlo, mhi);
                            }
                            base += __popc(bal);
                            k0 += 32;
                        } while (k0 < cnt && base + 32 <= lay.ops_cap);
                    } else {
                        #pragma unroll 1
                        do {
                            const long long jx = j0 + t;
                            bool keep = false;
                            double val = 0.0;
                            unsigned mlo = 0u, mhi = 0u;
                            if (jx < t1) {
                                const int4 raw = __ldg(reinterpret_cast<const int4*>(tmpl + jx));
                                val = __hiloint2double(raw.y, raw.x);
                                if (raw.z < 0) {
                                    keep = true;
                                    if (!MASKW) {
                                        mlo = (unsigned)raw.w;
                                    } else if (raw.w == V6_KEY_ALWAYS) {
                                        mlo = mhi = ~0u;
                                    } else {
                                        const int mx = raw.w - V6_KEY_MODEL;
                                        if (mx < b.n_models) {
                                            mlo = s_mm[2 * mx];
                                            mhi = s_mm[2 * mx + 1];
                                        }
                                    }
                                } else {
#ifdef FATE_AB
                                    const int L = (lay.diag & 8) ? (raw.z & 1) - 1 + (raw.z & 2)
                                                                 : loc_row[raw.z];
#else
                                    const int L = loc_row[raw.z];
#endif
                                    keep = L >= 0;
                                    if (!MASKW) {
                                        mlo = (unsigned)(OVR ? V6_KEY_SIGMA + L : L);
                                    } else {
                                        mlo = L < 32 ? ~(1u << (L & 31)) : ~0u;
                                        mhi = L >= 32 ? ~(1u << (L & 31)) : ~0u;
                                    }
                                }
                            }
                            const unsigned bal = __ballot_sync(FULL, keep);
                            if (keep) {
                                const int pos = base + __popc(bal & ((1u << t) - 1u));
                                s_opval[pos] = val;
                                if (MASKW)
                                    s_opmask[pos] = make_uint2(mlo, mhi);
                                else
                                    s_opkey[pos] = (int)mlo;
                            }
                            base += __popc(bal);
                            j0 += 32;
                        } while (j0 < t1 && base + 32 <= lay.ops_cap);
                    }
                    // walk the buffered chunk
#ifdef FATE_AB
                    if (lay.diag & 4) {
                        __syncwarp();
                        continue;
                    }
#endif
                    if (MASKW) {
                        // pad to a multiple of 8 with entries that match no device;
                        // walk 8 ops per iteration (four 16-byte mask loads, four
                        // 16-byte value loads; measured: C4 -1.5 % against 4)
                        const int nb8 = (base + 7) & ~7;
                        if (t < nb8 - base) {
                            s_opval[base + t] = 0.0;
                            s_opmask[base + t] = make_uint2(0u, 0u);
                        }
                        __syncwarp();
                        #pragma unroll 1
                        for (int o = 0; o < nb8; o += 8) {
#pragma unroll
                            for (int h = 0; h < 8; h += 4) {
                                const uint4 ma = *reinterpret_cast<const uint4*>(s_opmask + o + h);
                                const uint4 mb = *reinterpret_cast<const uint4*>(s_opmask + o + h + 2);
                                const double2 va = *reinterpret_cast<const double2*>(s_opval + o + h);
                                const double2 vb = *reinterpret_cast<const double2*>(s_opval + o + h + 2);
                                v6_apply_m<DPL>(aff, va.x, ma.x, ma.y, lanebit);
                                v6_apply_m<DPL>(aff, va.y, ma.z, ma.w, lanebit);
                                v6_apply_m<DPL>(aff, vb.x, mb.x, mb.y, lanebit);
                                v6_apply_m<DPL>(aff, vb.y, mb.z, mb.w, lanebit);
                            }
                        }
                    } else if (!OVR) {
                        const int nb4 = (base + 3) & ~3;
                        if (t < nb4 - base) {
                            s_opval[base + t] = 0.0;
                            s_opkey[base + t] = V6_KEY_NOOP;
                        }
                        __syncwarp();
                        #pragma unroll 1
                        for (int o = 0; o < nb4; o += 4) {
                            const int4 k4 = *reinterpret_cast<const int4*>(s_opkey + o);
                            const double2 va = *reinterpret_cast<const double2*>(s_opval + o);
                            const double2 vb = *reinterpret_cast<const double2*>(s_opval + o + 2);
                            v6_apply<DPL>(aff, va.x, k4.x, dv, tgt);
                            v6_apply<DPL>(aff, va.y, k4.y, dv, tgt);
                            v6_apply<DPL>(aff, vb.x, k4.z, dv, tgt);
                            v6_apply<DPL>(aff, vb.y, k4.w, dv, tgt);
                        }
                    } else {
                        __syncwarp();
                        #pragma unroll 1
                        for (int o = 0; o < base; ++o) {
                            const int k = s_opkey[o];
                            const double val = s_opval[o];
#pragma unroll
                            for (int j = 0; j < DPL; ++j) {
                                if (k < V6_KEY_MODEL) {
                                    if (k != dv[j]) aff[j] += val;
                                } else if (k < V6_KEY_SIGMA) {
                                    if (k - V6_KEY_MODEL == dmc[j]) aff[j] += val;
                                } else if (k - V6_KEY_SIGMA != dv[j]) {
                                    aff[j] -= lam_tr *
                                              b.beta[(size_t)(k - V6_KEY_SIGMA) * D +
                                                     (live[j] ? dv[j] : 0)] *
                                              val * tr_x * loc_sc;
                                }
                            }
                        }
                    }
                    __syncwarp();  // op buffer reused by the next chunk / level
                }
            }
#pragma unroll
            for (int j = 0; j < DPL; ++j)
                tail[j] += w.gamma_pow[l + 1] * (aff[j] / (double)n_b + w.demand_coeff * dml);
        }
    }

#ifdef FATE_AB
    if (lay.diag & 2) {
        if (t == 0) out.psi[work.psi_off[item]] = tail[0] + bb;
        return;
    }
#endif
    // ---- P4: per-device assembly ----------------------------------------------------------------
    // Shard bound R = 2 with every class tabulated:
    // a device's second shard always goes to the first idle device other than
    // itself, so each device's shard-1 total sw + tr + shard sum is computed
    // once and the two candidates (first / second idle device) are shuffled --
    // the values and the max are _parallel_benefit's (costs.py:181-201) as in
    // the general loop below.
    bool fast2 = false;
    double t1_e1 = 0.0, t1_e2 = 0.0;
    int e1 = -1, e2 = -1;
    if (R == 2 && !no_shard && kb == 2) {
        int sl[DPL];
        bool all_tab = true;
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            sl[j] = ok[j] ? s_cslot[dv[j]] : 0;
            all_tab = all_tab && sl[j] >= 0;
        }
        fast2 = __all_sync(FULL, all_tab);
        if (fast2) {
            double t1self[DPL];
#pragma unroll
            for (int j = 0; j < DPL; ++j)
                t1self[j] = ok[j] ? s_sw[dv[j]] + s_tr[dv[j]] +
                                        s_shard[(sl[j] * 2 + 0) * V6_KT + 1]
                                  : 0.0;
            e1 = idle_m ? __ffsll((long long)idle_m) - 1 : 0;
            const unsigned long long r2 = idle_m & (idle_m - 1ull);
            e2 = r2 ? __ffsll((long long)r2) - 1 : 0;
            // device e lives in lane e % 32, slot e / 32 (warp-uniform choice)
            t1_e1 = __shfl_sync(FULL, (DPL > 1 && e1 >= 32) ? t1self[DPL - 1] : t1self[0], e1 & 31);
            t1_e2 = __shfl_sync(FULL, (DPL > 1 && e2 >= 32) ? t1self[DPL - 1] : t1self[0], e2 & 31);
        }
    }
    double* psi = out.psi + work.psi_off[item];
    const double split = no_loc ? 0.0 : (bound > 1 ? c2.y : 0.0);
    const bool no_pre = !UNIT && (w.ablation & FATE_NO_PREFIX);
    // One copy of the assembly code for both device slots (the loop is not
    // unrolled; slot values are selected, not indexed): halves this phase's
    // SASS for D > 32, which is instruction-cache bound.
#define V6_PICK(x) (J ? x[DPL - 1] : x[0])
#pragma unroll 1
    for (int j = 0; j < DPL; ++j) {
        const bool J = DPL > 1 && j != 0;
        if (!V6_PICK(live)) continue;
        const int d = V6_PICK(dv);
        const long long orow = item * D + d;
        const double tail_j = V6_PICK(tail);
        const double here_j = V6_PICK(here);
        const int hit_j = V6_PICK(hit);
        if (!V6_PICK(ok)) {
            const double qnan = __longlong_as_double(0x7ff8000000000000LL);
            #pragma unroll 1
            for (int k = 0; k < bound; ++k) psi[(long long)k * D + d] = qnan;
            if (out.sched) out.sched[orow] = qnan;
            if (out.tail) out.tail[orow] = qnan;
            if (out.completion) out.completion[orow] = qnan;
            if (out.timing) {
                out.timing[3 * orow + 0] = qnan;
                out.timing[3 * orow + 1] = qnan;
                out.timing[3 * orow + 2] = qnan;
            }
            continue;
        }
        const double wait = py_max0(V6_PICK(fr) - clock);
        const double sw = s_sw[d];
        const double tr = s_tr[d];
        // 0 / n == +0.0 exactly: divide only when a parent is co-located
        const int npar = pa1 - pa0;
        const double colo =
            (npar > 0 && hit_j > 0)
                ? (npar <= V6_COLO_N ? __ldg(&g_v6_colo[npar * (npar + 1) / 2 + hit_j])
                                     : v6_div((double)hit_j, (double)npar))
                : 0.0;

        // prefix_overlap_thousands (costs.py:127-145), integer-exact
        long long tokens = 0;
        if (cache_reuse) tokens += it.Pv - V6_PICK(cs);  // min(cached, P) = P - sp
        if (per_device_rows) {
            const long long row = it.dev_row0 + d;
            const int32_t* kap = st.kappa + row * it.cap4;
            const int kn = st.kappa_n[row];
            #pragma unroll 1
            for (int q = 0; q < nq; ++q) {
                const int qg = b.q_group[it.q0 + q];
                if (qg == -1) continue;
                const long long c = cached_tokens(kap, kn, qg, m);
                const long long qp = b.q_prompt[it.q0 + q];
                tokens += c < qp ? c : qp;
            }
        }
        const double prefix =
            kap_p * (tokens == 0 ? 0.0 : v6_div1000(tokens)) * pre_x;

        // _parallel_benefit (costs.py:181-201)
        const double full_total = sw + tr + here_j;
        double parallel = 0.0;
        if (R > 1 && !no_shard) {
            const bool self_idle = (idle_m >> d) & 1ull;
            const int others = n_idle - (self_idle ? 1 : 0);
            const int k = R < 1 + others ? R : 1 + others;
            if (k > 1 && fast2) {
                const int slot = s_cslot[d];
                const double tot0 = s_sw[d] + s_tr[d] + s_shard[(slot * 2 + 0) * V6_KT + 0];
                const double tot1 = d == e1 ? t1_e2 : t1_e1;
                const double worst = tot1 > tot0 ? tot1 : tot0;
                const double overhead = w.shard_overhead_frac * here_j * (double)(k - 1);
                parallel = py_max0(full_total - worst - overhead);
            } else if (k > 1) {
                const int kslot = (k == kb && kb_ok) ? 0 : 1;
                const bool tab = kslot == 0 || (k == ki && ki_ok);
                unsigned long long rest = idle_m & ~(1ull << d);
                double worst = 0.0;
                #pragma unroll 1
                for (int i = 0; i < k; ++i) {
                    int dev = d;
                    if (i > 0) {
                        dev = __ffsll((long long)rest) - 1;
                        rest &= rest - 1;
                    }
                    const int slot = s_cslot[dev];
                    double ssum;
                    if (tab && slot >= 0) {
                        ssum = s_shard[(slot * 2 + kslot) * V6_KT + i];
                    } else {
                        int lo, hi;
                        shard_range(nq, k, i, &lo, &hi);
                        PySum acc;
                        #pragma unroll 1
                        for (int q = lo; q < hi; ++q)
                            acc.add(slot >= V6_ROW0 ? s_rows[(slot - V6_ROW0) * Bmax + q]
                                                    : v6_qc<QG>(b, st, it, s_key, dev, q));
                        ssum = acc.result();
                    }
                    const double tot = s_sw[dev] + s_tr[dev] + ssum;
                    if (i == 0 || tot > worst) worst = tot;
                }
                const double overhead = w.shard_overhead_frac * here_j * (double)(k - 1);
                parallel = py_max0(full_total - worst - overhead);
            }
        }

        // sched_score (costs.py:210-231)
        const double tr_s = no_loc ? 0.0 : tr;
        const double colo_s = no_loc ? 0.0 : colo;
        const double prefix_s = no_pre ? 0.0 : prefix;
        const double par_s = no_shard ? 0.0 : parallel;
        const double S = -lam_q * wait - lam_s * sw * st_sc
                         - lam_tr * tr_s * loc_sc
                         + w.lambda_c * colo_s * loc_sc
                         + w.lambda_p * prefix_s * pre_sc + w.lambda_r * par_s;

        if (out.sched) out.sched[orow] = S;
        if (out.tail) out.tail[orow] = tail_j;
        if (out.completion) out.completion[orow] = wait + full_total;
        if (out.timing) {  // ShardTiming(switch_s, transfer_s, compute_s), costs.py:398-414
            out.timing[3 * orow + 0] = sw;
            out.timing[3 * orow + 1] = tr;
            out.timing[3 * orow + 2] = here_j;
        }
        psi[d] = S + tail_j;

        // _marginal_shard_score (costs.py:249-279)
        if (bound > 1) {
            const double hv = here_j > bb ? here_j : bb;
            const double overhead = w.shard_overhead_frac * bb;
            const double tr_m = no_loc ? 0.0 : tr;
            #pragma unroll 1
            for (int k = 1; k < bound; ++k) {
                // x / 1 == x and x / 2 == x * 0.5 exactly (both correctly rounded x/2)
                const double q1 = k == 1 ? bb : v6_div(bb, (double)k);
                const double q2 = k == 1 ? hv * 0.5 : v6_div(hv, (double)(k + 1));
                const double reduction = q1 - q2;
                psi[(long long)k * D + d] = w.lambda_r * (reduction - overhead) -
                                            lam_q * wait - lam_s * sw * st_sc -
                                            lam_tr * (tr_m + split) * loc_sc;
            }
        }
    }
#undef V6_PICK
}

// Work distribution: a persistent grid (every resident CTA slot once) whose
// warps pull items from a global ticket counter (ticket sizes: see below),
// until the batch is exhausted: a warp that finishes a cheap item takes the
// next one instead of holding a CTA slot idle (item costs vary several-fold
// with the number of walked horizon levels, and consecutive items -- stages
// of one scenario in index order -- have correlated costs).  Each launch uses
// its own counter slot and the last warp of a launch resets the slot to zero,
// so a captured graph replays without a reset node.  A work list may bring
// its own counter (fate_work.queue; runtime.DeviceWork passes one per
// (work list, stream)), so launches in flight never share one however many
// there are.  Without it: slots [0, V6_QDIRECT) rotate over direct
// fate_score calls; the rest are reserved per host pipeline compute stream
// (fate_internal_reserve_queue_slot), so a captured pipeline graph never
// shares a counter with a concurrent direct launch.
constexpr int V6_QSLOTS = 256;
constexpr int V6_QDIRECT = 128;
__device__ unsigned int g_v6_queue[2 * V6_QSLOTS];  // per slot: next ticket, warps done

template <int DPL, bool OVR, bool SL, int MINB, bool QG, bool UNIT>
__global__ void __launch_bounds__(128, MINB) fate_score_v6_kernel(fate_bank b, fate_weights w,
                                                                  fate_windows win,
                                                                  fate_derived der, fate_state st,
                                                                  fate_work work, fate_out out,
                                                                  V6Layout lay, int qslot,
                                                                  int fetch) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int t = threadIdx.x & 31;
    const int wi = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    unsigned int* q = work.queue ? work.queue : g_v6_queue + 2 * qslot;
    const long long n = work.n_items;
    unsigned char* sb = smem_raw + lay.item_bytes * wi;
    // fetch > 0: fixed items per ticket; fetch == 0: guided -- a ticket takes
    // 1/(4 * warps) of what the warp last saw remaining (at least one), so
    // early tickets are large (few atomics) and late ones single items (tail
    // balance)
    const unsigned nw = gridDim.x * (blockDim.x >> 5);
    const float inv_share = 0.25f / (float)nw;
    // first ticket without the atomic: warp g takes items [g f0, (g+1) f0)
    // (f0 = the launch's static first share, else one ticket); the counter
    // hands out the items from nw f0 on (an atomic round trip less on every
    // warp's critical path -- it matters when each warp scores only a few
    // items, i.e. small shards)
    // fetch = items per ticket | (items of the static first ticket << 8)
    const unsigned first_take = (unsigned)fetch >> 8;
    fetch &= 0xff;
    const unsigned f0 = first_take ? first_take : (fetch > 0 ? (unsigned)fetch : 1u);
    const unsigned gw = blockIdx.x * (blockDim.x >> 5) + (unsigned)wi;
    bool first = true;
    long long seen = 0;
    for (;;) {
        long long take = fetch;
        if (fetch == 0) {  // heuristic size: a float estimate is enough
            take = (long long)((float)(n - seen) * inv_share);
            take = take < 1 ? 1 : (take > 16 ? 16 : take);
        }
        long long i;
        if (first) {
            take = f0;
            i = (long long)gw * f0;
            first = false;
        } else {
            unsigned int k = 0;
            if (t == 0) k = atomicAdd(q, (unsigned)take);
            i = (long long)__shfl_sync(0xffffffffu, k, 0) + (long long)nw * f0;
        }
        seen = i + take;
        if (i >= n) break;
        const long long i1 = i + take < n ? i + take : n;
#pragma unroll 1
        for (long long it = i; it < i1; ++it) {
            v6_item<DPL, OVR, SL, QG, UNIT>(b, w, win, der, st, work, out, lay, it, sb);
            __syncwarp();  // the slice is reused by the next item
        }
    }
    if (t == 0) {
        __threadfence();
        const unsigned done = atomicAdd(q + 1, 1u);
        if (done == gridDim.x * (blockDim.x >> 5) - 1) {  // last warp of the launch
            q[0] = 0u;
            q[1] = 0u;
            __threadfence();
        }
    }
}
