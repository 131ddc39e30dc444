// fate_prologue.cuh -- static tail tables of fate_prepare (once per (bank,
// weights)).  Included by fate_kernels.cu inside its anonymous namespace.
//
// The tail (costs.py:281-352) of a candidate depends on the scenario only
// through its locality ops (located parents of the window's descendants) and
// the displacement class of the device (the resident model it would
// displace).  Without locality ops the per-level affinity chain is static per
// (stage, level, displacement class), and so is the whole tail; the scoring
// kernel reads these tables whenever the scenario leaves a level (or the
// whole horizon) without located window parents.


// Prologue: static tail level terms (no locality op applied) per (stage,
// level, displacement class): class 0 = not displacing, class 1+m = displaces
// with resident model m.  The affinity chain (costs.py:307-331) is folded
// into the level's term gamma**l * (affinity/len(bucket) + demand_coeff *
// demand) (costs.py:349-351) with the reference's operations, so a scoring
// launch adds the stored term for a level without located window parents
// (bit-identical to computing it there); 0 for an empty bucket.
__global__ void fate_prepare_tail_static_kernel(fate_bank b, fate_weights w, fate_windows win,
                                                fate_derived der, double* tail_static) {
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
    const long long n = win.ptr[vl + 1] - win.ptr[vl];
    const int l = (int)(vl - (long long)v * LV);
    tail_static[t] =
        n > 0 ? w.gamma_pow[l + 1] * (aff / (double)n + w.demand_coeff * der.demand[vl]) : 0.0;
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
        total += der.tail_static[vl * M1 + c];  // the level's term
    }
    der.tail_sum[t] = total;
}


// Partial-hit prefix classes (one thread per stage v).  A device's cached
// stage-group tokens come from _seed_prefixes (state.py:236-247): a
// keep_cache stage of the group seeds its prompt proxy and _merge_entry keeps
// the maximum, so the cache-aware stage part is P(v) - P(u) for a keep_cache
// stage u of v's group (or 0 / P(v), the static classes of row_sums).  Up to
// three such token counts t (the largest, 0 < t < P(v)) get their row sums
// tabulated -- full batch and the two k=2 shards, Neumaier like the kernel
// (costs.py:257, :404-405) -- so the scoring kernel can skip the dynamic-row
// phase for them.  Tabulated only under uniform speed and for instances
// without query prefix groups (the cases where a row depends on sp alone).
__global__ void fate_prepare_tok_kernel(fate_bank b, fate_derived der) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= b.n_stages) return;
    int tv[3] = {0, 0, 0};
    int nt = 0;
    const int inst = b.st_inst[g];
    const int gv = b.st_group[g], Pv = b.st_prompt[g];
    const bool ok = (b.flags & FATE_BANK_UNIFORM_SPEED) && gv != -1 &&
                    (b.st_flags[g] & FATE_STAGE_CACHE_REUSE) && !der.inst_qgroups[inst];
    if (ok) {
        const int u0 = b.inst_stage_off[inst], u1 = u0 + b.inst_n_stages[inst];
        for (int u = u0; u < u1; ++u) {
            if (b.st_group[u] != gv || !(b.st_flags[u] & FATE_STAGE_KEEP_CACHE)) continue;
            const int P = b.st_prompt[u];
            if (P <= 0 || P >= Pv || P == tv[0] || P == tv[1] || P == tv[2]) continue;
            // keep the three largest distinct values, descending
            if (nt == 3 && P <= tv[2]) continue;
            int k = nt < 3 ? nt++ : 2;  // fill, or replace the smallest
            while (k > 0 && tv[k - 1] < P) {
                tv[k] = tv[k - 1];
                --k;
            }
            tv[k] = P;
        }
    }
    der.tok_vals[(size_t)g * 4 + 0] = tv[0];
    der.tok_vals[(size_t)g * 4 + 1] = tv[1];
    der.tok_vals[(size_t)g * 4 + 2] = tv[2];
    der.tok_vals[(size_t)g * 4 + 3] = nt;
    const int m = b.st_model[g], r = b.st_role[g];
    const double pcoef = m >= 0 ? b.model_prefill[m] : 1.0;
    const double dcoef = m >= 0 ? b.model_decode[m] : 0.0;
    const double pscale = b.role_prefill[r], cplx = b.role_cplx[r];
    const double decode = (double)b.st_out[g] * dcoef * b.role_decode[r];
    const int q0 = b.inst_query_off[inst], nq = b.inst_n_queries[inst];
    const int half = nq / 2 + (nq % 2);
    for (int k = 0; k < 3; ++k) {
        double all = 0.0, s0 = 0.0, s1 = 0.0;
        if (k < nt) {
            const long long sp = Pv - tv[k];
            PySum a, x0, x1;
            for (int q = 0; q < nq; ++q) {
                const double x = qc_value(sp, b.q_prompt[q0 + q], pcoef, pscale, decode, cplx,
                                          b.dev_speed[0]);
                a.add(x);
                if (q < half) x0.add(x);
                else x1.add(x);
            }
            all = a.result();
            s0 = x0.result();
            s1 = x1.result();
        }
        der.tok_sums[(size_t)g * 9 + 3 * k + 0] = all;
        der.tok_sums[(size_t)g * 9 + 3 * k + 1] = s0;
        der.tok_sums[(size_t)g * 9 + 3 * k + 2] = s1;
    }
}
