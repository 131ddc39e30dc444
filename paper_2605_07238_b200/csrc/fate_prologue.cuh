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

