// issue_probe.cu -- diagnostic: the secondary ceilings of the scoring kernel,
// measured ("FP64 non-FMA instruction throughput ... measure with
// a DADD/DMUL microbenchmark on the box").
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/issue_probe.cu -o tools/bin/issue_probe
//   tools/bin/issue_probe > profiles/r01_issue_probe.json
//
// Every kernel runs 148 x 16 CTAs of 128 threads (64 warps per SM), each
// thread a loop of independent chains; warp instructions are counted from the
// loop body (checked against cuobjdump -sass: the unrolled body is exactly
// the listed ops plus the loop's ISETP + BRA + IADD, which the count
// includes).  Timed with CUDA events after a warm-up launch; one JSON line.
//   int_issue : LOP3 chains              -> warp-instruction issue ceiling
//   dadd      : add.rn.f64 chains        -> FP64 add pipe ceiling
//   walk      : fate_score_v6's device-mask walk loop (64 devices = two
//               slots per lane): warp-level ops (one op over 64 devices) / s
#include <cuda_runtime.h>

#include <cstdio>

constexpr int ITERS = 4096;

__global__ void k_int(unsigned* out, unsigned seed) {
    unsigned a0 = seed ^ threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4,
             a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
#pragma unroll 1
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            asm volatile("lop3.b32 %0, %0, %8, %9, 0x96;\n\t"
                         "lop3.b32 %1, %1, %8, %9, 0x96;\n\t"
                         "lop3.b32 %2, %2, %8, %9, 0x96;\n\t"
                         "lop3.b32 %3, %3, %8, %9, 0x96;\n\t"
                         "lop3.b32 %4, %4, %8, %9, 0x96;\n\t"
                         "lop3.b32 %5, %5, %8, %9, 0x96;\n\t"
                         "lop3.b32 %6, %6, %8, %9, 0x96;\n\t"
                         "lop3.b32 %7, %7, %8, %9, 0x96;"
                         : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3), "+r"(a4), "+r"(a5), "+r"(a6),
                           "+r"(a7)
                         : "r"(seed), "r"(i));
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}

__global__ void k_dadd(double* out, double v) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
#pragma unroll 1
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            asm volatile("add.rn.f64 %0, %0, %8;\n\t"
                         "add.rn.f64 %1, %1, %8;\n\t"
                         "add.rn.f64 %2, %2, %8;\n\t"
                         "add.rn.f64 %3, %3, %8;\n\t"
                         "add.rn.f64 %4, %4, %8;\n\t"
                         "add.rn.f64 %5, %5, %8;\n\t"
                         "add.rn.f64 %6, %6, %8;\n\t"
                         "add.rn.f64 %7, %7, %8;"
                         : "+d"(a0), "+d"(a1), "+d"(a2), "+d"(a3), "+d"(a4), "+d"(a5), "+d"(a6),
                           "+d"(a7)
                         : "d"(v));
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// the v6 device-mask walk loop for two device slots: 4 ops per iteration,
// masks and values from shared memory (two 16-byte mask loads, two 16-byte
// value loads), exactly the production loop's shape
template <int MODE>
__global__ void k_walk(double* out, const uint2* gmask, const double* gval) {
    __shared__ __align__(16) uint2 sm[4][64];
    __shared__ __align__(16) double sv[4][64];
    const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
    for (int k = t; k < 64; k += 32) {
        sm[w][k] = gmask[k];
        sv[w][k] = gval[k];
    }
    __syncwarp();
    double a0 = 0.0, a1 = 0.0;
    const unsigned lb = 1u << t;
#pragma unroll 1
    for (int i = 0; i < ITERS; ++i) {
        const int o = (i * 4) & 63;
        const uint4 ma = *reinterpret_cast<const uint4*>(&sm[w][o]);
        const uint4 mb = *reinterpret_cast<const uint4*>(&sm[w][o + 2]);
        const double2 va = *reinterpret_cast<const double2*>(&sv[w][o]);
        const double2 vb = *reinterpret_cast<const double2*>(&sv[w][o + 2]);
        const unsigned ml[4] = {ma.x, ma.z, mb.x, mb.z}, mh[4] = {ma.y, ma.w, mb.y, mb.w};
        const double vv[4] = {va.x, va.y, vb.x, vb.y};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (MODE == 0)  // production: predicated add (ptxas: DADD + FSEL pair)
                asm("{\n\t.reg .pred p, q;\n\t.reg .b32 x, y;\n\t"
                    "and.b32 x, %2, %4;\n\t"
                    "and.b32 y, %3, %4;\n\t"
                    "setp.ne.b32 p, x, 0;\n\t"
                    "setp.ne.b32 q, y, 0;\n\t"
                    "@p add.rn.f64 %0, %0, %5;\n\t"
                    "@q add.rn.f64 %1, %1, %5;\n\t}"
                    : "+d"(a0), "+d"(a1)
                    : "r"(ml[r]), "r"(mh[r]), "r"(lb), "d"(vv[r]));
            else if (MODE == 1)  // 0/1 factor: select the high word of 1.0, one DFMA
                asm("{\n\t.reg .pred p, q;\n\t.reg .b32 x, y, hx, hy;\n\t.reg .f64 f, g;\n\t"
                    "and.b32 x, %2, %4;\n\t"
                    "and.b32 y, %3, %4;\n\t"
                    "setp.ne.b32 p, x, 0;\n\t"
                    "setp.ne.b32 q, y, 0;\n\t"
                    "selp.b32 hx, 0x3ff00000, 0, p;\n\t"
                    "selp.b32 hy, 0x3ff00000, 0, q;\n\t"
                    "mov.b64 f, {0, hx};\n\t"
                    "mov.b64 g, {0, hy};\n\t"
                    "fma.rn.f64 %0, %5, f, %0;\n\t"
                    "fma.rn.f64 %1, %5, g, %1;\n\t}"
                    : "+d"(a0), "+d"(a1)
                    : "r"(ml[r]), "r"(mh[r]), "r"(lb), "d"(vv[r]));
            else  // select the addend (value or +0.0), then add
                asm("{\n\t.reg .pred p, q;\n\t.reg .b32 x, y;\n\t.reg .f64 u, w;\n\t"
                    "and.b32 x, %2, %4;\n\t"
                    "and.b32 y, %3, %4;\n\t"
                    "setp.ne.b32 p, x, 0;\n\t"
                    "setp.ne.b32 q, y, 0;\n\t"
                    "selp.f64 u, %5, 0d0000000000000000, p;\n\t"
                    "selp.f64 w, %5, 0d0000000000000000, q;\n\t"
                    "add.rn.f64 %0, %0, u;\n\t"
                    "add.rn.f64 %1, %1, w;\n\t}"
                    : "+d"(a0), "+d"(a1)
                    : "r"(ml[r]), "r"(mh[r]), "r"(lb), "d"(vv[r]));
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const int blocks = sms * 16, threads = 128;
    const double warps = (double)blocks * threads / 32.0;
    void* buf;
    cudaMalloc(&buf, (size_t)blocks * threads * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        return best * 1e-3;
    };
    // loop body warp instructions per iteration (ops + ISETP/BRA/IADD of the loop)
    const double s_int = time([&] { k_int<<<blocks, threads>>>((unsigned*)buf, 7u); });
    const double s_dadd = time([&] { k_dadd<<<blocks, threads>>>((double*)buf, 1e-3); });
    uint2* gmask;
    double* gval;
    cudaMalloc(&gmask, 64 * sizeof(uint2));
    cudaMalloc(&gval, 64 * sizeof(double));
    {
        uint2 hm[64];
        double hv[64];
        for (int k = 0; k < 64; ++k) {
            hm[k] = make_uint2(~(1u << (k % 32)), k % 5 ? ~0u : 0x0f0f0f0fu);
            hv[k] = 1e-3 * (k + 1);
        }
        cudaMemcpy(gmask, hm, sizeof(hm), cudaMemcpyHostToDevice);
        cudaMemcpy(gval, hv, sizeof(hv), cudaMemcpyHostToDevice);
    }
    const double s_walk = time([&] { k_walk<0><<<blocks, threads>>>((double*)buf, gmask, gval); });
    const double s_walk_fma =
        time([&] { k_walk<1><<<blocks, threads>>>((double*)buf, gmask, gval); });
    const double s_walk_sel =
        time([&] { k_walk<2><<<blocks, threads>>>((double*)buf, gmask, gval); });
    const double it = (double)ITERS;
    const double int_inst = warps * it * (32 + 3);
    const double dadd_inst = warps * it * 32;
    const double walk_ops = warps * it * 4;  // ops per iteration (each over 64 devices)
    const double peak_issue = (double)sms * 4 * clk_khz * 1e3;
    printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, "
           "\"issue_peak_ginst_s_at_attr_clock\": %.2f, "
           "\"int_issue_ginst_s\": %.2f, \"dadd_ginst_s\": %.2f, \"dadd_gflops\": %.1f, "
           "\"walk_warp_ops_g_per_s\": %.2f, \"walk_fma01_warp_ops_g_per_s\": %.2f, "
           "\"walk_seladd_warp_ops_g_per_s\": %.2f, "
           "\"seconds\": {\"int\": %.6f, \"dadd\": %.6f, \"walk\": %.6f}}\n",
           sms, clk_khz / 1e3, peak_issue / 1e9, int_inst / s_int / 1e9, dadd_inst / s_dadd / 1e9,
           dadd_inst * 32 / s_dadd / 1e9, walk_ops / s_walk / 1e9, walk_ops / s_walk_fma / 1e9,
           walk_ops / s_walk_sel / 1e9, s_int, s_dadd, s_walk);
    cudaFree(buf);
    return 0;
}
