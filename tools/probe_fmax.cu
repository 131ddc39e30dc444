// Probe: is max.f64(x, +0.0) bit-identical to Python's max(0.0, x)
// (x > 0.0 ? x : +0.0) for the special values?  nvcc -arch=sm_100a probe_fmax.cu
#include <cstdio>
#include <cstring>
#include <cmath>
#include <cstdint>
__global__ void k(const double* x, double* a, double* b, int n) {
    int i = threadIdx.x;
    if (i < n) {
        double r;
        asm("max.f64 %0, %1, %2;" : "=d"(r) : "d"(x[i]), "d"(0.0));
        a[i] = r;
        b[i] = x[i] > 0.0 ? x[i] : 0.0;
    }
}
int main() {
    double h[16] = {0.0, -0.0, 1.0, -1.0, INFINITY, -INFINITY, NAN, -NAN, 4.9e-324, -4.9e-324,
                    1e308, -1e308, 2.2250738585072014e-308, -2.2250738585072014e-308, 0.5, -0.5};
    double *dx, *da, *db;
    cudaMalloc(&dx, sizeof h); cudaMalloc(&da, sizeof h); cudaMalloc(&db, sizeof h);
    cudaMemcpy(dx, h, sizeof h, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dx, da, db, 16);
    double a[16], b[16];
    cudaMemcpy(a, da, sizeof a, cudaMemcpyDeviceToHost);
    cudaMemcpy(b, db, sizeof b, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 16; ++i) {
        uint64_t ua, ub; memcpy(&ua, &a[i], 8); memcpy(&ub, &b[i], 8);
        if (ua != ub) { ++bad; printf("x=%g max=%016llx tern=%016llx\n", h[i], (unsigned long long)ua, (unsigned long long)ub); }
    }
    printf("{\"mismatches\": %d}\n", bad);
    return 0;
}
