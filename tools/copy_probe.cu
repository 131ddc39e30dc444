// copy_probe.cu -- diagnostic: PCIe copy-engine behaviour for the host pipeline.
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/copy_probe.cu -o /tmp/copy_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void spin(long long cycles) {
    long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
}

int main() {
    const size_t IN = 18350080, OUT = 45777664;
    char *hi, *ho, *di, *dout;
    cudaHostAlloc(&hi, IN, 0);
    cudaHostAlloc(&ho, OUT, 0);
    cudaMalloc(&di, IN);
    cudaMalloc(&dout, OUT);
    cudaStream_t a, b, c;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking);
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    std::vector<cudaEvent_t> ev(64);
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    auto run = [&](const char* name, auto body) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(t0, 0);
            body();
            cudaEventRecord(t1, 0);
            cudaEventSynchronize(t1);
            float ms;
            cudaEventElapsedTime(&ms, t0, t1);
            if (rep == 2) printf("%-40s %8.1f us\n", name, ms * 1e3);
        }
    };
    auto join = [&](cudaStream_t s, int k) {
        cudaEventRecord(ev[k], s);
        cudaStreamWaitEvent(0, ev[k], 0);
    };
    auto fork = [&](cudaStream_t s, int k) {
        cudaEventRecord(ev[k], 0);
        cudaStreamWaitEvent(s, ev[k], 0);
    };
    run("h2d 18MB (legacy stream)", [&] { cudaMemcpyAsync(di, hi, IN, cudaMemcpyHostToDevice, 0); });
    run("d2h 46MB (legacy stream)", [&] { cudaMemcpyAsync(ho, dout, OUT, cudaMemcpyDeviceToHost, 0); });
    run("h2d || d2h (2 streams)", [&] {
        fork(a, 0); fork(b, 1);
        cudaMemcpyAsync(di, hi, IN, cudaMemcpyHostToDevice, a);
        cudaMemcpyAsync(ho, dout, OUT, cudaMemcpyDeviceToHost, b);
        join(a, 2); join(b, 3);
    });
    for (int n : {4, 8, 16}) {
        char name[96];
        snprintf(name, sizeof name, "chunked x%d h2d->spin->d2h (3 role streams)", n);
        run(name, [&] {
            fork(a, 0); fork(b, 1); fork(c, 2);
            const size_t ci = IN / n, co = OUT / n;
            for (int k = 0; k < n; ++k) {
                cudaMemcpyAsync(di + k * ci, hi + k * ci, ci, cudaMemcpyHostToDevice, a);
                cudaEventRecord(ev[3 + 2 * k], a);
                cudaStreamWaitEvent(c, ev[3 + 2 * k], 0);
                spin<<<1, 32, 0, c>>>(60000);  // ~30 us
                cudaEventRecord(ev[4 + 2 * k], c);
                cudaStreamWaitEvent(b, ev[4 + 2 * k], 0);
                cudaMemcpyAsync(ho + k * co, dout + k * co, co, cudaMemcpyDeviceToHost, b);
            }
            join(a, 60); join(b, 61); join(c, 62);
        });
        snprintf(name, sizeof name, "chunked x%d h2d->spin->d2h (1 stream/chunk rr2)", n);
        run(name, [&] {
            fork(a, 0); fork(b, 1);
            const size_t ci = IN / n, co = OUT / n;
            for (int k = 0; k < n; ++k) {
                cudaStream_t s = (k & 1) ? b : a;
                cudaMemcpyAsync(di + k * ci, hi + k * ci, ci, cudaMemcpyHostToDevice, s);
                spin<<<1, 32, 0, s>>>(60000);
                cudaMemcpyAsync(ho + k * co, dout + k * co, co, cudaMemcpyDeviceToHost, s);
            }
            join(a, 60); join(b, 61);
        });
    }
    // does a full-GPU kernel slow a concurrent H2D / D2H?
    run("spin full GPU ~300us alone", [&] { spin<<<148 * 8, 128>>>(600000); });
    run("h2d 18MB || full-GPU spin", [&] {
        fork(a, 0); fork(b, 1);
        cudaMemcpyAsync(di, hi, IN, cudaMemcpyHostToDevice, a);
        spin<<<148 * 8, 128, 0, b>>>(600000);
        join(a, 2); join(b, 3);
    });
    run("d2h 46MB || full-GPU spin", [&] {
        fork(a, 0); fork(b, 1);
        cudaMemcpyAsync(ho, dout, OUT, cudaMemcpyDeviceToHost, a);
        spin<<<148 * 8, 128, 0, b>>>(600000);
        join(a, 2); join(b, 3);
    });
    run("h2d 18MB as 3 copies || full-GPU spin", [&] {
        fork(a, 0); fork(b, 1);
        cudaMemcpyAsync(di, hi, 6000000, cudaMemcpyHostToDevice, a);
        cudaMemcpyAsync(di + 6000000, hi + 6000000, 8000000, cudaMemcpyHostToDevice, a);
        cudaMemcpyAsync(di + 14000000, hi + 14000000, IN - 14000000, cudaMemcpyHostToDevice, a);
        spin<<<148 * 8, 128, 0, b>>>(600000);
        join(a, 2); join(b, 3);
    });
    return 0;
}
