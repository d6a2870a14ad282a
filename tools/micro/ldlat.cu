// Microbenchmark: dependent-load latency on B200 for the load flavours the traversal could use
// (single thread, pointer chase over a small L1-resident ring and a 64 MB L2-resident ring).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void chase(const unsigned* __restrict__ next, int iters, unsigned start, long long* out, unsigned* sink) {
    unsigned p = start;
    // warm
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) p = __ldg(next + p);
        if (MODE == 1) p = next[p];
        if (MODE == 2) asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(p) : "l"(next + p));
        if (MODE == 3) asm volatile("ld.global.nc.L1::evict_last.u32 %0, [%1];" : "=r"(p) : "l"(next + p));
    }
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) p = __ldg(next + p);
        if (MODE == 1) p = next[p];
        if (MODE == 2) asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(p) : "l"(next + p));
        if (MODE == 3) asm volatile("ld.global.nc.L1::evict_last.u32 %0, [%1];" : "=r"(p) : "l"(next + p));
    }
    const long long t1 = clock64();
    out[0] = t1 - t0;
    sink[0] = p;
}
int main() {
    const size_t big = 16u << 20;   // 64 MB of uint32
    unsigned* h = new unsigned[big];
    unsigned *d, *sink;
    long long* out;
    cudaMalloc(&d, big * 4);
    cudaMalloc(&sink, 4);
    cudaMalloc(&out, 8);
    for (int ring : {256, 4096, (int)big}) {
        // ring of `ring` elements with a stride of 8 uint32 (one 32-B sector per hop) scattered
        const size_t n = ring;
        for (size_t i = 0; i < n; ++i) h[(i * 8) % big] = (unsigned)((((i + 1) % n) * 8) % big);
        cudaMemcpy(d, h, big * 4, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 4; ++mode) {
            const int iters = 2000;
            if (mode == 0) chase<0><<<1, 1>>>(d, iters, 0, out, sink);
            if (mode == 1) chase<1><<<1, 1>>>(d, iters, 0, out, sink);
            if (mode == 2) chase<2><<<1, 1>>>(d, iters, 0, out, sink);
            if (mode == 3) chase<3><<<1, 1>>>(d, iters, 0, out, sink);
            long long c;
            cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
            printf("ring %9d sectors (%8.1f KB) mode %s: %.1f cycles/load\n", ring, ring * 32 / 1024.0,
                   mode == 0 ? "__ldg      " : mode == 1 ? "plain      " : mode == 2 ? "ld.ca      " : "nc.evict_last",
                   (double)c / iters);
        }
    }
    return 0;
}
