// Microbenchmark: GPU stores into mapped pinned host memory (po_render_host's direct image
// writes) -- PCIe efficiency of the store pattern.  7.68 MB = one 800x800 fp32 RGB image.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int W = 800, H = 800;
// pattern 0: linear float4 stores, 32 lanes x 16 B = 512 B contiguous per warp instruction
__global__ void k_linear(float4* out, int n4) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x)
        out[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}
// pattern 1: 8x4 warp tiles, each row of a tile 96 B (24 lanes x float4), as store_tile_rgb
__global__ void k_tile(float* out) {
    const int lane = threadIdx.x & 31;
    const int tiles = (W / 8) * (H / 4);
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < tiles; t += (gridDim.x * blockDim.x) >> 5) {
        const int tx = t % (W / 8), ty = t / (W / 8);
        const int r = lane / 6, q = lane % 6;
        if (lane < 24)
            reinterpret_cast<float4*>(out + ((size_t)(ty * 4 + r) * W + tx * 8) * 3)[q] = make_float4(1.f, 2.f, 3.f, 4.f);
    }
}
// pattern 2: 16x16 blocks, a warp writes two 192-B block rows per instruction (24 lanes) -- rows
// of the 16-px block, 64-B aligned
__global__ void k_block(float* out) {
    const int lane = threadIdx.x & 31;
    const int rowsegs = (W / 16) * H;   // 192-B row segments
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < rowsegs / 2; t += (gridDim.x * blockDim.x) >> 5) {
        const int seg = 2 * t + (lane >= 12 ? 1 : 0), q = lane % 12;
        const int bx = seg % (W / 16), y = seg / (W / 16);
        if (lane < 24)
            reinterpret_cast<float4*>(out + ((size_t)y * W + bx * 16) * 3)[q] = make_float4(1.f, 2.f, 3.f, 4.f);
    }
}
int main() {
    float* h;
    const size_t bytes = (size_t)W * H * 3 * 4;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    float* d;
    cudaHostGetDevicePointer(&d, h, 0);
    float* dev;
    cudaMalloc(&dev, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int dst = 0; dst < 2; ++dst) {
        float* o = dst ? dev : d;
        for (int p = 0; p < 3; ++p) {
            for (int grid : {148 * 2, 148 * 8}) {
                float best = 1e9;
                for (int it = 0; it < 20; ++it) {
                    cudaEventRecord(a);
                    if (p == 0) k_linear<<<grid, 256>>>(reinterpret_cast<float4*>(o), (int)(bytes / 16));
                    if (p == 1) k_tile<<<grid, 256>>>(o);
                    if (p == 2) k_block<<<grid, 256>>>(o);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (it > 2 && ms < best) best = ms;
                }
                printf("%s pattern %s grid %d: %.1f us = %.1f GB/s\n", dst ? "device" : "host-mapped",
                       p == 0 ? "linear-512B" : (p == 1 ? "tile-96B" : "block-192B"), grid, best * 1e3,
                       bytes / (best * 1e-3) / 1e9);
            }
        }
    }
    return 0;
}
