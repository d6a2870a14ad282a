// CUDA kernels of the PlenOctree hot path for sm_100a.
//
//   k_render        a1..a6   one thread per pixel, warp = 8x4 pixel tile, CTA = 16x16
//   k_render_rays   a2..a6   one thread per ray (optionally double-precision totals, aux)
//   k_backward      a7+a8    two passes per ray in ONE thread: pass 1 (or aux)
//                            gives the total sum_k c_k w_k, pass 2 re-traverses with a
//                            double prefix and scatter-adds per-leaf gradients
//   k_trace/k_stats          parity / measurement visitors over the same traversal
//   k_l2_loss, k_sgd         Eq. (3) gradient helper and the SGD update
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "kernels.h"
#include "traverse.cuh"

namespace po {

// ---------------------------------------------------------------------------------------
// Visitors
// ---------------------------------------------------------------------------------------
template <int DEG, bool F16>
struct FwdVisitor {
    const DevTree& tr;
    float Y[ShDim<DEG>::B];
    float T, gamma;
    float C[3];
    __device__ FwdVisitor(const DevTree& t, const float d[3], float g) : tr(t), T(1.f), gamma(g) {
        ray_basis<DEG>(t, d, Y);
        C[0] = C[1] = C[2] = 0.f;
    }
    __device__ __forceinline__ void on_node() {}
    __device__ __forceinline__ bool shade(uint32_t idx, float t0, float t1) {
        const float st = __ldg(tr.sigma + idx);
        float z[3];
        sh_dot<DEG, F16>(tr, idx, Y, z);   // row loads issued together with the sigma load
        if (!(st > 0.f)) return true;      // sigma = (sigma~)_+ = 0: alpha = 0 (reading Q10)
        const Absorb a = absorb(T, st, __fsub_rn(t1, t0));
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) C[ch] = fmaf(a.w, sigmoidf_(z[ch]), C[ch]);
        T = a.Tn;
        return !(T < gamma);
    }
    __device__ __forceinline__ bool on_leaf(uint32_t idx, float t0, float t1) { return shade(idx, t0, t1); }
};

// Stored pass-1 segments (po_segments): record k of ray i = two float4 at (k n + i) * 2:
// (leaf index bits, delta, w, T_{i+1}), (c_r, c_g, c_b, 0) -- every value pass 2 needs, so it
// replays the segments instead of re-traversing the tree.  count[i] = number of sigma~ > 0
// segments, max_seg + 1 when they did not fit (pass 2 then re-traverses that ray).
struct SegOut {
    float4* __restrict__ rec;
    int32_t* __restrict__ count;
    int64_t n;
    int32_t max_seg;
};

// Forward with the colour sum accumulated in double (pass 1 of the backward).
template <int DEG, bool F16>
struct TotalVisitor {
    const DevTree& tr;
    float Y[ShDim<DEG>::B];
    float T, gamma;
    double C[3];
    uint32_t lo, hi;   // [lo, hi]: index span of the sigma~ > 0 leaves composited (po_backward_plan)
    float4* __restrict__ seg;   // this ray's first record (SegOut) or null
    int64_t seg_stride;         // 2 n float4 between consecutive records of a ray
    int32_t nseg, max_seg;      // max_seg < 0: no segment bookkeeping
    __device__ TotalVisitor(const DevTree& t, const float d[3], float g)
        : tr(t), T(1.f), gamma(g), lo(0xFFFFFFFFu), hi(0u), seg(nullptr), seg_stride(0), nseg(0), max_seg(-1) {
        ray_basis<DEG>(t, d, Y);
        C[0] = C[1] = C[2] = 0.0;
    }
    __device__ __forceinline__ void on_node() {}
    __device__ __forceinline__ bool on_leaf(uint32_t idx, float t0, float t1) {
        const float st = __ldg(tr.sigma + idx);
        float z[3];
        sh_dot<DEG, F16>(tr, idx, Y, z);   // row loads in flight together with sigma
        if (!(st > 0.f)) return true;
        lo = min(lo, idx);
        hi = max(hi, idx);
        const float delta = __fsub_rn(t1, t0);
        const Absorb a = absorb(T, st, delta);
        float c[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            c[ch] = sigmoidf_(z[ch]);
            C[ch] += (double)a.w * (double)c[ch];
        }
        if (max_seg >= 0) {
            if (nseg < max_seg) {
                float4* r = seg + (int64_t)nseg * seg_stride;
                r[0] = make_float4(__uint_as_float(idx), delta, a.w, a.Tn);
                r[1] = make_float4(c[0], c[1], c[2], 0.f);
            }
            nseg = min(nseg + 1, max_seg + 1);
        }
        T = a.Tn;
        return !(T < gamma);
    }
};

// Pass 2: prefix P_i = sum_{k<=i} c_k w_k (double); S_i = total - P_i;
// dL/dsigma~_i = [sigma~_i > 0] delta_i sum_ch g_ch (c_i,ch T_{i+1} - S_i,ch)
// dL/dk_i,b,ch = g_ch w_i c_i,ch (1 - c_i,ch) Y_b
template <int DEG, bool F16>
struct GradVisitor {
    const DevTree& tr;
    float Y[ShDim<DEG>::B];
    float T, gamma;
    double P[3], Ctot[3];
    float g[3];
    float* __restrict__ grad_sigma;
    float* __restrict__ grad_sh;
    __device__ GradVisitor(const DevTree& t, const float d[3], float gm, float* gs, float* gk)
        : tr(t), T(1.f), gamma(gm), grad_sigma(gs), grad_sh(gk) {
        ray_basis<DEG>(t, d, Y);
        P[0] = P[1] = P[2] = 0.0;
    }
    __device__ __forceinline__ void on_node() {}
    __device__ __forceinline__ bool on_leaf(uint32_t idx, float t0, float t1) {
        const float st = __ldg(tr.sigma + idx);
        float z[3], c[3];
        sh_dot<DEG, F16>(tr, idx, Y, z);   // row loads in flight together with sigma
        if (!(st > 0.f)) return true;   // ReLU gate: w = 0 and dsigma = 0
        const float delta = __fsub_rn(t1, t0);
        const Absorb a = absorb(T, st, delta);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) c[ch] = sigmoidf_(z[ch]);
        seg(idx, delta, a.w, a.Tn, c);
        T = a.Tn;
        return !(T < gamma);
    }
    // gradient of one sigma~ > 0 segment from its forward values (w_i, T_{i+1}, c_i): used by
    // the re-traversal above and by the stored-segment replay (identical arithmetic)
    __device__ __forceinline__ void seg(uint32_t idx, float delta, float w, float Tn, const float c[3]) {
        double acc = 0.0;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            P[ch] += (double)w * (double)c[ch];
            acc += (double)g[ch] * ((double)c[ch] * (double)Tn - (Ctot[ch] - P[ch]));
        }
        atomicAdd(grad_sigma + idx, (float)((double)delta * acc));
        constexpr int B = ShDim<DEG>::B;
        constexpr int NE = 3 * B;
        float gz[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) gz[ch] = g[ch] * w * c[ch] * (1.f - c[ch]);
        float* row = grad_sh + (size_t)idx * NE;
        if constexpr (NE % 4 == 0) {
#pragma unroll
            for (int j = 0; j < NE / 4; ++j) {
                float v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = gz[(4 * j + q) % 3] * Y[(4 * j + q) / 3];
                float* p = row + 4 * j;
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v[0]), "f"(v[1]),
                             "f"(v[2]), "f"(v[3])
                             : "memory");
            }
        } else {
#pragma unroll
            for (int el = 0; el < NE; ++el) atomicAdd(row + el, gz[el % 3] * Y[el / 3]);
        }
    }
};

// NEXT f4 (P:638 depth map, P:468 alpha map; reading Q34): alpha = 1 - T_stop and the
// expected depth sum_i w_i (t_in + t_out) / 2 over the composited segments.  sigma~ only:
// no SH rows are read.
struct DepthVisitor {
    const DevTree& tr;
    float T, gamma, D;
    __device__ __forceinline__ void on_node() {}
    __device__ __forceinline__ bool on_leaf(uint32_t idx, float t0, float t1) {
        const float st = __ldg(tr.sigma + idx);
        if (!(st > 0.f)) return true;
        const Absorb a = absorb(T, st, __fsub_rn(t1, t0));
        D = fmaf(a.w, 0.5f * (t0 + t1), D);
        T = a.Tn;
        return !(T < gamma);
    }
};

// NEXT f1, visibility filtering (reading Q33): per-leaf maximum over rays of the
// ray weight 1 - exp(-sigma delta) for every leaf composited before termination.  alpha >= 0,
// so the IEEE bit pattern orders like the value and atomicMax on it is a float max.
struct MaxAlphaVisitor {
    const DevTree& tr;
    float T, gamma;
    unsigned* __restrict__ max_alpha;
    __device__ __forceinline__ void on_node() {}
    __device__ __forceinline__ bool on_leaf(uint32_t idx, float t0, float t1) {
        const float st = __ldg(tr.sigma + idx);
        if (!(st > 0.f)) return true;   // alpha = 0: the maximum is unchanged
        const Absorb a = absorb(T, st, __fsub_rn(t1, t0));
        atomicMax(max_alpha + idx, __float_as_uint(__fsub_rn(1.0f, a.e)));
        T = a.Tn;
        return !(T < gamma);
    }
};

struct TraceVisitor {
    const DevTree& tr;
    float T, gamma;
    int32_t* ids;
    int32_t max_leaves, count, nodes;
    __device__ __forceinline__ void on_node() { ++nodes; }
    __device__ __forceinline__ bool on_leaf(uint32_t idx, float t0, float t1) {
        if (count < max_leaves) ids[count] = (int32_t)idx;
        ++count;
        const float st = __ldg(tr.sigma + idx);
        if (!(st > 0.f)) return true;
        T = absorb(T, st, __fsub_rn(t1, t0)).Tn;
        return !(T < gamma);
    }
};

struct StatsVisitor {
    const DevTree& tr;
    float T, gamma;
    unsigned long long leaves, sh_rows, nodes, boxes, leaf_level_boxes;
    __device__ __forceinline__ void on_node() { ++nodes; }
    __device__ __forceinline__ void on_box(int shift) {
        ++boxes;
        leaf_level_boxes += (shift == 0);
    }
    __device__ __forceinline__ bool on_leaf(uint32_t idx, float t0, float t1) {
        ++leaves;
        const float st = __ldg(tr.sigma + idx);
        if (!(st > 0.f)) return true;
        ++sh_rows;
        T = absorb(T, st, __fsub_rn(t1, t0)).Tn;
        return !(T < gamma);
    }
};

// ---------------------------------------------------------------------------------------
// a1: pixel -> ray (reading Q5)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void camera_ray_of(const float c[16], int px, int py, float o[3], float d[3]) {
    // explicit round-to-nearest ops (no FMA contraction): the ray is reproducible bit for bit
    // by any IEEE fp32 implementation of the same expression (po_camera_rays exports it)
    const float dx = __fdiv_rn(__fsub_rn(__fadd_rn((float)px, 0.5f), c[14]), c[12]);
    const float dy = -__fdiv_rn(__fsub_rn(__fadd_rn((float)py, 0.5f), c[15]), c[13]);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        d[k] = __fsub_rn(__fadd_rn(__fmul_rn(c[k * 4 + 0], dx), __fmul_rn(c[k * 4 + 1], dy)), c[k * 4 + 2]);
        o[k] = c[k * 4 + 3];
    }
}

__device__ __forceinline__ void camera_ray(const po_camera* __restrict__ cams, int view, int px, int py, float o[3],
                                           float d[3]) {
    const float* cm = reinterpret_cast<const float*>(cams + view);
    float c[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) c[k] = __ldg(cm + k);
    camera_ray_of(c, px, py, o, d);
}

__global__ void __launch_bounds__(256) k_camera_rays(const po_camera* __restrict__ cams, int n_cams, int W, int H,
                                                     float* __restrict__ rays) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)W * H;
    if (i >= per * n_cams) return;
    const int view = (int)(i / per);
    const int p = (int)(i - (int64_t)view * per);
    float o[3], d[3];
    camera_ray(cams, view, p % W, p / W, o, d);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        rays[i * 6 + k] = o[k];
        rays[i * 6 + 3 + k] = d[k];
    }
}

cudaError_t launch_camera_rays(const po_camera* cams, int n_cams, int W, int H, float* rays, cudaStream_t s) {
    const int64_t n = (int64_t)W * H * n_cams;
    if (n == 0) return cudaSuccess;
    k_camera_rays<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(cams, n_cams, W, H, rays);
    return cudaGetLastError();
}

// Store an 8x4 warp tile's RGB (lane = pixel: x = lane & 7, y = lane >> 3).  When the tile is
// whole and rows are 16-B aligned (W % 4 == 0), the 4 rows x 96 contiguous bytes go out as
// 24 float4 stores assembled with shuffles (whole 16-B words also when `out` is pinned host
// memory written over PCIe by po_render_host); otherwise (edge tiles, odd W, a buffer not
// 16-B aligned) 3 scalar stores per pixel.
__device__ __forceinline__ void store_tile_rgb(float* __restrict__ out, size_t row0, int W, int H, int px0, int py0,
                                               const float C[3]) {
    const int lane = threadIdx.x & 31;
    if (px0 + 8 <= W && py0 + 4 <= H && (W & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0) {
        const int r = lane / 6, q = lane - 6 * (lane / 6);   // lanes 0..23: row r, float4 q of 6
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int f = 4 * q + k, src = 8 * r + f / 3, ch = f % 3;
            const float c0 = __shfl_sync(0xFFFFFFFFu, C[0], src & 31);
            const float c1 = __shfl_sync(0xFFFFFFFFu, C[1], src & 31);
            const float c2 = __shfl_sync(0xFFFFFFFFu, C[2], src & 31);
            v[k] = ch == 0 ? c0 : (ch == 1 ? c1 : c2);
        }
        if (lane < 24)
            reinterpret_cast<float4*>(out + ((row0 + py0 + r) * W + px0) * 3)[q] = make_float4(v[0], v[1], v[2], v[3]);
    } else {
        const int px = px0 + (lane & 7), py = py0 + (lane >> 3);
        if (px < W && py < H) {
            float* p = out + ((row0 + py) * W + px) * 3;
            p[0] = C[0];
            p[1] = C[1];
            p[2] = C[2];
        }
    }
}

// CTA = 16x16 pixels = 8 warps, each warp an 8x4 pixel tile (warp-coherent ray packets).
__device__ __forceinline__ bool tile_pixel(int W, int H, int& px, int& py) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    px = blockIdx.x * 16 + (warp & 1) * 8 + (lane & 7);
    py = blockIdx.y * 16 + (warp >> 1) * 4 + (lane >> 3);
    return px < W && py < H;
}

// Persistent render: grid = #SMs x resident CTAs.  Work = 16x16-pixel blocks (8 warp tiles
// of 8x4 pixels, raster order over views x block rows x block columns), claimed from a
// global counter one block per CTA "slot".  Inside a CTA the warps take warp tiles from a
// shared ticket counter: ticket k -> slot k/8, tile k%8; the warp drawing tile 0 of a slot
// claims that slot's block and publishes it.  So a CTA's warps stay on one or two
// neighbouring blocks (rays of a CTA share nodes and leaves in L1) while no warp ever waits
// for a slower one, and the uneven per-block cost (misses vs. surface hits) is balanced
// across SMs with no tail wave.  The last CTA to finish resets the global counters
// (work[0] = next block, work[1] = finished CTAs) for the next launch on the stream.
constexpr int kSlotRing = 16;

// Cost-ordered hand-out (DESIGN.md §6.1 v13).  A frame ends with its slowest warp tiles (grazing
// rays along the surface shell); handing their blocks out first makes them start at t = 0
// instead of in the second wave.  Consecutive frames of a moving camera have nearly the same
// per-block costs, so each single-view launch measures them (max SM cycles of a block's warp
// tiles) and its last CTA rewrites the stream's order table for the next launch: a counting
// sort over 256 log2-spaced cost buckets (2^(1/8) apart), costliest first.  Pixel values do not
// depend on the order.  key8 = shared scratch of >= nb bytes.
// With split_k > 0 the split_k costliest blocks are expanded into split_f positions each
// (entry = block | (8 | sub-block) << 28), placed first; order[-1] = number of positions.
// With zip the blocks after the split ones alternate costliest / cheapest (po_render_host).
__device__ __forceinline__ void reorder_blocks(unsigned* __restrict__ cost, unsigned* __restrict__ order, unsigned nb,
                                               uint8_t* __restrict__ key8, int split_k, int split_f, bool zip) {
    __shared__ unsigned hist[256];
    __shared__ unsigned top[64];
    const unsigned K = (split_f > 1) ? min((unsigned)split_k, min(nb, 64u)) : 0u;
    const unsigned extra = K * (unsigned)(split_f - 1);
    const unsigned tid = threadIdx.x;
    for (unsigned i = tid; i < 256u; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    for (unsigned i = tid; i < nb; i += blockDim.x) {
        const unsigned c = atomicExch(cost + i, 0u);   // read and reset for the next launch
        const int lg = c == 0u ? 0 : min(255, (int)(8.f * __log2f((float)c)));
        const unsigned k = 255u - (unsigned)lg;         // costliest -> bucket 0
        key8[i] = (uint8_t)k;
        atomicAdd(&hist[k], 1u);
    }
    __syncthreads();
    if (tid < 32u) {   // exclusive scan of the 256 buckets, 8 per lane
        unsigned v[8], sum = 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            v[j] = hist[tid * 8u + j];
            sum += v[j];
        }
        unsigned x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if ((int)tid >= o) x += y;
        }
        unsigned base = x - sum;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            hist[tid * 8u + j] = base;
            base += v[j];
        }
    }
    __syncthreads();
    const unsigned n2 = nb - K;   // blocks after the split ones
    for (unsigned i = tid; i < nb; i += blockDim.x) {
        unsigned r = atomicAdd(&hist[key8[i]], 1u);   // rank, costliest first
        if (zip && r >= K) {
            const unsigned q = r - K;
            r = K + (q < (n2 + 1u) / 2u ? 2u * q : 2u * (n2 - 1u - q) + 1u);
        }
        order[extra + r] = i;
    }
    if (K > 0u) {
        __syncthreads();
        if (tid < K) top[tid] = order[extra + tid];
        __syncthreads();
        for (unsigned i = tid; i < K * (unsigned)split_f; i += blockDim.x)
            order[i] = top[i / (unsigned)split_f] | ((8u | (i % (unsigned)split_f)) << 28);
    }
    if (tid == 0) order[-1] = nb + extra;
}

template <int DEG, bool F16, int MINB, int OPT>
__global__ void __launch_bounds__(256, MINB) k_render(DevTree tr, const po_camera* __restrict__ cams, int n_cams, int W,
                                                int H, RenderOpts opt, float* __restrict__ out,
                                                unsigned* __restrict__ work, const unsigned* __restrict__ order,
                                                unsigned long long* __restrict__ timeline) {
    PO_DECLARE_STACK(stk);
    __shared__ unsigned s_ticket;
    __shared__ unsigned s_block[kSlotRing];
    __shared__ unsigned s_pub[kSlotRing];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_ticket = 0;
    if (threadIdx.x < kSlotRing) s_pub[threadIdx.x] = 0xFFFFFFFFu;
    __syncthreads();
    const unsigned bx_n = (unsigned)(W + 15) >> 4, by_n = (unsigned)(H + 15) >> 4;
    const unsigned per_view = bx_n * by_n;
    // blocks of this shard per view: hand-out positions k = local * shard_count + shard_index
    const unsigned sc = (unsigned)opt.shard_count, si = (unsigned)opt.shard_index;
    const unsigned local_per_view = (per_view + sc - 1u - si) / sc;
    // cost-ordered single-view launches: order[-1] = hand-out positions (split blocks count
    // split_f times, reorder_blocks); otherwise blocks of this shard x views
    const unsigned total = opt.blk_cost != nullptr ? __ldg(order - 1) : local_per_view * (unsigned)n_cams;
    while (true) {
        // hand-off through shared-memory atomics (ordered by the block fences): the warp that
        // opens a slot claims the block and publishes it; the other 7 wait for the flag.  The
        // control flow is warp-uniform (lane 0 does the atomics, every branch decision is
        // shuffled to the whole warp), and waiting warps sleep between polls.
        unsigned k = 0;
        if (lane == 0) k = atomicAdd(&s_ticket, 1u);
        k = __shfl_sync(0xffffffffu, k, 0);
        const unsigned slot = k >> 3, sub = k & 7u;
        if (sub == 0) {
            if (lane == 0) {
                atomicExch(&s_block[slot % kSlotRing], atomicAdd(work, 1u));
                __threadfence_block();
                atomicExch(&s_pub[slot % kSlotRing], slot);
            }
        } else {
            while (true) {
                unsigned p = 0;
                if (lane == 0) p = atomicAdd(&s_pub[slot % kSlotRing], 0u);
                if (__shfl_sync(0xffffffffu, p, 0) == slot) break;
                __nanosleep(64);
            }
            __threadfence_block();
        }
        unsigned blk = 0;
        if (lane == 0) blk = atomicAdd(&s_block[slot % kSlotRing], 0u);
        blk = __shfl_sync(0xffffffffu, blk, 0);
        if (blk >= total) break;
        const unsigned view = opt.blk_cost != nullptr ? 0u : blk / local_per_view;
        unsigned rem = opt.blk_cost != nullptr ? blk : (blk - view * local_per_view) * sc + si;   // hand-out position
        if (order != nullptr) rem = __ldg(order + rem);   // block hand-out order (see launch_render)
        const unsigned split = rem >> 28;                 // 0, or 8 | sub-block of a split block
        rem &= 0x0FFFFFFFu;
        unsigned long long t_tile = 0;
        if (timeline != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_tile));
        const unsigned c_tile = opt.blk_cost != nullptr ? (unsigned)clock() : 0u;
        const int by = (int)(rem / bx_n), bx = (int)(rem - (unsigned)by * bx_n);
        int px, py;
        bool act = true;
        if (split == 0u) {   // 8x4-pixel warp tile
            px = bx * 16 + (int)(sub & 1u) * 8 + (lane & 7);
            py = by * 16 + (int)(sub >> 1) * 4 + (lane >> 3);
        } else {             // 4 x (8/F) pixels, lanes < 32/F (sub-block q of 16 x 16/F pixels)
            const int F = opt.split_f, q = (int)(split & 7u);
            px = bx * 16 + (int)(sub & 3u) * 4 + (lane & 3);
            py = by * 16 + q * (16 / F) + (int)(sub >> 2) * (8 / F) + (lane >> 2);
            act = lane < 32 / F;
        }
        float C[3] = {opt.bg[0], opt.bg[1], opt.bg[2]};
        if (act && px < W && py < H) {
            float o[3], d[3];
            if (opt.cam_inline) {   // single view passed by value (po_render_host): no H2D copy
                float c[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) c[k] = opt.cam[k];
                camera_ray_of(c, px, py, o, d);
            } else {
                camera_ray(cams, (int)view, px, py, o, d);
            }
            RayState r;
            if (ray_setup(tr, o, d, r)) {
#ifdef PO_DIAG
                if constexpr ((OPT & kOptProbeNoShade) != 0) {
                    // measurement probe only (PO_RENDER_OPT=64, wrong colours): the traversal and
                    // transmittance without any SH row, to size a traversal/shading split
                    struct Probe {
                        const DevTree& tr;
                        float T, gamma;
                        __device__ __forceinline__ void on_node() {}
                        __device__ __forceinline__ bool on_leaf(uint32_t idx, float t0, float t1) {
                            const float st = __ldg(tr.sigma + idx);
                            if (!(st > 0.f)) return true;
                            T = absorb(T, st, __fsub_rn(t1, t0)).Tn;
                            return !(T < gamma);
                        }
                    } v{tr, 1.f, opt.gamma};
                    traverse<kOptLean>(tr, r, v, stk);
                    C[0] = C[1] = C[2] = v.T;
                } else
#endif
                {
                    FwdVisitor<DEG, F16> v(tr, r.d, opt.gamma);
                    traverse<OPT & (kOptLean | kOptGrid)>(tr, r, v, stk);
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) C[ch] = fmaf(v.T, opt.bg[ch], v.C[ch]);
                }
            }
        }
        if (split == 0u) {
            store_tile_rgb(out, (size_t)view * H, W, H, bx * 16 + (int)(sub & 1u) * 8, by * 16 + (int)(sub >> 1) * 4, C);
        } else if (act && px < W && py < H) {
            float* p = out + ((size_t)py * W + px) * 3;
            p[0] = C[0];
            p[1] = C[1];
            p[2] = C[2];
        }
        if (opt.blk_cost != nullptr) {   // this tile's cost (SM cycles) for the next launch's order
            __syncwarp();
            // a split block's tiles have 1/F of the rays: scaled so it keeps its rank.  The cost
            // goes to the block AND its 8 neighbours (lanes 0..8): the next view sees the costly
            // silhouette a block or so away (c3: 234-259 us with the previous view's own block
            // costs, 210-211 us dilated, 212 us with the view's own costs; DESIGN.md §6.1 v15)
            // (neighbours get the unscaled cycles, so a split block keeps its own top rank)
            const unsigned c = __shfl_sync(0xFFFFFFFFu, (unsigned)clock() - c_tile, 0);
            const int nx = bx + lane % 3 - 1, ny = by + lane / 3 - 1;
            if (lane < 9 && nx >= 0 && ny >= 0 && nx < (int)bx_n && ny < (int)by_n)
                atomicMax(opt.blk_cost + (unsigned)ny * bx_n + (unsigned)nx,
                          lane == 4 && split ? c * (unsigned)opt.split_f : c);
        }
        if (opt.band_done != nullptr) {   // this tile's pixels are stored: count it for its band
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicAdd(opt.band_done + by / opt.band_rows, 1ull);
        }
        if (timeline != nullptr) {   // measurement mode (po_render_timeline): one record per warp tile
            __syncwarp();
            if (lane == 0) {
                unsigned long long t1;
                unsigned sm32;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                asm volatile("mov.u32 %0, %%smid;" : "=r"(sm32));
                const unsigned long long sm = sm32;
                unsigned long long* rec = timeline + 4 * ((size_t)blk * 8 + sub);
                rec[0] = t_tile;
                rec[1] = t1;
                rec[2] = (sm << 32) | rem;
                rec[3] = view | ((unsigned long long)split << 32);
            }
        }
    }
    __syncthreads();
    __shared__ unsigned s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        const bool last = atomicAdd(work + 1, 1u) == gridDim.x - 1;
        if (last) {
            atomicExch(work, 0u);
            atomicExch(work + 1, 0u);
        }
        s_last = last ? 1u : 0u;
    }
    if (opt.blk_cost != nullptr) {
        __syncthreads();
        if (s_last) {   // every other CTA has finished: build the next launch's order
            __threadfence();
            reorder_blocks(opt.blk_cost, const_cast<unsigned*>(order), per_view, reinterpret_cast<uint8_t*>(stk_storage),
                           opt.split_k, opt.split_f, opt.zip_order != 0);
        }
    }
}

// One ray of po_render_rays (forward, or pass 1 with aux / leaf span / stored segments).
template <int DEG, bool F16>
__device__ __forceinline__ void render_ray(const DevTree& tr, const float* __restrict__ rays, int64_t i,
                                           const RenderOpts& opt, float* __restrict__ out, double* __restrict__ aux,
                                           uint32_t* __restrict__ span, const SegOut& so, const SmemStack& stk) {
    float o[3], d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[k] = __ldg(rays + i * 6 + k);
        d[k] = __ldg(rays + i * 6 + 3 + k);
    }
    RayState r;
    const bool hit = ray_setup(tr, o, d, r);
    if (aux == nullptr) {
        float C[3] = {opt.bg[0], opt.bg[1], opt.bg[2]};
        if (hit) {
            FwdVisitor<DEG, F16> v(tr, r.d, opt.gamma);
            traverse<kOptDefault | kOptGrid>(tr, r, v, stk);   // cell index when built
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) C[ch] = fmaf(v.T, opt.bg[ch], v.C[ch]);
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) out[i * 3 + ch] = C[ch];
    } else {
        double C[3] = {opt.bg[0], opt.bg[1], opt.bg[2]};
        float T = 1.f;
        uint32_t lo = 0xFFFFFFFFu, hi = 0u;
        int32_t nseg = 0;
        if (hit) {
            TotalVisitor<DEG, F16> v(tr, r.d, opt.gamma);
            if (so.count != nullptr) {
                v.seg = so.rec != nullptr ? so.rec + 2 * i : nullptr;
                v.seg_stride = 2 * so.n;
                v.max_seg = so.max_seg;
            }
            traverse<kOptDefault | kOptGrid>(tr, r, v, stk);   // cell index when built
            nseg = v.nseg;
            T = v.T;
            lo = v.lo;
            hi = v.hi;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) C[ch] = v.C[ch] + (double)v.T * (double)opt.bg[ch];
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            out[i * 3 + ch] = (float)C[ch];
            aux[i * 4 + ch] = C[ch];
        }
        aux[i * 4 + 3] = (double)T;
        if (span != nullptr) reinterpret_cast<uint2*>(span)[i] = make_uint2(lo, hi);
        if (so.count != nullptr) so.count[i] = nseg;
    }
}

template <int DEG, bool F16>
__global__ void __launch_bounds__(256, 2) k_render_rays(DevTree tr, const float* __restrict__ rays, int64_t n,
                                                     RenderOpts opt, float* __restrict__ out, double* __restrict__ aux,
                                                     uint32_t* __restrict__ span, SegOut so) {
    PO_DECLARE_STACK(stk);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    render_ray<DEG, F16>(tr, rays, i, opt, out, aux, span, so, stk);
}

// Persistent variant: every warp claims the next 32 consecutive rays from a global counter, so
// a warp slot is refilled as soon as its own rays finish (a one-thread-per-ray grid holds each
// CTA's slot until its slowest warp ends: at gamma = 0 the ray lengths vary widely).  work[0] =
// next chunk, work[1] = finished CTAs; both zero on entry, reset by the last CTA.
template <int DEG, bool F16>
#ifndef PO_RAYS_MINB
#define PO_RAYS_MINB 2
#endif
__global__ void __launch_bounds__(256, PO_RAYS_MINB) k_render_rays_p(DevTree tr, const float* __restrict__ rays, int64_t n,
                                                       RenderOpts opt, float* __restrict__ out,
                                                       double* __restrict__ aux, uint32_t* __restrict__ span,
                                                       SegOut so, unsigned* __restrict__ work) {
    PO_DECLARE_STACK(stk);
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned c = 0;
        if (lane == 0) c = atomicAdd(work, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        if ((int64_t)c * 32 >= n) break;
        const int64_t i0 = 32 * (int64_t)(opt.group_order != nullptr ? __ldg(opt.group_order + c) : (int32_t)c);
        if (i0 + lane < n) render_ray<DEG, F16>(tr, rays, i0 + lane, opt, out, aux, span, so, stk);
        __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(work + 1, 1u) == gridDim.x - 1) {
            atomicExch(work, 0u);
            atomicExch(work + 1, 0u);
        }
    }
}

#ifdef PO_DIAG
// Measurement variants of the plain forward over a ray list (PO_RAYS_OPT, SH-3 fp32 only):
// 128 = the default lean step, 64 = traversal + T only (wrong colours).  Used by
// tools/diag_tail.py to time single warp tiles alone ("where the tail comes from").
template <int OPT>
__global__ void __launch_bounds__(256, 2) k_render_rays_diag(DevTree tr, const float* __restrict__ rays, int64_t n,
                                                          RenderOpts opt, float* __restrict__ out) {
    PO_DECLARE_STACK(stk);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float o[3], d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[k] = __ldg(rays + i * 6 + k);
        d[k] = __ldg(rays + i * 6 + 3 + k);
    }
    RayState r;
    float C[3] = {opt.bg[0], opt.bg[1], opt.bg[2]};
    if (ray_setup(tr, o, d, r)) {
        if constexpr (OPT == kOptProbeNoShade) {
            struct Probe {
                const DevTree& tr;
                float T, gamma;
                __device__ __forceinline__ void on_node() {}
                __device__ __forceinline__ bool on_leaf(uint32_t idx, float t0, float t1) {
                    const float st = __ldg(tr.sigma + idx);
                    if (!(st > 0.f)) return true;
                    T = absorb(T, st, __fsub_rn(t1, t0)).Tn;
                    return !(T < gamma);
                }
            } v{tr, 1.f, opt.gamma};
            traverse<kOptLean>(tr, r, v, stk);
            C[0] = C[1] = C[2] = v.T;
        } else {
            FwdVisitor<3, false> v(tr, r.d, opt.gamma);
            traverse<OPT>(tr, r, v, stk);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) C[ch] = fmaf(v.T, opt.bg[ch], v.C[ch]);
        }
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) out[i * 3 + ch] = C[ch];
}

// Measurement: per-box-step SM cycles of the forward (po_ray_step_timing).  Record k of a ray =
// (cycles since the previous box step, loads << 8 | shift << 1 | previous box was a shaded leaf):
// the cycles cover the previous box's leaf work, the neighbour step and this box's descent.
template <int DEG>
struct StepTimingVisitor : FwdVisitor<DEG, false> {
    uint32_t* rec;
    int32_t max_steps, steps, loads;
    long long last;
    bool leaf_prev;
    __device__ StepTimingVisitor(const DevTree& t, const float d[3], float g) : FwdVisitor<DEG, false>(t, d, g) {}
    __device__ __forceinline__ void on_node() { ++loads; }
    __device__ __forceinline__ void on_box(int shift) {
        const long long now = clock64();
        if (steps < max_steps) {
            rec[2 * steps] = (uint32_t)min(now - last, 0xFFFFFFFFll);
            rec[2 * steps + 1] = ((uint32_t)loads << 8) | ((uint32_t)shift << 1) | (leaf_prev ? 1u : 0u);
        }
        ++steps;
        loads = 0;
        leaf_prev = false;
        last = clock64();
    }
    __device__ __forceinline__ bool on_leaf(uint32_t idx, float t0, float t1) {
        leaf_prev = true;
        return FwdVisitor<DEG, false>::on_leaf(idx, t0, t1);
    }
};

__global__ void __launch_bounds__(256, 2) k_ray_step_timing(DevTree tr, const float* __restrict__ rays, int64_t n,
                                                         RenderOpts opt, int32_t max_steps, uint32_t* __restrict__ rec,
                                                         int32_t* __restrict__ steps) {
    PO_DECLARE_STACK(stk);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float o[3], d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[k] = __ldg(rays + i * 6 + k);
        d[k] = __ldg(rays + i * 6 + 3 + k);
    }
    RayState r;
    int32_t ns = 0;
    if (ray_setup(tr, o, d, r)) {
        StepTimingVisitor<3> v(tr, r.d, opt.gamma);
        v.rec = rec + (size_t)i * max_steps * 2;
        v.max_steps = max_steps;
        v.steps = 0;
        v.loads = 0;
        v.leaf_prev = false;
        v.last = clock64();
        traverse(tr, r, v, stk);
        ns = v.steps;
    }
    steps[i] = ns;
}

cudaError_t launch_ray_step_timing(const DevTree& tr, const float* rays, int64_t n, const RenderOpts& opt,
                                   int32_t max_steps, uint32_t* rec, int32_t* steps, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_ray_step_timing<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(tr, rays, n, opt, max_steps, rec, steps);
    return cudaGetLastError();
}

#endif  // PO_DIAG

struct SegIn {
    const float4* __restrict__ rec;
    const int32_t* __restrict__ count;
    int64_t n;
    int32_t max_seg;
};

// One training ray of pass 2 (a7 + a8): total from aux (or its own pass 1), then the
// gradient traversal.  Shared by k_backward (one thread per ray) and k_backward_chunk.
// kSkipReplay: rays whose segments are stored return at once (k_backward_replay has them)
template <int DEG, bool F16, bool kSkipReplay = false>
__device__ __forceinline__ void backward_ray(const DevTree& tr, const float* __restrict__ rays, int64_t i,
                                             const float* __restrict__ dL_dC, const double* __restrict__ aux,
                                             const SegIn& si, const RenderOpts& opt, float* __restrict__ grad_sigma,
                                             float* __restrict__ grad_sh, const SmemStack& stk) {
    if constexpr (kSkipReplay) {
        if (__ldg(si.count + i) <= si.max_seg) return;
    }
    float o[3], d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[k] = __ldg(rays + i * 6 + k);
        d[k] = __ldg(rays + i * 6 + 3 + k);
    }
    RayState r;
    if (!ray_setup(tr, o, d, r)) return;   // a miss touches no leaf
    GradVisitor<DEG, F16> gv(tr, r.d, opt.gamma, grad_sigma, grad_sh);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) gv.g[ch] = __ldg(dL_dC + i * 3 + ch);
    if (gv.g[0] == 0.f && gv.g[1] == 0.f && gv.g[2] == 0.f) return;
    if (aux != nullptr && si.count != nullptr) {
        const int32_t ns = __ldg(si.count + i);
        if (ns <= si.max_seg) {   // replay the stored segments: no traversal, no SH rows
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) gv.Ctot[ch] = aux[i * 4 + ch];
            const float4* rec = si.rec + 2 * i;   // unused when ns == 0 (max_seg may be 0)
            for (int32_t k = 0; k < ns; ++k, rec += 2 * si.n) {
                const float4 a = __ldg(rec), b = __ldg(rec + 1);
                const float c[3] = {b.x, b.y, b.z};
                gv.seg(__float_as_uint(a.x), a.y, a.z, a.w, c);
            }
            return;
        }
    }
    if (aux != nullptr) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) gv.Ctot[ch] = aux[i * 4 + ch];
    } else {   // pass 1: total = sum_{k<=N} c_k w_k including the background
        TotalVisitor<DEG, F16> tv(tr, r.d, opt.gamma);
        traverse<kOptDefault | kOptGrid>(tr, r, tv, stk);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) gv.Ctot[ch] = tv.C[ch] + (double)tv.T * (double)opt.bg[ch];
    }
    traverse<kOptDefault | kOptGrid>(tr, r, gv, stk);
}

template <int DEG, bool F16, bool kSkipReplay>
__global__ void __launch_bounds__(256, 2) k_backward(DevTree tr, const float* __restrict__ rays, int64_t n,
                                                  const float* __restrict__ dL_dC, const double* __restrict__ aux,
                                                  SegIn si, RenderOpts opt, float* __restrict__ grad_sigma,
                                                  float* __restrict__ grad_sh, int* __restrict__ overflow_flag) {
    PO_DECLARE_STACK(stk);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if constexpr (kSkipReplay) {   // po_render_backward_sgd: some ray's gradient went to the buffer
        if (overflow_flag != nullptr && __ldg(si.count + i) > si.max_seg) *overflow_flag = 1;
    }
    backward_ray<DEG, F16, kSkipReplay>(tr, rays, i, dL_dC, aux, si, opt, grad_sigma, grad_sh, stk);
}

// Stored-segment pass 2, one WARP per ray: lane l takes segments l, l+32, ... of the ray, so
// the record loads of a ray are in flight together instead of forming a per-thread chain
// (the one-thread-per-ray replay was load-latency bound: 1.27 ms on c4, 70 % long-scoreboard
// stalls).  The prefix P_i = sum_{k<=i} w_k c_k is an inclusive warp scan in double carried
// across 32-segment rounds (same sum as the sequential pass up to double rounding order);
// then every lane applies GradVisitor::seg's formula to its own segment.  Rays whose segments
// overflowed (count > max_seg) are left to k_backward<..., true>.
// Where the replay puts each segment's gradient: atomically into the leaf rows (default), or as
// a record for the deterministic segmented reduction (po_render_backward_deterministic).  Sinks
// are called by the whole warp once per round of up to 32 segments (lane l holds segment
// base + l when `act`); the active lanes are 0..n-1.
//
// Row reductions, lane-cooperative (SH-1 / SH-3: rows of 3B = 12 / 48 floats, whole float4
// quads).  A lane-per-segment red.v4 loop sends every lane to a different 192-B row, so each of
// the 12 red instructions of a round is 32 scattered L1 wavefronts (the replay's bound, r01:
// issue-active 17 %).  Instead the round's n segments x QPR quads are flattened and dealt to the
// 32 lanes in order: quad q = 32 it + lane belongs to segment q / QPR and row quad q % QPR, so one
// red.v4 instruction covers 512 contiguous bytes of ~3 consecutive-segment rows.  A lane's quad
// index cycles through 3 values (32 it mod QPR), so its basis values and channel selectors are
// three precomputed sets; the segment's gz comes by shuffle.  Same per-element products
// gz[ch] * Y[b] (scaled by `scale`), only the order of the atomic adds changes.
template <int DEG>
struct CoopRows {
    static constexpr int NE = 3 * ShDim<DEG>::B;
    static constexpr int QPR = NE / 4;   // quads per row
    static constexpr bool kCoop = (NE % 4) == 0;
    float yv[3][4];   // [phase][k]: Y of element 4 qq + k
    int ch[3][4];     // its channel
    int qq[3];
    __device__ __forceinline__ CoopRows(const float* Y, float scale) {
        if constexpr (kCoop) {
            const int lane = threadIdx.x & 31;
            // lane b holds Y[b] (a sum of 0/1-masked terms: no register array is indexed by the
            // lane, which would put Y in local memory); lanes then fetch Y[el / 3] by shuffle
            float ydist = 0.f;
#pragma unroll
            for (int b = 0; b < ShDim<DEG>::B; ++b) ydist = fmaf(Y[b], (float)(lane == b), ydist);
#pragma unroll
            for (int p = 0; p < 3; ++p) {
                qq[p] = (lane + 32 * p) % QPR;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int el = 4 * qq[p] + k;
                    yv[p][k] = scale * __shfl_sync(0xffffffffu, ydist, el / 3);
                    ch[p][k] = el % 3;
                }
            }
        }
    }
    // rows of `stride` floats at base; active lanes 0..n-1 hold (idx, gz)
    __device__ __forceinline__ void add(float* __restrict__ base, int64_t stride, int n, uint32_t idx,
                                        const float gz[3]) const {
        const int lane = threadIdx.x & 31;
        const int total = n * QPR;
        for (int it0 = 0; it0 * 32 < total; it0 += 3) {
#pragma unroll
            for (int p = 0; p < 3; ++p) {
                const int q = (it0 + p) * 32 + lane;
                const int sgi = min(q / QPR, 31);
                const uint32_t id = __shfl_sync(0xffffffffu, idx, sgi);
                const float g0 = __shfl_sync(0xffffffffu, gz[0], sgi);
                const float g1 = __shfl_sync(0xffffffffu, gz[1], sgi);
                const float g2 = __shfl_sync(0xffffffffu, gz[2], sgi);
                if (q < total) {
                    float v[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) v[k] = (ch[p][k] == 0 ? g0 : (ch[p][k] == 1 ? g1 : g2)) * yv[p][k];
                    float* a = base + (size_t)id * stride + 4 * qq[p];
                    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(v[0]), "f"(v[1]),
                                 "f"(v[2]), "f"(v[3])
                                 : "memory");
                }
            }
        }
    }
};

template <int DEG>
struct AtomicSink {
    float* __restrict__ grad_sigma;
    float* __restrict__ grad_sh;
    __device__ __forceinline__ void round(const CoopRows<DEG>& rows, int32_t, bool act, int n, uint32_t idx, float gsig,
                                          const float gz[3], const float* Y) {
        constexpr int NE = 3 * ShDim<DEG>::B;
        if (act) atomicAdd(grad_sigma + idx, gsig);
        if constexpr (CoopRows<DEG>::kCoop) {
            rows.add(grad_sh, NE, n, idx, gz);
        } else if (act) {
            float* row = grad_sh + (size_t)idx * NE;
#pragma unroll
            for (int el = 0; el < NE; ++el) atomicAdd(row + el, gz[el % 3] * Y[el / 3]);
        }
    }
};

struct EmitSink {   // segment k of ray `ray` -> flat slot f0 + k
    uint32_t* __restrict__ key;
    uint32_t* __restrict__ val;
    float4* __restrict__ contrib;
    int32_t* __restrict__ ray_of;
    int64_t f0;
    int32_t ray;
    template <class R>
    __device__ __forceinline__ void round(const R&, int32_t k, bool act, int, uint32_t idx, float gsig,
                                          const float gz[3], const float*) {
        if (!act) return;
        const int64_t f = f0 + k;
        key[f] = idx;
        val[f] = (uint32_t)f;
        contrib[f] = make_float4(gsig, gz[0], gz[1], gz[2]);
        ray_of[f] = ray;
    }
};

template <int DEG, class Sink>
__device__ __forceinline__ void replay_ray(const DevTree& tr, const float* __restrict__ rays, int64_t i,
                                           const float* __restrict__ dL_dC, const double* __restrict__ aux,
                                           const SegIn& si, Sink& sink, float row_scale) {
    constexpr int B = ShDim<DEG>::B;
    const int lane = threadIdx.x & 31;
    const int32_t ns = __ldg(si.count + i);
    if (ns == 0 || ns > si.max_seg) return;
    float g[3], dir[3], d[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) g[ch] = __ldg(dL_dC + i * 3 + ch);
    if (g[0] == 0.f && g[1] == 0.f && g[2] == 0.f) return;
#pragma unroll
    for (int k = 0; k < 3; ++k) dir[k] = __ldg(rays + i * 6 + 3 + k);
    if (!unit_direction(dir, d)) return;
    float Y[B];
    ray_basis<DEG>(tr, d, Y);
    const CoopRows<DEG> rows(Y, row_scale);
    double Ctot[3], carry[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) Ctot[ch] = aux[i * 4 + ch];
    for (int32_t base = 0; base < ns; base += 32) {
        const int32_t k = base + lane;
        const bool act = k < ns;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        if (act) {
            const float4* rec = si.rec + 2 * ((int64_t)k * si.n + i);
            a = __ldg(rec);
            b = __ldg(rec + 1);
        }
        const float c[3] = {b.x, b.y, b.z};
        double P[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            double v = (double)a.z * (double)c[ch];   // w_k c_k (0 for inactive lanes)
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const double u = __shfl_up_sync(0xFFFFFFFFu, v, off);
                if (lane >= off) v += u;
            }
            P[ch] = carry[ch] + v;
            carry[ch] = __shfl_sync(0xFFFFFFFFu, P[ch], 31);
        }
        const uint32_t idx = __float_as_uint(a.x);
        const float delta = a.y, w = a.z, Tn = a.w;
        double acc = 0.0;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) acc += (double)g[ch] * ((double)c[ch] * (double)Tn - (Ctot[ch] - P[ch]));
        float gz[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) gz[ch] = act ? g[ch] * w * c[ch] * (1.f - c[ch]) : 0.f;
        sink.round(rows, k, act, min(ns - base, 32), idx, (float)((double)delta * acc), gz, Y);
    }
}

template <int DEG>
__global__ void __launch_bounds__(256, 3) k_backward_replay(DevTree tr, const float* __restrict__ rays, int64_t n,
                                                         const float* __restrict__ dL_dC,
                                                         const double* __restrict__ aux, SegIn si,
                                                         float* __restrict__ grad_sigma,
                                                         float* __restrict__ grad_sh) {
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= n) return;
    AtomicSink<DEG> sink{grad_sigma, grad_sh};
    replay_ray<DEG>(tr, rays, i, dL_dC, aux, si, sink, 1.f);
}

// a8 + a9 fused (po_render_backward_sgd, one replica): each segment's contribution scaled by
// -lr goes straight into the tree's own sigma~ and padded SH rows, so plain SGD
// needs no gradient buffer and no separate update pass (the update is linear in the summed
// gradient; only the fp32 summation order differs from gradient-then-SGD)
template <int DEG>
struct SgdSink {
    float* __restrict__ sigma;
    float* __restrict__ sh;
    int32_t sh_row;
    float neg_lr;
    __device__ __forceinline__ void round(const CoopRows<DEG>& rows, int32_t, bool act, int n, uint32_t idx, float gsig,
                                          const float gz[3], const float* Y) {
        constexpr int NE = 3 * ShDim<DEG>::B;
        if (act) atomicAdd(sigma + idx, neg_lr * gsig);
        if constexpr (CoopRows<DEG>::kCoop) {
            rows.add(sh, sh_row, n, idx, gz);   // rows were built with scale = -lr
        } else if (act) {
            float* row = sh + (size_t)idx * sh_row;
#pragma unroll
            for (int el = 0; el < NE; ++el) atomicAdd(row + el, neg_lr * (gz[el % 3] * Y[el / 3]));
        }
    }
};

template <int DEG>
#ifndef PO_REPLAY_MINB
#define PO_REPLAY_MINB 4   // 4 CTAs/SM (64 registers, 104-B spill) measured +1.2 % over 3 (80, none): DESIGN.md §6.2
#endif
__global__ void __launch_bounds__(256, PO_REPLAY_MINB) k_backward_replay_sgd(DevTree tr, const float* __restrict__ rays, int64_t n,
                                                             const float* __restrict__ dL_dC,
                                                             const double* __restrict__ aux, SegIn si,
                                                             float* __restrict__ sigma, float* __restrict__ sh,
                                                             int32_t sh_row, float neg_lr) {
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= n) return;
    SgdSink<DEG> sink{sigma, sh, sh_row, neg_lr};
    replay_ray<DEG>(tr, rays, i, dL_dC, aux, si, sink, neg_lr);
}

// the same over one chunk of a po_backward_plan (bounds on the device): a persistent grid
// whose warps stride over perm[chunk_end[c-1] .. chunk_end[c]) (static: ~100 rays per warp on
// c4, balanced without a shared counter)
template <int DEG>
__global__ void __launch_bounds__(256, 2) k_backward_replay_chunk(DevTree tr, const float* __restrict__ rays,
                                                               const int32_t* __restrict__ perm,
                                                               const int64_t* __restrict__ chunk_end, int chunk,
                                                               const float* __restrict__ dL_dC,
                                                               const double* __restrict__ aux, SegIn si,
                                                               float* __restrict__ grad_sigma,
                                                               float* __restrict__ grad_sh) {
    const int64_t b = chunk > 0 ? chunk_end[chunk - 1] : 0, e = chunk_end[chunk];
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    AtomicSink<DEG> sink{grad_sigma, grad_sh};
    for (int64_t j = b + w0; j < e; j += nw)
        replay_ray<DEG>(tr, rays, (int64_t)__ldg(perm + j), dL_dC, aux, si, sink, 1.f);
}

// ---- deterministic pass 2: segmented reduction into leaves (NEXT f2 "deterministic-reduction
// mode"; the north star's alternative to atomics).  1) per ray, the number of segments it will
// emit (0 where the atomic replay would return early; overflow rays are counted and left to
// the re-traversal); 2) exclusive scan -> flat slots; 3) the replay emits (leaf, slot) keys and
// (dL/dsigma~, gz) records; 4) stable radix sort by leaf; 5) one thread per leaf sums its run in
// slot order (= ray order, then k) and adds the sums once: every float sum has a fixed order.
__global__ void __launch_bounds__(256) k_det_counts(const float* __restrict__ rays, int64_t n,
                                                    const float* __restrict__ dL_dC, SegIn si,
                                                    int32_t* __restrict__ cnt, int32_t* __restrict__ n_overflow) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i == n) {   // trailing 0: the exclusive scan then ends with the total
        cnt[i] = 0;
        return;
    }
    const int32_t ns = __ldg(si.count + i);
    int32_t c = ns;
    if (ns > si.max_seg) {
        c = 0;
        if (n_overflow) atomicAdd(n_overflow, 1);
    } else if (ns > 0) {
        float dir[3], d[3];
        const float g0 = __ldg(dL_dC + i * 3), g1 = __ldg(dL_dC + i * 3 + 1), g2 = __ldg(dL_dC + i * 3 + 2);
#pragma unroll
        for (int k = 0; k < 3; ++k) dir[k] = __ldg(rays + i * 6 + 3 + k);
        if ((g0 == 0.f && g1 == 0.f && g2 == 0.f) || !unit_direction(dir, d)) c = 0;
    }
    cnt[i] = c;
}

template <int DEG>
__global__ void __launch_bounds__(256, 3) k_det_emit(DevTree tr, const float* __restrict__ rays, int64_t n,
                                                  const float* __restrict__ dL_dC, const double* __restrict__ aux,
                                                  SegIn si, const int32_t* __restrict__ offs,
                                                  uint32_t* __restrict__ key, uint32_t* __restrict__ val,
                                                  float4* __restrict__ contrib, int32_t* __restrict__ ray_of) {
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= n) return;
    EmitSink sink{key, val, contrib, ray_of, (int64_t)__ldg(offs + i), (int32_t)i};
    replay_ray<DEG>(tr, rays, i, dL_dC, aux, si, sink, 1.f);
}

template <int DEG>
__global__ void __launch_bounds__(256) k_det_reduce(DevTree tr, const float* __restrict__ rays,
                                                    const uint32_t* __restrict__ skey,
                                                    const uint32_t* __restrict__ sval, int64_t S,
                                                    const float4* __restrict__ contrib,
                                                    const int32_t* __restrict__ ray_of, float* __restrict__ grad_sigma,
                                                    float* __restrict__ grad_sh) {
    constexpr int B = ShDim<DEG>::B;
    constexpr int NE = 3 * B;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S) return;
    const uint32_t leaf = skey[j];
    if (j > 0 && skey[j - 1] == leaf) return;   // one thread per run of equal leaves
    float ss = 0.f, acc[NE];
#pragma unroll
    for (int el = 0; el < NE; ++el) acc[el] = 0.f;
    for (int64_t m = j; m < S && skey[m] == leaf; ++m) {
        const uint32_t f = sval[m];
        const float4 c4 = contrib[f];
        const int32_t r = ray_of[f];
        float dir[3], d[3], Y[B];
#pragma unroll
        for (int k = 0; k < 3; ++k) dir[k] = __ldg(rays + (int64_t)r * 6 + 3 + k);
        unit_direction(dir, d);
        ray_basis<DEG>(tr, d, Y);
        const float gz[3] = {c4.y, c4.z, c4.w};
        ss += c4.x;
#pragma unroll
        for (int el = 0; el < NE; ++el) acc[el] += gz[el % 3] * Y[el / 3];
    }
    grad_sigma[leaf] += ss;
    float* row = grad_sh + (size_t)leaf * NE;
#pragma unroll
    for (int el = 0; el < NE; ++el) row[el] += acc[el];
}

// Pass 2 over one chunk of a po_backward_plan: rays perm[chunk_end[c-1] .. chunk_end[c]).
// The bounds live on the device (no host sync between the plan and the chunks), so the grid
// is persistent and warps claim 32-ray batches from a global counter (work[0]); no warp waits
// for a slower one (CTA-wide 256-ray claims measured 5 % slower at K = 2 and 4); the last CTA
// resets the counters (work[1] = finished CTAs) for the next launch on the stream.
template <int DEG, bool F16, bool kSkipReplay>
__global__ void __launch_bounds__(256, 2) k_backward_chunk(DevTree tr, const float* __restrict__ rays,
                                                        const int32_t* __restrict__ perm,
                                                        const int64_t* __restrict__ chunk_end, int chunk,
                                                        const float* __restrict__ dL_dC,
                                                        const double* __restrict__ aux, SegIn si, RenderOpts opt,
                                                        float* __restrict__ grad_sigma, float* __restrict__ grad_sh,
                                                        unsigned* __restrict__ work) {
    PO_DECLARE_STACK(stk);
    const int64_t b = chunk > 0 ? chunk_end[chunk - 1] : 0, e = chunk_end[chunk];
    const int64_t nb = (e - b + 31) >> 5;
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned k = 0;
        if (lane == 0) k = atomicAdd(work, 1u);
        k = __shfl_sync(0xFFFFFFFFu, k, 0);
        if ((int64_t)k >= nb) break;
        const int64_t j = b + ((int64_t)k << 5) + lane;
        if (j < e)
            backward_ray<DEG, F16, kSkipReplay>(tr, rays, (int64_t)__ldg(perm + j), dL_dC, aux, si, opt, grad_sigma,
                                                grad_sh, stk);
        __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(work + 1, 1u) == gridDim.x - 1) {
            atomicExch(work, 0u);
            atomicExch(work + 1, 0u);
        }
    }
}

// po_backward_plan helpers: sort keys = first sigma~>0 leaf of each ray (n_leaves if none)
__global__ void __launch_bounds__(256) k_plan_keys(const uint32_t* __restrict__ span, int64_t n, uint32_t n_leaves,
                                                   uint32_t* __restrict__ keys, int32_t* __restrict__ idx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = min(__ldg(span + 2 * i), n_leaves);
    idx[i] = (int32_t)i;
}

// chunk_end[j] = #rays whose key < b_j (bounds from the host); quant[j] (optional) = the key
// that splits the rays with a sigma>0 leaf into K equal parts -- balanced bounds for the next
// plan (the caller feeds them back; any monotone bounds keep the finality invariant)
__global__ void k_plan_ends(const uint32_t* __restrict__ sorted_keys, int64_t n, int64_t n_leaves, PlanBounds bounds,
                            int64_t* __restrict__ chunk_end, int64_t* __restrict__ quant) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= bounds.K) return;
    auto lower_bound = [&](int64_t v) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)sorted_keys[mid] < v) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    chunk_end[j] = lower_bound(bounds.b[j]);
    if (quant != nullptr) {
        const int64_t n_hit = lower_bound(n_leaves);
        const int64_t pos = n_hit * (int64_t)(j + 1) / bounds.K;
        quant[j] = (j == bounds.K - 1 || pos >= n_hit) ? n_leaves : (int64_t)sorted_keys[pos];
    }
}

__global__ void __launch_bounds__(256) k_render_depth(DevTree tr, const float* __restrict__ rays, int64_t n,
                                                      float gamma, float* __restrict__ alpha,
                                                      float* __restrict__ depth) {
    PO_DECLARE_STACK(stk);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float o[3], d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[k] = __ldg(rays + i * 6 + k);
        d[k] = __ldg(rays + i * 6 + 3 + k);
    }
    DepthVisitor v{tr, 1.f, gamma, 0.f};
    RayState r;
    if (ray_setup(tr, o, d, r)) traverse<kOptDefault | kOptGrid>(tr, r, v, stk);
    alpha[i] = __fsub_rn(1.0f, v.T);
    depth[i] = v.D;
}

__global__ void __launch_bounds__(256) k_leaf_max_alpha(DevTree tr, const float* __restrict__ rays, int64_t n,
                                                        float gamma, unsigned* __restrict__ max_alpha) {
    PO_DECLARE_STACK(stk);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float o[3], d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[k] = __ldg(rays + i * 6 + k);
        d[k] = __ldg(rays + i * 6 + 3 + k);
    }
    MaxAlphaVisitor v{tr, 1.f, gamma, max_alpha};
    RayState r;
    if (ray_setup(tr, o, d, r)) traverse<kOptDefault | kOptGrid>(tr, r, v, stk);
}

// Parity / measurement trace.  GRID = the production traversal (the level-(D-1) cell index when
// the tree has one, exactly as k_render / k_render_rays / the backward run it); !GRID = the
// classic descent from the deepest common ancestor, which also counts the internal nodes met.
template <bool GRID>
__global__ void __launch_bounds__(256) k_trace(DevTree tr, const float* __restrict__ rays, int64_t n, float gamma,
                                               int32_t max_leaves, int32_t* __restrict__ leaf_ids,
                                               int32_t* __restrict__ counts, int32_t* __restrict__ node_counts) {
    PO_DECLARE_STACK(stk);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float o[3], d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[k] = rays[i * 6 + k];
        d[k] = rays[i * 6 + 3 + k];
    }
    int32_t* ids = leaf_ids ? leaf_ids + i * max_leaves : nullptr;
    for (int j = 0; j < max_leaves && ids; ++j) ids[j] = -1;
    TraceVisitor v{tr, 1.f, gamma, ids, ids ? max_leaves : 0, 0, 0};
    RayState r;
    if (ray_setup(tr, o, d, r, GRID)) {   // the classic reference walks the whole cube
        if constexpr (GRID) traverse<kOptDefault | kOptGrid>(tr, r, v, stk);
        else traverse<kOptDefault>(tr, r, v, stk);
    }
    if (counts) counts[i] = v.count;
    if (node_counts) node_counts[i] = v.nodes;
}

constexpr int kStatCounters = 7;
__global__ void __launch_bounds__(256) k_stats(DevTree tr, const po_camera* __restrict__ cams, int W, int H,
                                               float gamma, unsigned long long* __restrict__ counters) {
    PO_DECLARE_STACK(stk);
    int px, py;
    unsigned long long v4[kStatCounters] = {0, 0, 0, 0, 0, 0, 0};
    if (tile_pixel(W, H, px, py)) {
        float o[3], d[3];
        camera_ray(cams, blockIdx.z, px, py, o, d);
        RayState r;
        if (ray_setup(tr, o, d, r, false)) {   // counts of the classic descent over the whole cube
            StatsVisitor v{tr, 1.f, gamma, 0, 0, 0, 0, 0};
            traverse(tr, r, v, stk);
            v4[0] = v.leaves;
            v4[1] = v.sh_rows;
            v4[2] = v.nodes;
            v4[3] = 1;
            v4[4] = v.boxes;
            v4[5] = v.leaf_level_boxes;
        }
    }
    // SIMT cost: boxes of the longest ray of each warp (the warp executes that many steps)
    v4[6] = (threadIdx.x & 31) == 0 ? __reduce_max_sync(0xffffffffu, (unsigned)v4[4])
                                    : (__reduce_max_sync(0xffffffffu, (unsigned)v4[4]), 0u);
#pragma unroll
    for (int k = 0; k < kStatCounters; ++k) {
        unsigned long long s = v4[k];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if ((threadIdx.x & 31) == 0 && s) atomicAdd(counters + k, s);
    }
}

__global__ void __launch_bounds__(256) k_l2_loss(const float* __restrict__ pred, const float* __restrict__ target,
                                                 int64_t n3, float* __restrict__ dL_dC, double* __restrict__ loss) {
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n3; i += (int64_t)gridDim.x * blockDim.x) {
        const float diff = pred[i] - target[i];
        dL_dC[i] = 2.0f * diff;
        acc += (double)diff * (double)diff;
    }
    if (loss == nullptr) return;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        atomicAdd(loss, s);
    }
}

// a9 SGD: p -= lr g over parameter indices [begin, end) ([0, n_leaves) sigma~, then
// the SH elements leaf-major).  Entries with g == 0 are skipped (p - lr 0 = p exactly), so
// leaves no ray touched cost one gradient read; zero_grad writes 0 over consumed entries
// (replaces the caller's memset).  The SH part moves float4 quads when rows are multiples of 4
// (16-B aligned in both the gradient and the padded leaf rows).
__global__ void __launch_bounds__(256) k_sgd(float* __restrict__ sigma, float* __restrict__ sh, int32_t sh_row,
                                             int32_t ne, int64_t n_leaves, float* __restrict__ grad_sigma,
                                             float* __restrict__ grad_sh, float lr, int64_t begin, int64_t end,
                                             bool zero_grad, const int* __restrict__ gate) {
    if (gate != nullptr && *gate == 0) return;   // po_render_backward_sgd: the buffer is all zero
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = begin + tid; i < min(end, n_leaves); i += nth) {
        const float g = grad_sigma[i];
        if (g != 0.f) {
            sigma[i] -= lr * g;
            if (zero_grad) grad_sigma[i] = 0.f;
        }
    }
    if (end <= n_leaves) return;
    const int64_t hb = max(begin, n_leaves) - n_leaves, he = end - n_leaves;   // SH element range
    auto scalar = [&](int64_t j) {
        const float g = grad_sh[j];
        if (g != 0.f) {
            const int64_t leaf = j / ne;
            sh[leaf * sh_row + (j - leaf * ne)] -= lr * g;
            if (zero_grad) grad_sh[j] = 0.f;
        }
    };
    if ((ne & 3) != 0) {
        for (int64_t j = hb + tid; j < he; j += nth) scalar(j);
        return;
    }
    const int64_t qb = (hb + 3) >> 2, qe = he >> 2;   // whole quads inside the range
    if (qb >= qe) {
        for (int64_t j = hb + tid; j < he; j += nth) scalar(j);
        return;
    }
    if (tid < 4) {   // ragged head / tail of the range
        const int64_t j0 = hb + tid, j1 = (qe << 2) + tid;
        if (j0 < (qb << 2)) scalar(j0);
        if (j1 < he) scalar(j1);
    }
    const uint32_t qpr = (uint32_t)(ne >> 2);   // quads per leaf row
    float4* __restrict__ g4 = reinterpret_cast<float4*>(grad_sh);
    for (int64_t q = qb + tid; q < qe; q += nth) {
        const float4 g = g4[q];
        if (g.x == 0.f && g.y == 0.f && g.z == 0.f && g.w == 0.f) continue;
        const int64_t leaf = (q < ((int64_t)1 << 32)) ? (int64_t)((uint32_t)q / qpr) : q / qpr;
        float4* p = reinterpret_cast<float4*>(sh + leaf * sh_row) + (q - leaf * qpr);
        float4 v = *p;
        v.x -= lr * g.x;
        v.y -= lr * g.y;
        v.z -= lr * g.z;
        v.w -= lr * g.w;
        *p = v;
        if (zero_grad) g4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// ---------------------------------------------------------------------------------------
// Launchers (dispatch on SH degree x payload)
// ---------------------------------------------------------------------------------------
#define PO_DISPATCH(DEGV, F16V, ...)                                   \
    switch ((DEGV) * 2 + ((F16V) ? 1 : 0)) {                           \
        case 0: { constexpr int DEG = 0; constexpr bool F16 = false; __VA_ARGS__; } break; \
        case 1: { constexpr int DEG = 0; constexpr bool F16 = true; __VA_ARGS__; } break;  \
        case 2: { constexpr int DEG = 1; constexpr bool F16 = false; __VA_ARGS__; } break; \
        case 3: { constexpr int DEG = 1; constexpr bool F16 = true; __VA_ARGS__; } break;  \
        case 4: { constexpr int DEG = 2; constexpr bool F16 = false; __VA_ARGS__; } break; \
        case 5: { constexpr int DEG = 2; constexpr bool F16 = true; __VA_ARGS__; } break;  \
        case 6: { constexpr int DEG = 3; constexpr bool F16 = false; __VA_ARGS__; } break; \
        case 7: { constexpr int DEG = 3; constexpr bool F16 = true; __VA_ARGS__; } break;  \
        case 8: { constexpr int DEG = 4; constexpr bool F16 = false; __VA_ARGS__; } break; \
        case 9: { constexpr int DEG = 4; constexpr bool F16 = true; __VA_ARGS__; } break;  \
        default: return cudaErrorInvalidValue;                         \
    }

static inline unsigned grid1d(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

// Ask for the smallest shared-memory carveout that still fits the register-limited number of
// resident CTAs, so the rest of the 256 KB L1/shared array stays L1: the traversal lives off
// L1 hits on nodes and leaf rows (r01: the driver's default picked a 102 KB carveout for the
// render kernel's 2 x 17.5 KB).  Returns CTAs per SM.
template <class K>
static int tune_carveout(K kernel, int block, size_t dyn_smem) {
    int dev = 0, per_sm = 0, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    if (dyn_smem > 0) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem);
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, dyn_smem);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kernel) == cudaSuccess && smem_sm > 0 && per_sm > 0) {
        const size_t need = (size_t)per_sm * (fa.sharedSizeBytes + dyn_smem + 1024);
        int pct = (int)((need * 100 + smem_sm - 1) / smem_sm);
        pct = pct < 1 ? 1 : (pct > 100 ? 100 : pct);
        cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    }
    return per_sm;
}

// tune_carveout once per kernel instance (non-persistent kernels, 256 threads, static smem)
template <class K>
static void carveout_once(K kernel) {
    static std::mutex mu;
    static std::map<const void*, bool> done;
    std::lock_guard<std::mutex> lk(mu);
    const void* key = reinterpret_cast<const void*>(kernel);
    if (done.count(key)) return;
    tune_carveout(kernel, 256, 0);
    done[key] = true;
}

template <class K>
static int persistent_grid(K kernel, int64_t max_ctas, size_t dyn_smem = 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    tune_carveout(kernel, 256, dyn_smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, dyn_smem);
    int64_t g = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    return (int)(g < max_ctas ? g : (max_ctas > 0 ? max_ctas : 1));
}

cudaError_t launch_render(const DevTree& tr, int deg, bool f16, const po_camera* cams, int n_cams, int W, int H,
                          const RenderOpts& opt, float* out, unsigned* work, const unsigned* order,
                          unsigned long long* timeline, cudaStream_t s) {
    const int64_t tiles = (int64_t)((W + 7) / 8) * ((H + 3) / 4) * n_cams;
    if (tiles >= (int64_t)0xFFFFFFF0u) return cudaErrorInvalidValue;
    // CTAs per SM the register budget is tuned for (SH-3 paths), chosen by the work per launch.
    // A single view is bounded by its slowest warp tiles: 2 CTAs/SM (<= 128
    // registers, all 12 LDG.128 of a leaf row in flight) gives those tiles the most issue slots
    // (c1: 4441 vs 3979 FPS at 3/SM).  With several views per launch the slow tiles overlap
    // other views and throughput wins: 3/SM from 2 views on (8 views: 7537 vs 6719 views/s),
    // 4/SM for very large launches (c2, 200 views: 8881 vs 8544 vs 7245 views/s at 4/3/2).
    // Rule in warp tiles per SM: < 200 -> 2, < 4000 -> 3, else 4.  PO_RENDER_MINB=1..4
    // overrides it; PO_RENDER_OPT (0 = plain neighbour step, 64 = traversal-only probe;
    // traverse.cuh) selects SH-3 fp32 variants for A/B experiments.
#ifdef PO_DIAG
    static const int env_minb = [] {
        const char* e = getenv("PO_RENDER_MINB");
        const int v = e ? atoi(e) : 0;
        return (v >= 1 && v <= 4) ? v : 0;
    }();
#else
    constexpr int env_minb = 0;
#endif
    static const int n_sm = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            v = 148;
        return v > 0 ? v : 148;
    }();
    const int64_t tiles_per_sm = tiles / n_sm;
    const int minb = env_minb ? env_minb : (tiles_per_sm < 200 ? 2 : (tiles_per_sm < 4000 ? 3 : 4));
#ifdef PO_DIAG
    static const int vopt = [] {
        const char* e = getenv("PO_RENDER_OPT");
        const int v = e ? atoi(e) : kRenderOptDefault;
        return (v == kOptPlain || v == kOptProbeNoShade || v == kOptLean) ? v : kRenderOptDefault;
    }();
#else
    constexpr int vopt = kRenderOptDefault;
#endif
    using KFn = void (*)(DevTree, const po_camera*, int, int, int, RenderOpts, float*, unsigned*, const unsigned*,
                         unsigned long long*);
    KFn fn = nullptr;
    if (deg == 3 && vopt == kRenderOptDefault) {
        static const KFn k32[4] = {k_render<3, false, 1, kRenderOptDefault>, k_render<3, false, 2, kRenderOptDefault>,
                                   k_render<3, false, 3, kRenderOptDefault>, k_render<3, false, 4, kRenderOptDefault>};
        static const KFn k16[4] = {k_render<3, true, 1, kRenderOptDefault>, k_render<3, true, 2, kRenderOptDefault>,
                                   k_render<3, true, 3, kRenderOptDefault>, k_render<3, true, 4, kRenderOptDefault>};
        fn = f16 ? k16[minb - 1] : k32[minb - 1];
    }
#ifdef PO_DIAG
    else if (deg == 3 && !f16) {
        static const KFn probe[4] = {k_render<3, false, 1, kOptProbeNoShade>, k_render<3, false, 2, kOptProbeNoShade>,
                                     k_render<3, false, 3, kOptProbeNoShade>, k_render<3, false, 4, kOptProbeNoShade>};
        if (vopt == kOptProbeNoShade) fn = probe[minb - 1];
        else if (vopt == kOptLean) fn = k_render<3, false, 2, kOptLean>;   // without the index
        else fn = k_render<3, false, 2, kOptPlain>;
    }
#endif
    else {
        PO_DISPATCH(deg, f16, fn = k_render<DEG, F16, 2, kRenderOptDefault>);
    }
    const size_t dyn = 0;
    static std::mutex mu;
    static std::map<KFn, int> grids;   // persistent grid size per kernel instance
    int grid;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = grids.find(fn);
        if (it == grids.end()) it = grids.emplace(fn, persistent_grid(fn, 1 << 30, dyn)).first;
        grid = it->second;
    }
    const int g = (int)((int64_t)grid < (tiles + 7) / 8 ? grid : (tiles + 7) / 8);
    fn<<<g, 256, dyn, s>>>(tr, cams, n_cams, W, H, opt, out, work, order, timeline);
    return cudaGetLastError();
}

cudaError_t launch_render_rays(const DevTree& tr, int deg, bool f16, const float* rays, int64_t n,
                               const RenderOpts& opt, float* out, double* aux, uint32_t* span, const Segments& sg,
                               cudaStream_t s, unsigned* work) {
    if (n == 0) return cudaSuccess;
    const SegOut so{static_cast<float4*>(sg.rec), sg.count, sg.n, sg.max_seg};
#ifdef PO_DIAG
    static const int dopt = [] {   // measurement variants (k_render_rays_diag)
        const char* e = getenv("PO_RAYS_OPT");
        return e ? atoi(e) : 0;
    }();
    if (dopt != 0 && deg == 3 && !f16 && aux == nullptr) {
        if (dopt == kOptProbeNoShade)
            k_render_rays_diag<kOptProbeNoShade><<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, opt, out);
        else
            k_render_rays_diag<kOptLean><<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, opt, out);
        return cudaGetLastError();
    }
    static const bool persist = [] {   // A/B: PO_RAYS_PERSIST=0 keeps one thread per ray
        const char* e = getenv("PO_RAYS_PERSIST");
        return !(e && std::strcmp(e, "0") == 0);
    }();
#else
    constexpr bool persist = true;
#endif
    if (persist && work != nullptr && (n + 31) / 32 < (int64_t)0xFFFFFFF0u) {
        PO_DISPATCH(deg, f16, {
            static const int grid = persistent_grid(k_render_rays_p<DEG, F16>, 1 << 30, 0);
            const int64_t need = (n + 255) / 256;
            k_render_rays_p<DEG, F16><<<(unsigned)(grid < need ? grid : need), 256, 0, s>>>(tr, rays, n, opt, out, aux,
                                                                                          span, so, work);
        });
        return cudaGetLastError();
    }
    PO_DISPATCH(deg, f16, {
        carveout_once(k_render_rays<DEG, F16>);
        k_render_rays<DEG, F16><<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, opt, out, aux, span, so);
    });
    return cudaGetLastError();
}

cudaError_t launch_backward_chunk(const DevTree& tr, int deg, bool f16, const float* rays, const int32_t* perm,
                                  const int64_t* chunk_end, int chunk, const float* dL_dC, const double* aux,
                                  const Segments& sg, const RenderOpts& opt, float* grad_sigma, float* grad_sh,
                                  unsigned* work, cudaStream_t s) {
    const SegIn si{static_cast<const float4*>(sg.rec), sg.count, sg.n, sg.max_seg};
    const bool replay = aux != nullptr && sg.count != nullptr;
    PO_DISPATCH(deg, f16, {
        if (replay) {   // stored segments warp-per-ray, then the chunk's overflow rays by re-traversal
            static const int rgrid = persistent_grid(k_backward_replay_chunk<DEG>, 1 << 30, 0);
            k_backward_replay_chunk<DEG><<<rgrid, 256, 0, s>>>(tr, rays, perm, chunk_end, chunk, dL_dC, aux, si,
                                                               grad_sigma, grad_sh);
            static const int grid = persistent_grid(k_backward_chunk<DEG, F16, true>, 1 << 30, 0);
            k_backward_chunk<DEG, F16, true><<<grid, 256, 0, s>>>(tr, rays, perm, chunk_end, chunk, dL_dC, aux, si,
                                                                  opt, grad_sigma, grad_sh, work);
        } else {
            static const int grid = persistent_grid(k_backward_chunk<DEG, F16, false>, 1 << 30, 0);
            k_backward_chunk<DEG, F16, false><<<grid, 256, 0, s>>>(tr, rays, perm, chunk_end, chunk, dL_dC, aux, si,
                                                                   opt, grad_sigma, grad_sh, work);
        }
    });
    return cudaGetLastError();
}

cudaError_t launch_det_counts(const float* rays, int64_t n, const float* dL_dC, const Segments& sg, int32_t* cnt,
                              int32_t* n_overflow, cudaStream_t s) {
    const SegIn si{static_cast<const float4*>(sg.rec), sg.count, sg.n, sg.max_seg};
    k_det_counts<<<grid1d(n + 1, 256), 256, 0, s>>>(rays, n, dL_dC, si, cnt, n_overflow);
    return cudaGetLastError();
}

cudaError_t launch_det_emit(const DevTree& tr, int deg, const float* rays, int64_t n, const float* dL_dC,
                            const double* aux, const Segments& sg, const int32_t* offs, uint32_t* key, uint32_t* val,
                            float4* contrib, int32_t* ray_of, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const SegIn si{static_cast<const float4*>(sg.rec), sg.count, sg.n, sg.max_seg};
    PO_DISPATCH(deg, false, {
        k_det_emit<DEG><<<grid1d(n, 8), 256, 0, s>>>(tr, rays, n, dL_dC, aux, si, offs, key, val, contrib, ray_of);
    });
    return cudaGetLastError();
}

cudaError_t launch_det_reduce(const DevTree& tr, int deg, const float* rays, const uint32_t* skey,
                              const uint32_t* sval, int64_t S, const float4* contrib, const int32_t* ray_of,
                              float* grad_sigma, float* grad_sh, cudaStream_t s) {
    if (S == 0) return cudaSuccess;
    PO_DISPATCH(deg, false, {
        k_det_reduce<DEG><<<grid1d(S, 256), 256, 0, s>>>(tr, rays, skey, sval, S, contrib, ray_of, grad_sigma,
                                                         grad_sh);
    });
    return cudaGetLastError();
}

cudaError_t launch_plan_keys(const uint32_t* span, int64_t n, uint32_t n_leaves, uint32_t* keys, int32_t* idx,
                             cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_plan_keys<<<grid1d(n, 256), 256, 0, s>>>(span, n, n_leaves, keys, idx);
    return cudaGetLastError();
}

cudaError_t launch_plan_ends(const uint32_t* sorted_keys, int64_t n, int64_t n_leaves, const PlanBounds& b,
                             int64_t* chunk_end, int64_t* quant, cudaStream_t s) {
    k_plan_ends<<<1, 64, 0, s>>>(sorted_keys, n, n_leaves, b, chunk_end, quant);
    return cudaGetLastError();
}

cudaError_t launch_backward(const DevTree& tr, int deg, bool f16, const float* rays, int64_t n, const float* dL_dC,
                            const double* aux, const Segments& sg, const RenderOpts& opt, float* grad_sigma,
                            float* grad_sh, cudaStream_t s, bool overflow_only) {
    if (n == 0) return cudaSuccess;
    const SegIn si{static_cast<const float4*>(sg.rec), sg.count, sg.n, sg.max_seg};
    const bool replay = aux != nullptr && sg.count != nullptr;
    PO_DISPATCH(deg, f16, {
        if (replay) {   // stored segments first, then the overflow rays by re-traversal
            carveout_once(k_backward_replay<DEG>);
            if (!overflow_only)
                k_backward_replay<DEG><<<grid1d(n, 8), 256, 0, s>>>(tr, rays, n, dL_dC, aux, si, grad_sigma, grad_sh);
            carveout_once(k_backward<DEG, F16, true>);
            k_backward<DEG, F16, true><<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, dL_dC, aux, si, opt, grad_sigma,
                                                                      grad_sh, nullptr);
        } else {
            carveout_once(k_backward<DEG, F16, false>);
            k_backward<DEG, F16, false><<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, dL_dC, aux, si, opt, grad_sigma,
                                                                       grad_sh, nullptr);
        }
    });
    return cudaGetLastError();
}

cudaError_t launch_render_depth(const DevTree& tr, const float* rays, int64_t n, float gamma, float* alpha,
                                float* depth, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    carveout_once(k_render_depth);
    k_render_depth<<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, gamma, alpha, depth);
    return cudaGetLastError();
}

cudaError_t launch_leaf_max_alpha(const DevTree& tr, const float* rays, int64_t n, float gamma, float* max_alpha,
                                  cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    carveout_once(k_leaf_max_alpha);
    k_leaf_max_alpha<<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, gamma, reinterpret_cast<unsigned*>(max_alpha));
    return cudaGetLastError();
}

cudaError_t launch_trace(const DevTree& tr, const float* rays, int64_t n, float gamma, int32_t max_leaves,
                         int32_t* leaf_ids, int32_t* counts, int32_t* node_counts, bool classic, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (classic || tr.grid == nullptr) {
        carveout_once(k_trace<false>);
        k_trace<false><<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, gamma, max_leaves, leaf_ids, counts, node_counts);
        return cudaGetLastError();
    }
    carveout_once(k_trace<true>);
    k_trace<true><<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, gamma, max_leaves, leaf_ids, counts, nullptr);
    if (node_counts != nullptr) {   // the node count is a property of the classic descent
        carveout_once(k_trace<false>);
        k_trace<false><<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, gamma, 0, nullptr, nullptr, node_counts);
    }
    return cudaGetLastError();
}

cudaError_t launch_stats(const DevTree& tr, const po_camera* cams, int n_cams, int W, int H, float gamma,
                         unsigned long long* counters, cudaStream_t s) {
    dim3 grid((W + 15) / 16, (H + 15) / 16, n_cams);
    carveout_once(k_stats);
    k_stats<<<grid, 256, 0, s>>>(tr, cams, W, H, gamma, counters);
    return cudaGetLastError();
}

cudaError_t launch_l2_loss(const float* pred, const float* target, int64_t n3, float* dL_dC, double* loss,
                           cudaStream_t s) {
    if (loss) {
        cudaError_t e = cudaMemsetAsync(loss, 0, sizeof(double), s);
        if (e != cudaSuccess) return e;
    }
    if (n3 == 0) return cudaSuccess;
    unsigned g = grid1d(n3, 256);
    if (g > 148 * 16) g = 148 * 16;
    k_l2_loss<<<g, 256, 0, s>>>(pred, target, n3, dL_dC, loss);
    return cudaGetLastError();
}

cudaError_t launch_sgd(float* sigma, float* sh, int32_t sh_row, int32_t ne, int64_t n_leaves, float* grad_sigma,
                       float* grad_sh, float lr, int64_t begin, int64_t end, bool zero_grad, cudaStream_t s) {
    if (end <= begin) return cudaSuccess;
    unsigned g = grid1d(end - begin, 256 * 4);
    if (g > 148 * 16) g = 148 * 16;
    k_sgd<<<g, 256, 0, s>>>(sigma, sh, sh_row, ne, n_leaves, grad_sigma, grad_sh, lr, begin, end, zero_grad, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_backward_sgd(const DevTree& tr, int deg, const float* rays, int64_t n, const float* dL_dC,
                                const double* aux, const Segments& sg, const RenderOpts& opt, float* sigma, float* sh,
                                int32_t sh_row, int64_t n_leaves, float lr, float* grad_sigma, float* grad_sh,
                                int* flag, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const SegIn si{static_cast<const float4*>(sg.rec), sg.count, sg.n, sg.max_seg};
    cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    PO_DISPATCH(deg, false, {
        // 1. rays whose segments overflowed: re-traversal of the tree as it is, into the buffer
        carveout_once(k_backward<DEG, false, true>);
        k_backward<DEG, false, true><<<grid1d(n, 256), 256, 0, s>>>(tr, rays, n, dL_dC, aux, si, opt, grad_sigma,
                                                                    grad_sh, flag);
        // 2. stored segments: -lr * gradient straight into the payload
        carveout_once(k_backward_replay_sgd<DEG>);
        k_backward_replay_sgd<DEG><<<grid1d(n, 8), 256, 0, s>>>(tr, rays, n, dL_dC, aux, si, sigma, sh, sh_row, -lr);
        // 3. the buffer's SGD (and zeroing), a no-op launch unless step 1 wrote to it
        const int ne = 3 * ShDim<DEG>::B;
        const int64_t end = n_leaves * (1 + ne);
        unsigned g = grid1d(end, 256 * 4);
        if (g > 148 * 16) g = 148 * 16;
        k_sgd<<<g, 256, 0, s>>>(sigma, sh, sh_row, ne, n_leaves, grad_sigma, grad_sh, lr, 0, end, true, flag);
    });
    return cudaGetLastError();
}

}  // namespace po
