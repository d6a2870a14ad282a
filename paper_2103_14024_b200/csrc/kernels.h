// Internal launcher interface between the C-ABI layer (api.cu) and the kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "plenoct.h"
#include "traverse.cuh"

namespace po {

struct RenderOpts {
    float gamma;
    float bg[3];
    // tile sharding of the render (po_render_shard): this launch takes the blocks of hand-out
    // position k with k % shard_count == shard_index
    int32_t shard_index = 0, shard_count = 1;
    // k_render only: one view's camera by value (cams unused), so a host camera needs no copy
    int32_t cam_inline = 0;
    float cam[16] = {};
    // k_render only (po_render_host band pipeline): after each warp tile's store, add 1 to
    // band_done[block_row / band_rows] (cumulative 64-bit counters a copy stream waits on)
    unsigned long long* band_done = nullptr;
    int32_t band_rows = 0;
    // k_render only, single-view launches (cost-ordered hand-out, DESIGN.md §6.1 v13): non-null
    // = device uint32[n_blocks] per-block cost (max SM cycles of its warp tiles), zero on entry;
    // the last CTA then rewrites `order` (costliest block first) for the next launch on the
    // stream and zeroes the costs again.  `order` must then be a mutable per-stream table.
    unsigned* blk_cost = nullptr;
    // with blk_cost: the split_k costliest blocks are rendered as split_f (2, 4 or 8) sub-blocks
    // of 8 warp tiles with 32 / split_f active lanes each (4x4, 4x2 or 4x1 pixels), so the slowest
    // tiles of the frame have fewer rays; order[-1] holds the number of hand-out positions
    int32_t split_k = 0, split_f = 1;
    // with blk_cost: blocks after the split ones zipped (costliest, cheapest, 2nd costliest, ...)
    // so in-kernel image stores over PCIe (po_render_host) spread over the launch
    int32_t zip_order = 0;
    // k_render_rays_p only: NULL, or device int32[ceil(n/32)], a permutation of the 32-ray groups
    // giving the order in which warps claim them (scheduling only; outputs stay per ray)
    const int32_t* group_order = nullptr;
};

// work: 2 device uint32 counters, zero on entry, reset to zero by the kernel on exit.
// order: NULL (raster) or a device permutation of the ceil(W/16)*ceil(H/16) blocks of a view
// giving the order in which blocks are handed out.
// timeline: NULL, or device uint64[n_blocks * 8][4] receiving one record per warp tile
// (globaltimer start, end, smid << 32 | block, view) -- measurement mode of po_render_timeline.
cudaError_t launch_render(const DevTree& tr, int deg, bool f16, const po_camera* cams, int n_cams, int W, int H,
                          const RenderOpts& opt, float* out, unsigned* work, const unsigned* order,
                          unsigned long long* timeline, cudaStream_t s);
cudaError_t launch_ray_step_timing(const DevTree& tr, const float* rays, int64_t n, const RenderOpts& opt,
                                   int32_t max_steps, uint32_t* rec, int32_t* steps, cudaStream_t s);
cudaError_t launch_camera_rays(const po_camera* cams, int n_cams, int W, int H, float* rays, cudaStream_t s);
// stored pass-1 segments (po_segments): rec = float[max_seg][n][8] or null
struct Segments {
    void* rec;
    int32_t* count;
    int64_t n;
    int32_t max_seg;
};
cudaError_t launch_render_rays(const DevTree& tr, int deg, bool f16, const float* rays, int64_t n,
                               const RenderOpts& opt, float* out, double* aux, uint32_t* span, const Segments& sg,
                               cudaStream_t s, unsigned* work = nullptr);   // work: 2 zeroed counters -> persistent
cudaError_t launch_backward_chunk(const DevTree& tr, int deg, bool f16, const float* rays, const int32_t* perm,
                                  const int64_t* chunk_end, int chunk, const float* dL_dC, const double* aux,
                                  const Segments& sg, const RenderOpts& opt, float* grad_sigma, float* grad_sh,
                                  unsigned* work, cudaStream_t s);
cudaError_t launch_det_counts(const float* rays, int64_t n, const float* dL_dC, const Segments& sg, int32_t* cnt,
                              int32_t* n_overflow, cudaStream_t s);
cudaError_t launch_det_emit(const DevTree& tr, int deg, const float* rays, int64_t n, const float* dL_dC,
                            const double* aux, const Segments& sg, const int32_t* offs, uint32_t* key, uint32_t* val,
                            float4* contrib, int32_t* ray_of, cudaStream_t s);
cudaError_t launch_det_reduce(const DevTree& tr, int deg, const float* rays, const uint32_t* skey,
                              const uint32_t* sval, int64_t S, const float4* contrib, const int32_t* ray_of,
                              float* grad_sigma, float* grad_sh, cudaStream_t s);
cudaError_t launch_plan_keys(const uint32_t* span, int64_t n, uint32_t n_leaves, uint32_t* keys, int32_t* idx,
                             cudaStream_t s);
constexpr int kMaxPlanChunks = 64;
struct PlanBounds {
    int64_t b[kMaxPlanChunks];   // leaf bounds b_0 <= ... <= b_{K-1} = n_leaves
    int K;
};
cudaError_t launch_plan_ends(const uint32_t* sorted_keys, int64_t n, int64_t n_leaves, const PlanBounds& b,
                             int64_t* chunk_end, int64_t* quant, cudaStream_t s);
// overflow_only (with segments): skip the replay, re-traverse only the rays that overflowed
cudaError_t launch_backward(const DevTree& tr, int deg, bool f16, const float* rays, int64_t n, const float* dL_dC,
                            const double* aux, const Segments& sg, const RenderOpts& opt, float* grad_sigma,
                            float* grad_sh, cudaStream_t s, bool overflow_only = false);
// a8 + a9 fused for one replica (po_render_backward_sgd): overflow rays into grad_* (zero on
// entry, zero again on exit), stored segments' -lr * gradient straight into sigma / sh (rows of
// sh_row elements), then the buffer's SGD gated on the device flag the overflow kernel sets.
cudaError_t launch_backward_sgd(const DevTree& tr, int deg, const float* rays, int64_t n, const float* dL_dC,
                                const double* aux, const Segments& sg, const RenderOpts& opt, float* sigma, float* sh,
                                int32_t sh_row, int64_t n_leaves, float lr, float* grad_sigma, float* grad_sh,
                                int* flag, cudaStream_t s);
cudaError_t launch_render_depth(const DevTree& tr, const float* rays, int64_t n, float gamma, float* alpha,
                                float* depth, cudaStream_t s);
cudaError_t launch_leaf_max_alpha(const DevTree& tr, const float* rays, int64_t n, float gamma, float* max_alpha,
                                  cudaStream_t s);
cudaError_t launch_trace(const DevTree& tr, const float* rays, int64_t n, float gamma, int32_t max_leaves,
                         int32_t* leaf_ids, int32_t* counts, int32_t* node_counts, bool classic, cudaStream_t s);
cudaError_t launch_stats(const DevTree& tr, const po_camera* cams, int n_cams, int W, int H, float gamma,
                         unsigned long long* counters, cudaStream_t s);
cudaError_t launch_l2_loss(const float* pred, const float* target, int64_t n3, float* dL_dC, double* loss,
                           cudaStream_t s);
cudaError_t launch_sgd(float* sigma, float* sh, int32_t sh_row, int32_t ne, int64_t n_leaves, float* grad_sigma,
                       float* grad_sh, float lr, int64_t begin, int64_t end, bool zero_grad, cudaStream_t s);

}  // namespace po
