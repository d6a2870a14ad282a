/* =====================================================================================
 *  libplenoct -- C ABI of the B200 PlenOctree rendering hot path (forward + analytic
 *  backward).  PAPER.md = arXiv 2103.14024 source, cited as P:<line>; SURVEY.md §8(b)
 *  lists these entry points.  Readings of the paper (Q1..Q32) are in DESIGN.md.
 *
 *  Conventions shared by every call
 *  - Status codes, never exceptions.  On a non-OK status po_last_error() returns a
 *    thread-local message naming the failing argument / index.
 *  - "device" pointers are CUDA device pointers on the tree's device; "host" pointers
 *    are ordinary (pageable or pinned) host memory.  The library never keeps a pointer
 *    it was given after the call returns (device calls: after the stream work is done).
 *  - po_stream is a cudaStream_t passed as void* (NULL = legacy default stream).  All
 *    render / backward / update calls are asynchronous on that stream; the caller
 *    orders them (e.g. po_tree_sgd_step after every render that reads the tree).
 *  - Renders of one tree may run concurrently on different streams.  The persistent
 *    kernels keep their work counters per (tree, stream): up to 256 distinct streams per
 *    tree (PO_ERR_UNSUPPORTED beyond).  A destroyed stream's counters are reused only by a
 *    stream with the same handle, i.e. after the old one's work has been ordered before it.
 *  - CUDA launch and asynchronous errors map to PO_ERR_CUDA (a sticky error from an
 *    earlier kernel is reported by the next call that checks).
 *  - There is NO CPU fallback: every compute call runs CUDA kernels for sm_100a.
 * ===================================================================================== */
#ifndef PLENOCT_H_
#define PLENOCT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PO_OK = 0,
    PO_ERR_INVALID_ARG = 1,   /* bad size, NULL where required, non-orthonormal camera, ... */
    PO_ERR_INVALID_TREE = 2,  /* malformed child table, NaN/Inf payload, leaf deeper than D  */
    PO_ERR_OOM = 3,           /* cudaMalloc failed                                           */
    PO_ERR_CUDA = 4,          /* any other CUDA runtime error                                */
    PO_ERR_UNSUPPORTED = 5    /* sh_degree > 4, unknown payload, op not defined for payload  */
} po_status;

enum { PO_F32 = 0, PO_F16 = 1 };          /* leaf SH payload precision (sigma~ is always f32, reading Q20) */
enum { PO_SH_CS = 0, PO_SH_NO_CS = 1 };   /* real-SH sign convention (reading Q16; default CS)          */

typedef void* po_stream;                  /* cudaStream_t */
typedef struct po_tree po_tree;           /* opaque; owns the device copy of the tree */

/* Tree geometry and payload format ("stores density and SH coefficients at each
 * leaf"; cube bbox, reading Q4).  Leaf grid = 2^max_depth cells per axis. */
typedef struct {
    float bbox_min[3];
    float bbox_edge;      /* > 0, world units                                  */
    int32_t max_depth;    /* D, 1..15                                          */
    int32_t sh_degree;    /* l_max, 0..4 (4 = SH-25); B = (l_max+1)^2 coefs/channel */
    int32_t payload;      /* PO_F32 | PO_F16                                   */
    int32_t sh_sign;      /* PO_SH_CS | PO_SH_NO_CS                            */
    int32_t device;       /* CUDA ordinal the tree lives on                    */
    int32_t flags;        /* 0 or PO_TREE_NO_INDEX                             */
} po_tree_desc;

/* po_tree_desc.flags.  By default po_tree_create also builds the tree's dense level-(D-1) cell
 * index (D in 2..10): 8 bytes per cell of the 2^(D-1)-per-axis grid, 8 * 8^(D-1) bytes
 * (134 MB at D = 9, 1.07 GB at D = 10; po_tree_index_bytes), through which every traversal
 * kernel finds the box that contains a cell with one load (two for a depth-(D-1) node whose
 * leaves are not numbered consecutively in octant order) instead of a re-descent (same boxes
 * and t values, bit-identical results).  PO_TREE_NO_INDEX skips it (every kernel
 * then descends from the deepest common ancestor).  Nothing is built later: renders and
 * backward calls never allocate or synchronise for it. */
enum { PO_TREE_NO_INDEX = 1 };

/* Pinhole camera (reading Q5): c2w = camera-to-world 3x4 (OpenGL axes: x right, y up,
 * -z forward; the 3x3 block must be orthonormal within 1e-4), focal lengths and principal
 * point in pixels.  Pixel (i, j), row 0 at the top, shoots through its centre:
 * d_cam = ((i+0.5-cx)/fx, -(j+0.5-cy)/fy, -1), d = normalize(R d_cam), o = c2w[:,3]. */
typedef struct {
    float c2w[3][4];
    float fx, fy, cx, cy;
} po_camera;

/* gamma: early-stop threshold on transmittance, P:435-437 (0 disables; default 0.01).
 * background: c_N, the background light intensity of App. B.3 P:855-868 (default white). */
typedef struct {
    float gamma;
    float background[3];
} po_render_opts;

const char* po_last_error(void);
const char* po_version(void);

/* ---- a0: tree upload ---------------------------------------------------------------
 * child  host uint32[n_nodes][8]: entry = tag<<30 | index, tag 0 empty, 1 internal node,
 *        2 leaf (reading Q1); octant = 4*bx + 2*by + bz (reading Q2); node 0 is the root.
 * sigma  host float[n_leaves]: sigma~ (pre-ReLU density per world unit).
 * sh     host float[n_leaves][B][3]: k_l^m per RGB channel, (l,m) lexicographic with
 *        m = -l..l, basis-major / channel-minor (reading Q17).  Converted to
 *        fp16 (round to nearest even) when desc->payload == PO_F16.
 * Validates: every index in range and referenced at most once, every node reachable,
 * leaves no deeper than D, finite payload (else PO_ERR_INVALID_TREE).  Synchronous.
 * Builds the cell index unless desc->flags has PO_TREE_NO_INDEX; PO_ERR_OOM if the index does
 * not fit (the message names its size; nothing is created then).
 * The caller keeps ownership of the host arrays; *out owns device memory until
 * po_tree_destroy. */
po_status po_tree_create(const po_tree_desc* desc, const uint32_t* child, int64_t n_nodes, const float* sigma,
                         const float* sh, int64_t n_leaves, po_tree** out);
/* NEXT f3, spherical Gaussians (SG-25 with a tree of sh_degree 4): replace the
 * tree's per-ray basis by B = (sh_degree+1)^2 lobes G_b(d) = exp(lambda_b (d . p_b - 1)); the
 * leaf rows then hold one RGB coefficient per lobe (same layout), and render, backward (dL/dk
 * uses G_b for Y_b) and every other kernel use them.  axes host float[B][3] (normalised here,
 * reading Q36), lambda host float[B]; axes == NULL restores the SH basis.  The lobes are fixed
 * (the paper learns them in NeRF-SG, before conversion).  Waits for the device first;
 * PO_ERR_INVALID_ARG for a zero / non-finite axis or a non-finite bandwidth. */
po_status po_tree_set_sg_basis(po_tree* tree, const float* axes, const float* lambda);

/* Overwrite every leaf's sigma~ and SH coefficients from host arrays laid out as in
 * po_tree_create (fp16 payloads round to nearest-even); the structure is unchanged.  Waits for
 * the device first; PO_ERR_INVALID_ARG on a non-finite value (nothing written then).  With
 * po_tree_read_leaves this snapshots / restores a tree during optimisation (early stopping). */
po_status po_tree_write_leaves(po_tree* tree, const float* sigma, const float* sh);

/* Device pointers to the tree's own leaf payload, for collectives that update it in place
 * (reduce-scatter SGD: each rank updates its leaf shard, then an all-gather writes every
 * shard into every rank's tree).  sigma: float[capacity]; sh: rows of sh_row elements (fp32 or
 * fp16 per the payload), [capacity][sh_row]; capacity = n_leaves + 4096 spare zeroed leaves
 * that no node references, so equal-size chunks may run past n_leaves.  The tree keeps
 * ownership; writes must be stream-ordered after the renders that read the tree. */
po_status po_tree_leaf_payload(po_tree* tree, float** sigma, void** sh, int32_t* sh_row, int64_t* capacity);

/* Export (NEXT f2; "the entire optimization process is done in float32 ... after it we
 * store the PlenOctree with float16"): a new tree with the same structure and leaf values
 * re-uploaded with `payload` (PO_F16: SH coefficients rounded to nearest-even, sigma~ stays
 * fp32, reading Q20).  Synchronous; src is unchanged and independent of *out. */
po_status po_tree_convert(const po_tree* src, int32_t payload, po_tree** out);
po_status po_tree_destroy(po_tree* tree);
/* sh_row_bytes: padded device row of one leaf's SH payload (16-byte multiple). */
po_status po_tree_info(const po_tree* tree, int64_t* n_nodes, int64_t* n_leaves, int32_t* sh_row_bytes);
/* Device bytes of the tree's cell index (0 when PO_TREE_NO_INDEX or D outside 2..10). */
po_status po_tree_index_bytes(const po_tree* tree, int64_t* bytes);
/* Copy the current leaf values back (host float sigma[n_leaves], sh[n_leaves][B][3]; either may
 * be NULL).  Synchronous (device-wide sync of the tree's device). */
po_status po_tree_read_leaves(const po_tree* tree, float* sigma, float* sh);

/* ---- a1..a6: forward render (Eq. 1-2, Eq. 5) ----------
 * cams     device po_camera[n_cams]
 * out_rgb  device float[n_cams][H][W][3], fp32 linear RGB (reading Q30)
 * For each pixel: ray generation, bbox clip (t_near = max(0, entry)), ordered octree
 * descent over positive-length leaf segments, sigma = max(sigma~,0), alpha =
 * 1-exp(-sigma delta), c = sigmoid(sum k Y(d)), C += T alpha c, stop once T < gamma
 * (after compositing that segment, reading Q11), then C += T c_N.
 * Scheduling (no effect on pixel values): a single-view render hands its 16x16 blocks out
 * costliest first by the per-block costs the previous single-view render of the same W x H on
 * the same stream measured, the 32 costliest split into 16-lane tiles (the first render on a
 * stream: centre-out).  The first single-view render of a size on a stream allocates that
 * stream's order table (8 B per block + 772 B; PO_ERR_OOM if that fails); up to 256 streams per
 * tree (PO_ERR_UNSUPPORTED beyond). */
po_status po_render(const po_tree* tree, const po_camera* cams, int32_t n_cams, int32_t W, int32_t H,
                    const po_render_opts* opts, float* out_rgb, po_stream stream);

/* Tile sharding of one render (SURVEY 8(e) single-view latency mode): writes only the 16x16
 * pixel blocks at hand-out positions k with k % shard_count == shard_index (the centre-out
 * order, so every shard gets an equal mix of costly central and cheap border blocks); the
 * other pixels of out_rgb are left untouched.  Shards 0..shard_count-1 rendered into zeroed
 * images on as many GPUs and summed (e.g. a NCCL allreduce of the image) give exactly
 * po_render's image.  shard_count 1..4096. */
po_status po_render_shard(const po_tree* tree, const po_camera* cams, int32_t n_cams, int32_t W, int32_t H,
                          const po_render_opts* opts, int32_t shard_index, int32_t shard_count, float* out_rgb,
                          po_stream stream);

/* Same as po_render with HOST cameras and a HOST output image: copies the cameras in,
 * renders, copies the image out and synchronises the stream (end-to-end entry point).  If
 * out_rgb_host is pinned (cudaHostAlloc / torch pin_memory: device-mapped under unified
 * addressing) the kernel writes the pixels straight into it over PCIe while rendering
 * (PO_HOST_DIRECT=0 forces the staged copy); pageable memory is staged and copied.  A single
 * view's camera is passed by value (no camera copy).  A pinned buffer of more than 12 MiB with
 * 4 or more views is filled by a chunk pipeline instead: chunks of views rendered into device
 * buffers owned by the tree, each copied out on a second stream while the next one renders
 * (PO_HOST_PIPE=0 disables it).  A single view of more than 12 MiB is rendered into a device
 * image whose bands of block rows are copied out as the kernel completes them (stream
 * memory-operation waits on per-band counters; PO_HOST_BANDS=0 disables it).  Calls on one tree
 * are serialised for these pipelines. */
po_status po_render_host(const po_tree* tree, const po_camera* cams_host, int32_t n_cams, int32_t W, int32_t H,
                         const po_render_opts* opts, float* out_rgb_host, po_stream stream);

/* a1 on its own: the exact fp32 rays po_render generates, device float[n_cams][H][W][6] =
 * (origin, un-normalised direction R d_cam).  po_render(cams) equals po_render_rays(these rays)
 * bit for bit.  Each component is an IEEE round-to-nearest evaluation of
 * dx = ((i + 0.5) - cx) / fx, dy = -(((j + 0.5) - cy) / fy), d_k = (R_k0 dx + R_k1 dy) - R_k2. */
po_status po_camera_rays(const po_camera* cams, int32_t n_cams, int32_t W, int32_t H, float* rays, int32_t device,
                         po_stream stream);

/* Stored pass-1 segments (optional, training path).  The paper's pass 2 re-traverses every
 * ray to recover the per-segment weights; with 180 GB of HBM per GPU the forward
 * can instead store, for every sigma~ > 0 segment i it composites, the values pass 2 needs:
 *   record (k, ray r) = 8 floats at records + (k * n_rays + r) * 8 (segment-major, so the
 *   lanes of a warp touch adjacent records):
 *   (leaf index as uint32 bits, delta_i, w_i, T_{i+1}, c_r, c_g, c_b, 0)
 *   count[r] = number of sigma~ > 0 segments, or max_seg + 1 if they did not fit (pass 2 then
 *   re-traverses that ray, so any max_seg >= 0 is exact).
 * Pass 2 replays the records through the same arithmetic as the re-traversal: the gradients
 * are identical up to the order of the atomic sums.  Memory: max_seg * n_rays * 32 B
 * (c4: 192 x 1 M rays = 6.4 GB), caller-owned, 16-byte aligned. */
typedef struct {
    float* records;     /* device float[max_seg][n_rays][8] */
    int32_t* count;     /* device int32[n_rays] */
    int64_t n_rays;     /* batch size the buffer is laid out for */
    int32_t max_seg;
} po_segments;

/* Forward render of explicit rays.
 * rays       device float[n][6] = (origin xyz, direction xyz); the direction is normalised
 *            by the library (zero direction => that ray returns the background).
 * out_rgb    device float[n][3]
 * aux        device double[n][4] or NULL: (C_r, C_g, C_b, T_final) accumulated in double;
 *            po_render_backward uses it to skip its own first pass.
 * leaf_span  device uint32[n][2] or NULL (needs aux, 8-byte aligned): the smallest and
 *            largest index of the sigma~ > 0 leaves the ray composited -- exactly the leaves
 *            its backward writes (P:961-963 gates the rest) -- or (0xFFFFFFFF, 0) for none.
 *            Input of po_backward_plan (SURVEY 8(e) overlap of pass 2 with the allreduce).
 * segments   NULL or a po_segments buffer with n_rays == n (needs aux): written for pass 2. */
po_status po_render_rays(const po_tree* tree, const float* rays, int64_t n, const po_render_opts* opts,
                         float* out_rgb, double* aux, uint32_t* leaf_span, const po_segments* segments,
                         po_stream stream);

/* po_render_rays with a processing order: group_order = device int32[ceil(n/32)], a permutation
 * of the groups of 32 consecutive rays (group g = rays [32g, 32g+32)); warps claim the groups
 * in that order.  Scheduling only: every output is the same as po_render_rays' (bitwise).  A
 * batch whose costliest groups come first ends without a tail of long groups started late
 * (c4 pass 1 at gamma 0: the per-ray leaf count is a constant of the fixed tree structure,
 * DESIGN.md §6.2).  group_order must be a permutation (not checked: rays of groups it omits are
 * not rendered).  NULL = po_render_rays. */
po_status po_render_rays_ordered(const po_tree* tree, const float* rays, int64_t n, const po_render_opts* opts,
                                 const int32_t* group_order, float* out_rgb, double* aux, uint32_t* leaf_span,
                                 const po_segments* segments, po_stream stream);

/* ---- a7/a8: analytic backward (App. B.3: P:886-892 colour, P:938-947 density,
 * P:949-957 two passes, P:959-963 ReLU) -----------------------------------------------
 * dL_dC       device float[n][3], the loss gradient per ray (e.g. 2(C^ - C) for Eq. 3).
 * aux         device double[n][4] from po_render_rays with the same tree/rays/opts, or NULL
 *             (then the kernel runs its own first pass to get the total sum_k c_k w_k).
 * segments    NULL, or the po_segments that same po_render_rays call wrote (needs aux):
 *             rays whose segments fit are replayed without traversal.
 * grad_sigma  device float[n_leaves]      d L / d sigma~   (ACCUMULATED: +=)
 * grad_sh     device float[n_leaves][B][3] d L / d k         (ACCUMULATED: +=)
 * The caller zeroes the gradients; cross-ray summation order is nondeterministic.
 * opts->gamma applies exactly as in the forward (gamma = 0 is the paper-literal optimiser,
 * reading Q12). */
po_status po_render_backward(const po_tree* tree, const float* rays, int64_t n, const float* dL_dC,
                             const double* aux, const po_segments* segments, const po_render_opts* opts,
                             float* grad_sigma, float* grad_sh, po_stream stream);

/* ---- a8/a9 overlap: pass 2 in K chunks whose gradient ranges become final in order ------
 * Leaves are numbered depth first, so each subtree is a contiguous index range (a0).  Given
 * leaf bounds b_0 <= ... <= b_{K-1} = n_leaves, chunk j holds the rays whose lowest sigma~>0
 * leaf index lies in [b_{j-1}, b_j) (b_{-1} = 0).  A ray writes no leaf below that index
 * (P:961-963 gates sigma~ <= 0 leaves to zero), so once chunks 0..j have run the gradient of
 * leaves [0, b_j) is FINAL: its allreduce + SGD can start while chunks j+1.. run.
 * Rays with no sigma~>0 leaf write nothing and are in no chunk.
 *
 * po_backward_plan
 *   leaf_span      device uint32[n][2] from po_render_rays (same tree, rays, opts)
 *   K              1..64 chunks
 *   leaf_bounds    host int64[K] or NULL (then b_j = floor(n_leaves (j+1) / K)); must be
 *                  non-decreasing with b_{K-1} = n_leaves, else PO_ERR_INVALID_ARG
 *   perm           device int32[n] out: ray indices sorted by lowest leaf (stable, so the
 *                  caller's ray order is kept inside a key); n < 2^31
 *   chunk_ray_end  device int64[K] out: chunk j = perm[chunk_ray_end[j-1] .. chunk_ray_end[j])
 *   leaf_end       host int64[K] out or NULL: the bounds b_j used (known without a device sync)
 *   key_quantiles  device int64[K] out or NULL: bounds that would split THIS batch's rays into
 *                  K equal chunks (last = n_leaves); a caller may feed them back as the next
 *                  step's leaf_bounds (batches of one scene have similar distributions)
 * Stream-ordered; uses sort scratch cached in the tree, so plans on one tree must not run
 * concurrently on different streams.  The chunk bounds stay on the device: the chunks are
 * launched without waiting for the plan.
 *
 * po_render_backward_chunk: po_render_backward over chunk `chunk` of a plan (rays, dL_dC and
 * aux indexed through perm).  Running all K chunks equals one po_render_backward over the
 * rays up to the order of the floating-point sums; chunks may run concurrently on several
 * streams (the gradient accumulation is atomic). */
po_status po_backward_plan(po_tree* tree, const uint32_t* leaf_span, int64_t n, int32_t K, const int64_t* leaf_bounds,
                           int32_t* perm, int64_t* chunk_ray_end, int64_t* leaf_end, int64_t* key_quantiles,
                           po_stream stream);
po_status po_render_backward_chunk(const po_tree* tree, const float* rays, const int32_t* perm,
                                   const int64_t* chunk_ray_end, int32_t chunk, const float* dL_dC,
                                   const double* aux, const po_segments* segments, const po_render_opts* opts,
                                   float* grad_sigma, float* grad_sh, po_stream stream);

/* a8 + a9 fused for a single replica (one GPU, no gradient exchange): pass 2 with the plain
 * SGD update of P:492 / P:973 folded into it.  Each stored segment's contribution, times -lr,
 * is added atomically straight into the tree's sigma~ and k (so sigma~ -= lr * dL/dsigma~ and
 * k -= lr * dL/dk over the whole batch, Eq. 3's sum over rays), with no gradient buffer
 * and no separate update pass.  Equal to po_render_backward + po_tree_sgd_step up to the fp32
 * summation order.  Needs aux and segments from the po_render_rays call of this batch on this
 * tree (the tree must not change in between); rays whose segments overflowed max_seg are
 * re-traversed FIRST (on the unmodified tree) into grad_sigma / grad_sh, which must be zero on
 * entry and are applied and zeroed again at the end (a no-op launch when no ray overflowed).
 * fp32 trees only (PO_ERR_UNSUPPORTED otherwise); lr finite.  Mutates the tree: stream-order it
 * after every render that reads the tree, as for po_tree_sgd_step.  Not for world_size > 1,
 * where the summed gradient must cross ranks first. */
po_status po_render_backward_sgd(po_tree* tree, const float* rays, int64_t n, const float* dL_dC, const double* aux,
                                 const po_segments* segments, const po_render_opts* opts, float lr,
                                 float* grad_sigma, float* grad_sh, po_stream stream);

/* Deterministic pass 2 (NEXT f2 "deterministic-reduction mode"): the same gradients as
 * po_render_backward with stored segments, accumulated by a segmented reduction instead of
 * atomics -- every segment's contribution is emitted with its leaf as key, the records are
 * sorted by leaf (stable: ray order, then segment order) and each leaf's run is summed in that
 * fixed order and added once -- so repeated calls give bit-identical gradients (the atomic path
 * is order-nondeterministic, reading Q24).  Needs aux and segments from the same
 * po_render_rays call.  Rays whose segments overflowed max_seg still go through the atomic
 * re-traversal; n_overflow (device int32 or NULL) receives their number, and the result is
 * order-fixed iff it is 0.  Synchronises the stream once (the segment total sizes the sort);
 * scratch (~36 B per segment) is cached in the tree, so calls on one tree must not overlap. */
po_status po_render_backward_deterministic(const po_tree* tree, const float* rays, int64_t n, const float* dL_dC,
                                           const double* aux, const po_segments* segments,
                                           const po_render_opts* opts, float* grad_sigma, float* grad_sh,
                                           int32_t* n_overflow, po_stream stream);

/* Eq. (3) helper: dL_dC[i] = 2 (pred[i] - target[i]) over n*3 floats; if loss != NULL,
 * *loss (device double) = sum (pred - target)^2 (overwritten). */
po_status po_l2_loss_grad(const float* pred, const float* target, int64_t n, float* dL_dC, double* loss,
                          int32_t device, po_stream stream);

/* a9 update: plain SGD on an fp32 tree, in place:
 * sigma~ -= lr * grad_sigma, k -= lr * grad_sh.  PO_ERR_UNSUPPORTED for fp16 payloads. */
po_status po_tree_sgd_step(po_tree* tree, const float* grad_sigma, const float* grad_sh, float lr,
                           po_stream stream);
/* Same update restricted to parameter indices [begin, end) of the index space
 * [0, n_leaves) = sigma~ of leaf i, n_leaves + j = j-th element of grad_sh / sh (leaf-major,
 * [B][3] within a leaf).  Lets the caller update each gradient bucket as soon as its
 * allreduce has landed (a9 overlap).  PO_ERR_INVALID_ARG if the range is outside.
 * Entries whose gradient is exactly 0 (leaves no ray of the batch composited) are left
 * untouched (p - lr * 0 = p), so only touched rows are read-modify-written.
 * flags: PO_SGD_ZERO_GRAD also writes 0 over every consumed gradient entry, so the caller
 * needs no separate memset before the next backward (the gradients are then non-const). */
#define PO_SGD_ZERO_GRAD 1
po_status po_tree_sgd_step_range(po_tree* tree, float* grad_sigma, float* grad_sh, float lr, int64_t begin,
                                 int64_t end, int32_t flags, po_stream stream);

/* ---- NEXT rows on the same traversal ------------------------------------
 * po_render_depth (f4; "render the depth map", alpha maps P:468; reading Q34):
 *   alpha[i] = 1 - T_stop and depth[i] = sum_i w_i (t_in,i + t_out,i) / 2 over the segments
 *   composited up to termination (w_i as in Eq. 1-2, t in world units along the unit
 *   direction from the ray origin; the background adds nothing, so depth / alpha is the
 *   normalised depth).  rays device float[n][6]; alpha, depth device float[n]; sigma~ only.
 * po_leaf_max_alpha (f1, visibility filtering; reading Q33): for every leaf a ray
 *   composites before it terminates (opts->gamma), max_alpha[leaf] = max(max_alpha[leaf],
 *   1 - exp(-sigma delta)) -- "the maximum ray weight ... at each voxel" -- over all n rays.
 *   max_alpha device float[n_leaves], MAX-accumulated: the caller initialises it with values
 *   >= 0 (the max is taken on the IEEE bit patterns, which order like non-negative floats; 0 for a
 *   fresh pass) and may accumulate over several calls (all training views).  Leaves whose
 *   maximum stays below tau_w are the ones the paper removes. */
po_status po_render_depth(const po_tree* tree, const float* rays, int64_t n, const po_render_opts* opts,
                          float* alpha, float* depth, po_stream stream);
po_status po_leaf_max_alpha(const po_tree* tree, const float* rays, int64_t n, const po_render_opts* opts,
                            float* max_alpha, po_stream stream);

/* ---- parity / measurement helpers ----------------------------------------------------
 * po_trace: the visited-leaf sequence of each ray up to termination, produced by the very
 * traversal the product kernels run (po_render, po_render_rays, the backward and the NEXT-row
 * kernels: the level-(D-1) cell index when the tree has one).  leaf_ids device
 * int32[n][max_leaves] (first max_leaves, -1 padded; may be NULL when max_leaves == 0), counts
 * device int32[n] (leaves composited, sigma~<=0 leaves included, reading Q10), node_counts
 * device int32[n] or NULL (internal nodes, root included, whose box the processed interval
 * meets: a property of the classic descent, counted by a second launch of it).
 * flags: 0, or PO_TRACE_CLASSIC = everything from the classic descent from the deepest common
 * ancestor (the path of trees without an index); both visit the same leaves with the same t
 * values, which the GPU tests check bit for bit. */
#define PO_TRACE_CLASSIC 1
po_status po_trace(const po_tree* tree, const float* rays, int64_t n, const po_render_opts* opts,
                   int32_t max_leaves, int32_t* leaf_ids, int32_t* counts, int32_t* node_counts, int32_t flags,
                   po_stream stream);

/* po_render_stats: counters of the po_render traversal over n_cams views, ADDED to
 * device uint64 counters[7] = {leaf visits, leaf visits with sigma~ > 0 (SH row read),
 * internal nodes met (root included), rays that hit the bbox, boxes stepped through (leaf or
 * empty), of which leaf-level cells, sum over 8x4-pixel warps of the longest ray's boxes}. */
po_status po_render_stats(const po_tree* tree, const po_camera* cams, int32_t n_cams, int32_t W, int32_t H,
                          const po_render_opts* opts, unsigned long long* counters, po_stream stream);

/* ---- diagnostics: only in libraries built with -DPO_DIAG (PO_NVCC_EXTRA=-DPO_DIAG); the
 * symbols exist in every build and return PO_ERR_UNSUPPORTED otherwise ---------------------
 * po_ray_step_timing (measurement, SH-3 fp32 trees): the po_render_rays forward of n rays, one
 * thread each, recording for every box step k < max_steps of ray i two uint32 at
 * rec[(i * max_steps + k) * 2]: the SM cycles since the previous box step (the previous box's
 * leaf work, the neighbour step and this box's descent) and (child-entry loads of this descent)
 * << 8 | (log2 box edge in leaf cells) << 1 | (previous box was a composited leaf).  steps[i] =
 * number of box steps (may exceed max_steps).  Used to find the critical path of slow warps
 * (DESIGN.md §6.1); no image is written. */
po_status po_ray_step_timing(const po_tree* tree, const float* rays, int64_t n, const po_render_opts* opts,
                             int32_t max_steps, uint32_t* rec, int32_t* steps, po_stream stream);

/* po_render_timeline: po_render that also records, for every warp tile, device uint64
 * timeline[(ceil(W/16)*ceil(H/16)*n_cams + 192)*8][4] (record = hand-out position * 8 + tile)
 * = {globaltimer ns at tile start, at tile end, SM id << 32 | block index in its view,
 * view | split << 32 (0, or 8 | sub-block of a split block)} (scheduling analysis; same image). */
po_status po_render_timeline(const po_tree* tree, const po_camera* cams, int32_t n_cams, int32_t W, int32_t H,
                             const po_render_opts* opts, float* out_rgb, unsigned long long* timeline,
                             po_stream stream);

/* po_set_block_order: replaces the tree's block hand-out order for W x H renders by the host
 * array order[ceil(W/16)*ceil(H/16)] (hand-out position -> block index in raster order; a
 * permutation, checked).  Scheduling experiments only. */
po_status po_set_block_order(po_tree* tree, int32_t W, int32_t H, const uint32_t* order);

/* Number of kernel launches the library has issued since load (bench accounting). */
int64_t po_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PLENOCT_H_ */
