// C-ABI layer of libplenoct (include/plenoct.h): argument validation, tree upload (a0),
// device selection and kernel launches.  No compute happens here; there is no CPU path.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda.h>   // driver API types only (cuStreamWaitValue64 comes via cudaGetDriverEntryPoint)
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <utility>
#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.h"
#include "plenoct.h"

struct po_tree {
    po_tree_desc desc;
    int64_t n_nodes = 0, n_leaves = 0;
    int B = 0, ne = 0;          // basis size, 3B elements per leaf
    int sh_row = 0;             // padded row in elements
    int sh_row_bytes = 0;
    uint32_t* d_child = nullptr;
    float* d_sigma = nullptr;
    void* d_sh = nullptr;
    po_camera* d_cams = nullptr;   // scratch for po_render_host
    int cam_cap = 0;
    float* d_img = nullptr;        // scratch image for po_render_host
    size_t img_cap = 0;
    // po_render_host's chunked pipeline (multi-view renders into pinned buffers): two device
    // chunk buffers, a copy stream and its events, used under host_mu
    float* d_pipe = nullptr;
    size_t pipe_cap = 0;
    cudaStream_t pipe_stream = nullptr;
    cudaEvent_t pipe_ev[4] = {nullptr, nullptr, nullptr, nullptr};   // rendered[2], copied[2]
    // po_render_host band pipeline (one view): cumulative per-band tile counters for W x H
    unsigned long long* d_band = nullptr;
    int band_w = 0, band_h = 0;
    unsigned long long band_calls = 0;
    // centre-out order of the 16x16 pixel blocks of a W x H view (built once per size)
    unsigned* d_order = nullptr;
    int order_w = 0, order_h = 0;
    // the same, zipped with its reverse (po_render_host writing a pinned image over PCIe)
    unsigned* d_order_zip = nullptr;
    int zip_w = 0, zip_h = 0;
    std::mutex order_mu;
    // work counters of the persistent kernels: one block of kWorkStride words per CUDA stream
    // that launched on this tree (launches on one stream are serialised, so they may share
    // a block; the last CTA of each launch resets it).  Up to kWorkSlots distinct streams.
    static constexpr int kWorkSlots = 256;
    static constexpr int kWorkStride = 8;
    unsigned* d_work = nullptr;
    std::mutex work_mu;
    std::vector<cudaStream_t> work_streams;
    int slot_of(cudaStream_t s) {   // caller holds work_mu
        for (size_t i = 0; i < work_streams.size(); ++i)
            if (work_streams[i] == s) return (int)i;
        if ((int)work_streams.size() >= kWorkSlots) return -1;
        work_streams.push_back(s);
        return (int)work_streams.size() - 1;
    }
    unsigned* work_for(cudaStream_t s) {
        std::lock_guard<std::mutex> lk(work_mu);
        const int i = slot_of(s);
        return i < 0 ? nullptr : d_work + kWorkStride * i;
    }
    int* sgd_flag() { return reinterpret_cast<int*>(d_work + kWorkStride * kWorkSlots); }
    // cost-ordered hand-out of single-view renders (DESIGN.md §6.1 v13): per work slot (stream)
    // a device table [n_blocks] order + [n_blocks] per-block cost for one W x H, rewritten by
    // every single-view render on that stream for the next one
    struct StreamOrder {
        unsigned* d = nullptr;
        int W = 0, H = 0;
    };
    std::vector<StreamOrder> stream_order;   // indexed like work_streams, under work_mu
    std::vector<uint32_t> h_child;   // the caller's child table as given (po_tree_convert)
    uint2* d_grid = nullptr;         // dense level-(D-1) cell index (build_grid, at po_tree_create)
    size_t grid_bytes = 0;
    // the smallest box of level-(D-1) cells holding every occupied cell (leaf units; the whole
    // cube without an index): rays are clipped to it (DESIGN.md §6.1 v18)
    int occ_lo[3] = {-1, -1, -1}, occ_hi[3] = {-1, -1, -1};
    // po_render_host holds this for its whole body (camera / image / pipeline scratch)
    std::mutex host_mu;
    static constexpr int64_t kPayloadPad = 4096;   // spare zero leaves after the payload arrays
    float4* d_sg = nullptr;          // spherical-Gaussian lobes (po_tree_set_sg_basis) or null
    std::vector<float> h_sg;         // the same on the host, [B][4]
    // po_render_backward_deterministic scratch, grown on demand
    void* d_det = nullptr;
    size_t det_cap = 0;
    std::mutex det_mu;
    // po_backward_plan scratch (sort keys/values + CUB temp), grown on demand
    void* d_plan = nullptr;
    size_t plan_cap = 0;
    std::mutex plan_mu;
};

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

po_status fail(po_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
po_status fail(po_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

po_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return PO_OK;
    if (e == cudaErrorMemoryAllocation) return fail(PO_ERR_OOM, "%s: %s", where, cudaGetErrorString(e));
    return fail(PO_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

// Switches the calling thread to the tree's device for the duration of a call.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        err = cudaGetDevice(&prev);
        if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// Block hand-out order for the persistent render: blocks sorted by the distance of their
// centre from the image centre, so the costly on-object blocks of object-centred views go
// first and the last claims (the tail of the launch) are cheap background blocks.
// PO_RENDER_ORDER=raster disables it.  Returns NULL for raster order.
const unsigned* block_order(po_tree* t, int W, int H, cudaStream_t s, cudaError_t* err, bool zip = false) {
    static const bool raster = [] {
        const char* e = getenv("PO_RENDER_ORDER");
        return e && std::strcmp(e, "raster") == 0;
    }();
    *err = cudaSuccess;
    if (raster) return nullptr;
    std::lock_guard<std::mutex> lk(t->order_mu);
    unsigned*& d_ord = zip ? t->d_order_zip : t->d_order;
    int& ow = zip ? t->zip_w : t->order_w;
    int& oh = zip ? t->zip_h : t->order_h;
    if (d_ord && ow == W && oh == H) return d_ord;
    const int bx = (W + 15) / 16, by = (H + 15) / 16;
    std::vector<unsigned> ord((size_t)bx * by);
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = (unsigned)i;
    const double cx = W * 0.5, cy = H * 0.5;
    auto dist = [&](unsigned b) {
        const double x = (b % bx) * 16.0 + 8.0 - cx, y = (b / bx) * 16.0 + 8.0 - cy;
        return x * x + y * y;
    };
    std::stable_sort(ord.begin(), ord.end(), [&](unsigned a, unsigned b) { return dist(a) < dist(b); });
    if (zip) {   // centre, border, next-to-centre, next-to-border, ...: image stores spread in time
        std::vector<unsigned> z;
        z.reserve(ord.size());
        for (size_t i = 0, j = ord.size(); i < j;) {
            z.push_back(ord[i++]);
            if (i < j) z.push_back(ord[--j]);
        }
        ord.swap(z);
    }
    if ((*err = cudaStreamSynchronize(s)) != cudaSuccess) return nullptr;   // old table may be in use
    if (d_ord) cudaFree(d_ord);
    d_ord = nullptr;
    if ((*err = cudaMalloc(&d_ord, ord.size() * sizeof(unsigned))) != cudaSuccess) return nullptr;
    if ((*err = cudaMemcpy(d_ord, ord.data(), ord.size() * sizeof(unsigned), cudaMemcpyHostToDevice)) != cudaSuccess)
        return nullptr;
    ow = W;
    oh = H;
    return d_ord;
}

// The level-(D-1) cell index (kOptGrid, traverse.cuh DevTree::grid): for every cell of the
// 2^(D-1)-per-axis grid an (E, F) pair -- the level of the empty box containing it, a depth-(D-1)
// leaf's entry, a depth-(D-1) node's child-table entry, or, when that node's leaves are numbered
// consecutively in octant order (the depth-first numbering of gen/ and of the paper's trees), its
// occupancy mask and first leaf so a leaf-level step needs no child-table load (E = 0xFFFFFFFF: a
// coarser leaf, traversed the classic way).  Built on the host from the caller's child table
// inside po_tree_create (D in 2..10; 134 MB at D = 9, 1.07 GB at D = 10) unless the descriptor
// sets PO_TREE_NO_INDEX; read-only afterwards, so renders stay asynchronous and allocation-free.
// Returns the CUDA error of the upload (cudaSuccess when D is outside 2..10: every kernel then
// descends classically).
static cudaError_t build_grid(po_tree* t) {
    const int D = t->desc.max_depth;
    if (t->d_grid || D < 2 || D > 10) return cudaSuccess;
    const int G2 = 1 << (D - 1);
    std::vector<uint2> g((size_t)G2 * G2 * G2, make_uint2(0u, 0u));
    auto fill = [&](int x0, int y0, int z0, int n, uint32_t v) {   // grid cells [x0, x0+n)^3
        for (int x = x0; x < x0 + n; ++x)
            for (int y = y0; y < y0 + n; ++y)
                for (int z = z0; z < z0 + n; ++z) g[((size_t)x * G2 + y) * G2 + z] = make_uint2(v, 0u);
    };
    // a depth-(D-1) node: packed (mask, first leaf) when its leaves are consecutive in octant order
    auto node_entry = [&](uint32_t e) -> uint2 {
        const uint32_t node = e & ((1u << 30) - 1u);
        uint32_t mask = 0u, first = 0u, rank = 0u;
        bool packed = true;
        for (int oct = 0; oct < 8; ++oct) {
            const uint32_t c = t->h_child[(size_t)node * 8 + oct];
            if ((c >> 30) == 0u) continue;
            const uint32_t idx = c & ((1u << 30) - 1u);
            if ((c >> 30) != 2u || (rank == 0 ? false : idx != first + rank)) packed = false;
            if (rank == 0) first = idx;
            mask |= 1u << oct;
            ++rank;
        }
        if (packed && rank > 0) return make_uint2((3u << 30) | mask, first);
        return make_uint2(e, 0u);
    };
    // node at `level` with its box corner in grid cells (level-(D-1) units), box edge 2^(D-1-level)
    std::function<void(uint32_t, int, int, int, int)> rec = [&](uint32_t node, int level, int x0, int y0, int z0) {
        const int half = 1 << (D - 2 - level);   // child edge in grid cells (level < D-1 here)
        for (int oct = 0; oct < 8; ++oct) {
            const uint32_t e = t->h_child[(size_t)node * 8 + oct];
            const int cx = x0 + ((oct >> 2) & 1) * half, cy = y0 + ((oct >> 1) & 1) * half, cz = z0 + (oct & 1) * half;
            const uint32_t tag = e >> 30;
            if (tag == 1u) {
                if (level + 1 == D - 1) g[((size_t)cx * G2 + cy) * G2 + cz] = node_entry(e);
                else rec(e & ((1u << 30) - 1u), level + 1, cx, cy, cz);
            } else if (tag == 2u) {
                fill(cx, cy, cz, half, level + 1 == D - 1 ? e : 0xFFFFFFFFu);
            } else {
                fill(cx, cy, cz, half, (uint32_t)(level + 1));   // empty box at level+1
            }
        }
    };
    rec(0u, 0, 0, 0, 0);
    // Empty cells also carry their Chebyshev distance (in level-(D-1) cells, capped at 255) to
    // the nearest occupied cell, so the traversal can leave the empty cube around the ray's
    // cell in one step when that reaches further than the cell's octree box (DESIGN.md §6.1
    // v17).  Exact L-infinity distance transform: two raster passes of the 3x3x3 unit-weight
    // chamfer over a grid padded by one cell of distance 255.
    {
        const int P = G2 + 2;
        std::vector<uint8_t> dist((size_t)P * P * P, 255);
        auto at = [&](int x, int y, int z) -> size_t { return ((size_t)x * P + y) * P + z; };
        for (int x = 0; x < G2; ++x)
            for (int y = 0; y < G2; ++y)
                for (int z = 0; z < G2; ++z) {
                    const uint32_t E = g[((size_t)x * G2 + y) * G2 + z].x;
                    if ((E >> 30) != 0u) dist[at(x + 1, y + 1, z + 1)] = 0;   // node, leaf or coarse leaf
                }
        long off[13];
        int n_off = 0;
        for (int dx = -1; dx <= 1; ++dx)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dz = -1; dz <= 1; ++dz)
                    if (dx < 0 || (dx == 0 && (dy < 0 || (dy == 0 && dz < 0)))) off[n_off++] = ((long)dx * P + dy) * P + dz;
        uint8_t* dp = dist.data();
        for (int x = 1; x <= G2; ++x)
            for (int y = 1; y <= G2; ++y) {
                uint8_t* row = dp + at(x, y, 1);
                for (int z = 0; z < G2; ++z) {
                    int m = row[z];
                    if (m == 0) continue;
                    for (int k = 0; k < 13; ++k) m = std::min(m, row[z + off[k]] + 1);
                    row[z] = (uint8_t)std::min(m, 255);
                }
            }
        for (int x = G2; x >= 1; --x)
            for (int y = G2; y >= 1; --y) {
                uint8_t* row = dp + at(x, y, 1);
                for (int z = G2 - 1; z >= 0; --z) {
                    int m = row[z];
                    if (m == 0) continue;
                    for (int k = 0; k < 13; ++k) m = std::min(m, row[z - off[k]] + 1);
                    row[z] = (uint8_t)std::min(m, 255);
                }
            }
        for (int x = 0; x < G2; ++x)
            for (int y = 0; y < G2; ++y)
                for (int z = 0; z < G2; ++z) {
                    uint2& c = g[((size_t)x * G2 + y) * G2 + z];
                    if ((c.x >> 30) == 0u) c.x = (c.x & 0xFFu) | ((uint32_t)dist[at(x + 1, y + 1, z + 1)] << 8);
                }
    }
    {   // occupied bounding box (level-(D-1) cells, in leaf units); an empty tree keeps the cube
        int lo[3] = {G2, G2, G2}, hi[3] = {-1, -1, -1};
        for (int x = 0; x < G2; ++x)
            for (int y = 0; y < G2; ++y)
                for (int z = 0; z < G2; ++z)
                    if ((g[((size_t)x * G2 + y) * G2 + z].x >> 30) != 0u) {
                        const int v[3] = {x, y, z};
                        for (int k = 0; k < 3; ++k) {
                            lo[k] = std::min(lo[k], v[k]);
                            hi[k] = std::max(hi[k], v[k]);
                        }
                    }
        if (hi[0] >= 0)
            for (int k = 0; k < 3; ++k) {
                t->occ_lo[k] = 2 * lo[k];
                t->occ_hi[k] = 2 * (hi[k] + 1);
            }
    }
    uint2* d = nullptr;
    cudaError_t e = cudaMalloc(&d, g.size() * sizeof(uint2));
    if (e != cudaSuccess) {
        (void)cudaGetLastError();   // not sticky: po_tree_create reports it
        return e;
    }
    if ((e = cudaMemcpy(d, g.data(), g.size() * sizeof(uint2), cudaMemcpyHostToDevice)) != cudaSuccess) {
        (void)cudaGetLastError();
        cudaFree(d);
        return e;
    }
    t->d_grid = d;
    t->grid_bytes = g.size() * sizeof(uint2);
    return cudaSuccess;
}

po::DevTree dev_tree(const po_tree* t) {
    po::DevTree d;
    d.grid = t->d_grid;
    d.child = t->d_child;
    d.sigma = t->d_sigma;
    d.sh = t->d_sh;
    d.sh_row = t->sh_row;
    d.depth = t->desc.max_depth;
    for (int k = 0; k < 3; ++k) d.bmin[k] = t->desc.bbox_min[k];
    d.scale = (float)std::ldexp(1.0, t->desc.max_depth) / t->desc.bbox_edge;
    d.odd_sign = t->desc.sh_sign == PO_SH_NO_CS ? -1.f : 1.f;
    d.sg = t->d_sg;
    const float G = (float)std::ldexp(1.0, t->desc.max_depth);
    for (int k = 0; k < 3; ++k) {
        d.clip_lo[k] = t->occ_lo[k] >= 0 ? (float)t->occ_lo[k] : 0.f;
        d.clip_hi[k] = t->occ_hi[k] >= 0 ? (float)t->occ_hi[k] : G;
    }
    return d;
}

po_status check_opts(const po_render_opts* o, po::RenderOpts* out) {
    if (!o) return fail(PO_ERR_INVALID_ARG, "opts is NULL");
    if (!(o->gamma >= 0.f && o->gamma <= 1.f)) return fail(PO_ERR_INVALID_ARG, "gamma %g outside [0,1]", o->gamma);
    out->gamma = o->gamma;
    for (int k = 0; k < 3; ++k) {
        if (!std::isfinite(o->background[k])) return fail(PO_ERR_INVALID_ARG, "background[%d] not finite", k);
        out->bg[k] = o->background[k];
    }
    return PO_OK;
}

po_status check_tree(const po_tree* t) {
    if (!t || !t->d_child) return fail(PO_ERR_INVALID_ARG, "tree is NULL or destroyed");
    return PO_OK;
}

po_status launched(cudaError_t e, const char* where) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_status(e, where);
}

}  // namespace

extern "C" {

const char* po_last_error(void) { return g_err.c_str(); }
const char* po_version(void) { return "libplenoct 0.1 sm_100a"; }
int64_t po_launch_count(void) { return g_launches.load(); }

po_status po_tree_create(const po_tree_desc* desc, const uint32_t* child, int64_t n_nodes, const float* sigma,
                         const float* sh, int64_t n_leaves, po_tree** out) {
    if (!out) return fail(PO_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!desc) return fail(PO_ERR_INVALID_ARG, "desc is NULL");
    if (!(desc->bbox_edge > 0.f) || !std::isfinite(desc->bbox_edge))
        return fail(PO_ERR_INVALID_ARG, "bbox_edge must be finite and > 0");
    for (int k = 0; k < 3; ++k)
        if (!std::isfinite(desc->bbox_min[k])) return fail(PO_ERR_INVALID_ARG, "bbox_min[%d] not finite", k);
    if (desc->max_depth < 1 || desc->max_depth > po::kMaxDepth)
        return fail(PO_ERR_INVALID_ARG, "max_depth %d outside [1,%d]", desc->max_depth, po::kMaxDepth);
    if (desc->sh_degree < 0 || desc->sh_degree > 4)
        return fail(PO_ERR_UNSUPPORTED, "sh_degree %d unsupported (0..4)", desc->sh_degree);
    if (desc->payload != PO_F32 && desc->payload != PO_F16)
        return fail(PO_ERR_UNSUPPORTED, "payload %d unsupported", desc->payload);
    if (desc->sh_sign != PO_SH_CS && desc->sh_sign != PO_SH_NO_CS)
        return fail(PO_ERR_INVALID_ARG, "sh_sign %d invalid", desc->sh_sign);
    if (desc->flags & ~PO_TREE_NO_INDEX) return fail(PO_ERR_INVALID_ARG, "unknown desc flags 0x%x", desc->flags);
    if (n_nodes < 1 || !child) return fail(PO_ERR_INVALID_ARG, "need n_nodes >= 1 and a child table");
    if (n_leaves < 0 || n_leaves > (int64_t)po::kIdxMask + 1 || n_nodes > ((int64_t)1 << 29))
        return fail(PO_ERR_INVALID_ARG, "n_leaves (<= 2^30) / n_nodes (<= 2^29) out of range");
    if (n_leaves > 0 && (!sigma || !sh)) return fail(PO_ERR_INVALID_ARG, "sigma / sh NULL with n_leaves > 0");

    // ---- structural validation: BFS from the root with levels ----
    const int D = desc->max_depth;
    std::vector<int8_t> node_level((size_t)n_nodes, -1);
    std::vector<uint8_t> leaf_seen((size_t)n_leaves, 0);
    std::vector<int64_t> queue;
    queue.reserve((size_t)n_nodes);
    queue.push_back(0);
    node_level[0] = 0;
    for (size_t qi = 0; qi < queue.size(); ++qi) {
        const int64_t nd = queue[qi];
        const int L = node_level[(size_t)nd];
        for (int o = 0; o < 8; ++o) {
            const uint32_t e = child[nd * 8 + o];
            const uint32_t tag = e >> 30, idx = e & po::kIdxMask;
            if (tag == po::kTagEmpty) continue;
            if (tag == po::kTagInternal) {
                if ((int64_t)idx >= n_nodes)
                    return fail(PO_ERR_INVALID_TREE, "node %lld slot %d: child node %u out of range", (long long)nd, o, idx);
                if (L + 1 >= D)
                    return fail(PO_ERR_INVALID_TREE, "node %lld slot %d: internal node at level %d >= max_depth", (long long)nd, o, L + 1);
                if (node_level[idx] >= 0 || idx == 0)
                    return fail(PO_ERR_INVALID_TREE, "node %u referenced twice", idx);
                node_level[idx] = (int8_t)(L + 1);
                queue.push_back(idx);
            } else if (tag == po::kTagLeaf) {
                if ((int64_t)idx >= n_leaves)
                    return fail(PO_ERR_INVALID_TREE, "node %lld slot %d: leaf %u out of range", (long long)nd, o, idx);
                if (leaf_seen[idx]) return fail(PO_ERR_INVALID_TREE, "leaf %u referenced twice", idx);
                leaf_seen[idx] = 1;
            } else {
                return fail(PO_ERR_INVALID_TREE, "node %lld slot %d: bad tag 3", (long long)nd, o);
            }
        }
    }
    if ((int64_t)queue.size() != n_nodes)
        return fail(PO_ERR_INVALID_TREE, "%lld of %lld nodes unreachable from the root",
                    (long long)(n_nodes - (int64_t)queue.size()), (long long)n_nodes);
    const int B = (desc->sh_degree + 1) * (desc->sh_degree + 1);
    const int ne = 3 * B;
    for (int64_t i = 0; i < n_leaves; ++i) {
        if (!std::isfinite(sigma[i])) return fail(PO_ERR_INVALID_TREE, "sigma of leaf %lld not finite", (long long)i);
        for (int j = 0; j < ne; ++j)
            if (!std::isfinite(sh[i * ne + j]))
                return fail(PO_ERR_INVALID_TREE, "sh of leaf %lld element %d not finite", (long long)i, j);
    }

    // ---- device layout: child table as is; sigma~ SoA; SH rows padded to 16 B ----
    const bool f16 = desc->payload == PO_F16;
    const int per16 = f16 ? 8 : 4;
    const int row = (ne + per16 - 1) / per16 * per16;
    const size_t elt = f16 ? 2 : 4;
    DeviceGuard g(desc->device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    po_tree* t = new po_tree();
    t->desc = *desc;
    t->n_nodes = n_nodes;
    t->n_leaves = n_leaves;
    t->B = B;
    t->ne = ne;
    t->sh_row = row;
    t->sh_row_bytes = (int)(row * elt);
    auto cleanup = [&](po_status s) {
        po_tree_destroy(t);
        return s;
    };
    cudaError_t e = cudaMalloc(&t->d_child, (size_t)n_nodes * 8 * sizeof(uint32_t));
    if (e != cudaSuccess) return cleanup(cuda_status(e, "cudaMalloc(child)"));
    // payload arrays carry kPayloadPad zeroed spare leaves at the end (never referenced by the
    // child table) so sharded updates can gather equal-size leaf chunks in place
    // (po_tree_leaf_payload, reduce-scatter SGD)
    const int64_t n_alloc = n_leaves + po_tree::kPayloadPad;
    e = cudaMalloc(&t->d_sigma, (size_t)n_alloc * sizeof(float));
    if (e != cudaSuccess) return cleanup(cuda_status(e, "cudaMalloc(sigma)"));
    e = cudaMalloc(&t->d_sh, (size_t)n_alloc * row * elt);
    if (e != cudaSuccess) return cleanup(cuda_status(e, "cudaMalloc(sh)"));
    if ((e = cudaMemset(t->d_sigma, 0, (size_t)n_alloc * sizeof(float))) == cudaSuccess)
        e = cudaMemset(t->d_sh, 0, (size_t)n_alloc * row * elt);
    if (e != cudaSuccess) return cleanup(cuda_status(e, "cudaMalloc(sh)"));
    // work counters + one device flag (po_render_backward_sgd: "an overflow ray wrote the buffer")
    const size_t work_words = (size_t)po_tree::kWorkStride * po_tree::kWorkSlots + 1;
    e = cudaMalloc(&t->d_work, sizeof(unsigned) * work_words);
    if (e != cudaSuccess) return cleanup(cuda_status(e, "cudaMalloc(work)"));
    e = cudaMemset(t->d_work, 0, sizeof(unsigned) * work_words);
    if (e != cudaSuccess) return cleanup(cuda_status(e, "memset(work)"));
    // the device child table is the caller's (ABI encoding, reading Q1)
    e = cudaMemcpy(t->d_child, child, (size_t)n_nodes * 8 * sizeof(uint32_t), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cleanup(cuda_status(e, "upload child"));
    if (n_leaves > 0) {
        e = cudaMemcpy(t->d_sigma, sigma, (size_t)n_leaves * sizeof(float), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cleanup(cuda_status(e, "upload sigma"));
        // pack rows in chunks through a host staging buffer
        const int64_t chunk = 1 << 16;
        std::vector<uint8_t> stage((size_t)chunk * row * elt);
        for (int64_t s0 = 0; s0 < n_leaves; s0 += chunk) {
            const int64_t nn = std::min(chunk, n_leaves - s0);
            std::memset(stage.data(), 0, stage.size());
            for (int64_t i = 0; i < nn; ++i) {
                const float* src = sh + (s0 + i) * ne;
                if (f16) {
                    __half* dst = reinterpret_cast<__half*>(stage.data()) + i * row;
                    for (int j = 0; j < ne; ++j) dst[j] = __float2half_rn(src[j]);
                } else {
                    float* dst = reinterpret_cast<float*>(stage.data()) + i * row;
                    std::memcpy(dst, src, ne * sizeof(float));
                }
            }
            e = cudaMemcpy(static_cast<uint8_t*>(t->d_sh) + (size_t)s0 * row * elt, stage.data(), (size_t)nn * row * elt,
                           cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return cleanup(cuda_status(e, "upload sh"));
        }
    }
    t->h_child.assign(child, child + (size_t)n_nodes * 8);
    if (!(desc->flags & PO_TREE_NO_INDEX)) {
        e = build_grid(t);
        if (e != cudaSuccess)
            return cleanup(fail(e == cudaErrorMemoryAllocation ? PO_ERR_OOM : PO_ERR_CUDA,
                                "level-(D-1) cell index (%.0f MB): %s; PO_TREE_NO_INDEX creates the tree without it",
                                std::ldexp(1.0, 3 * (D - 1)) * 8 / 1e6, cudaGetErrorString(e)));
    }
    *out = t;
    return PO_OK;
}

po_status po_tree_set_sg_basis(po_tree* t, const float* axes, const float* lambda) {
    if (po_status s = check_tree(t)) return s;
    const int B = t->B;
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    cudaError_t e = cudaDeviceSynchronize();   // no render may be reading the old basis
    if (e != cudaSuccess) return cuda_status(e, "sync");
    if (!axes) {   // back to spherical harmonics
        if (t->d_sg) cudaFree(t->d_sg);
        t->d_sg = nullptr;
        t->h_sg.clear();
        return PO_OK;
    }
    if (!lambda) return fail(PO_ERR_INVALID_ARG, "lambda NULL");
    std::vector<float> h((size_t)B * 4);
    for (int b = 0; b < B; ++b) {
        const double x = axes[3 * b], y = axes[3 * b + 1], z = axes[3 * b + 2];
        const double n = std::sqrt(x * x + y * y + z * z);
        if (!(n > 0.0) || !std::isfinite(n) || !std::isfinite(lambda[b]))
            return fail(PO_ERR_INVALID_ARG, "lobe %d: zero / non-finite axis or bandwidth", b);
        h[4 * b] = (float)(x / n);
        h[4 * b + 1] = (float)(y / n);
        h[4 * b + 2] = (float)(z / n);
        h[4 * b + 3] = lambda[b];
    }
    if (!t->d_sg && (e = cudaMalloc(&t->d_sg, sizeof(float4) * B)) != cudaSuccess)
        return cuda_status(e, "cudaMalloc(sg)");
    if ((e = cudaMemcpy(t->d_sg, h.data(), sizeof(float4) * B, cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_status(e, "upload sg");
    t->h_sg = h;
    return PO_OK;
}

po_status po_tree_write_leaves(po_tree* t, const float* sigma, const float* sh) {
    if (po_status s = check_tree(t)) return s;
    if (t->n_leaves == 0) return PO_OK;
    if (!sigma || !sh) return fail(PO_ERR_INVALID_ARG, "sigma / sh NULL");
    for (int64_t i = 0; i < t->n_leaves; ++i) {
        if (!std::isfinite(sigma[i])) return fail(PO_ERR_INVALID_ARG, "sigma of leaf %lld not finite", (long long)i);
        for (int j = 0; j < t->ne; ++j)
            if (!std::isfinite(sh[i * t->ne + j]))
                return fail(PO_ERR_INVALID_ARG, "sh of leaf %lld not finite", (long long)i);
    }
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    cudaError_t e = cudaDeviceSynchronize();   // stream-ordered writers of the tree finish first
    if (e != cudaSuccess) return cuda_status(e, "sync");
    if ((e = cudaMemcpy(t->d_sigma, sigma, (size_t)t->n_leaves * sizeof(float), cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_status(e, "write sigma");
    const bool f16 = t->desc.payload == PO_F16;
    const size_t elt = f16 ? 2 : 4;
    std::vector<uint8_t> buf((size_t)t->n_leaves * t->sh_row * elt, 0);
    for (int64_t i = 0; i < t->n_leaves; ++i)
        for (int j = 0; j < t->ne; ++j) {
            if (f16) reinterpret_cast<__half*>(buf.data())[i * t->sh_row + j] = __float2half_rn(sh[i * t->ne + j]);
            else reinterpret_cast<float*>(buf.data())[i * t->sh_row + j] = sh[i * t->ne + j];
        }
    if ((e = cudaMemcpy(t->d_sh, buf.data(), buf.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_status(e, "write sh");
    return PO_OK;
}

po_status po_tree_leaf_payload(po_tree* t, float** sigma, void** sh, int32_t* sh_row, int64_t* capacity) {
    if (po_status s = check_tree(t)) return s;
    if (sigma) *sigma = t->d_sigma;
    if (sh) *sh = t->d_sh;
    if (sh_row) *sh_row = t->sh_row;
    if (capacity) *capacity = t->n_leaves + po_tree::kPayloadPad;
    return PO_OK;
}

po_status po_tree_convert(const po_tree* src, int32_t payload, po_tree** out) {
    if (!out) return fail(PO_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (po_status s = check_tree(src)) return s;
    std::vector<float> sigma((size_t)src->n_leaves), sh((size_t)src->n_leaves * src->ne);
    if (po_status s = po_tree_read_leaves(src, sigma.data(), sh.data())) return s;
    po_tree_desc d = src->desc;
    d.payload = payload;
    po_status st = po_tree_create(&d, src->h_child.data(), src->n_nodes, sigma.data(), sh.data(), src->n_leaves, out);
    if (st == PO_OK && !src->h_sg.empty()) {   // keep a spherical-Gaussian basis
        std::vector<float> ax((size_t)src->B * 3), lam((size_t)src->B);
        for (int b = 0; b < src->B; ++b) {
            for (int k = 0; k < 3; ++k) ax[3 * b + k] = src->h_sg[4 * b + k];
            lam[b] = src->h_sg[4 * b + 3];
        }
        st = po_tree_set_sg_basis(*out, ax.data(), lam.data());
        if (st != PO_OK) {
            po_tree_destroy(*out);
            *out = nullptr;
        }
    }
    return st;
}

po_status po_tree_destroy(po_tree* t) {
    if (!t) return PO_OK;
    DeviceGuard g(t->desc.device);
    if (t->d_child) cudaFree(t->d_child);
    if (t->d_sigma) cudaFree(t->d_sigma);
    if (t->d_sh) cudaFree(t->d_sh);
    if (t->d_cams) cudaFree(t->d_cams);
    if (t->d_work) cudaFree(t->d_work);
    if (t->d_img) cudaFree(t->d_img);
    if (t->d_pipe) cudaFree(t->d_pipe);
    if (t->d_band) cudaFree(t->d_band);
    for (cudaEvent_t ev : t->pipe_ev)
        if (ev) cudaEventDestroy(ev);
    if (t->pipe_stream) cudaStreamDestroy(t->pipe_stream);
    if (t->d_order) cudaFree(t->d_order);
    if (t->d_order_zip) cudaFree(t->d_order_zip);
    for (auto& so : t->stream_order)
        if (so.d) cudaFree(so.d);
    if (t->d_grid) cudaFree(t->d_grid);
    if (t->d_plan) cudaFree(t->d_plan);
    if (t->d_det) cudaFree(t->d_det);
    if (t->d_sg) cudaFree(t->d_sg);
    t->d_child = nullptr;
    delete t;
    return PO_OK;
}

po_status po_tree_info(const po_tree* t, int64_t* n_nodes, int64_t* n_leaves, int32_t* sh_row_bytes) {
    if (po_status s = check_tree(t)) return s;
    if (n_nodes) *n_nodes = t->n_nodes;
    if (n_leaves) *n_leaves = t->n_leaves;
    if (sh_row_bytes) *sh_row_bytes = t->sh_row_bytes;
    return PO_OK;
}

po_status po_tree_index_bytes(const po_tree* t, int64_t* bytes) {
    if (po_status s = check_tree(t)) return s;
    if (!bytes) return fail(PO_ERR_INVALID_ARG, "bytes is NULL");
    *bytes = (int64_t)t->grid_bytes;
    return PO_OK;
}

po_status po_tree_read_leaves(const po_tree* t, float* sigma, float* sh) {
    if (po_status s = check_tree(t)) return s;
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_status(e, "sync");
    if (t->n_leaves == 0) return PO_OK;
    if (sigma) {
        e = cudaMemcpy(sigma, t->d_sigma, (size_t)t->n_leaves * sizeof(float), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_status(e, "read sigma");
    }
    if (sh) {
        const bool f16 = t->desc.payload == PO_F16;
        const size_t elt = f16 ? 2 : 4;
        std::vector<uint8_t> buf((size_t)t->n_leaves * t->sh_row * elt);
        e = cudaMemcpy(buf.data(), t->d_sh, buf.size(), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_status(e, "read sh");
        for (int64_t i = 0; i < t->n_leaves; ++i)
            for (int j = 0; j < t->ne; ++j)
                sh[i * t->ne + j] = f16 ? __half2float(reinterpret_cast<const __half*>(buf.data())[i * t->sh_row + j])
                                        : reinterpret_cast<const float*>(buf.data())[i * t->sh_row + j];
    }
    return PO_OK;
}

static po_status check_image(int32_t n_cams, int32_t W, int32_t H) {
    if (n_cams < 0 || W <= 0 || H <= 0) return fail(PO_ERR_INVALID_ARG, "need n_cams >= 0, W > 0, H > 0");
    if (n_cams > 65535) return fail(PO_ERR_INVALID_ARG, "n_cams > 65535 per call");
    return PO_OK;
}

static po_status check_cams_host(const po_camera* c, int32_t n) {
    for (int i = 0; i < n; ++i) {
        if (!(c[i].fx > 0.f) || !(c[i].fy > 0.f)) return fail(PO_ERR_INVALID_ARG, "camera %d: focal <= 0", i);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double dot = 0.0;
                for (int k = 0; k < 3; ++k) dot += (double)c[i].c2w[k][a] * c[i].c2w[k][b];
                if (std::fabs(dot - (a == b ? 1.0 : 0.0)) > 1e-4)
                    return fail(PO_ERR_INVALID_ARG, "camera %d: rotation not orthonormal", i);
            }
    }
    return PO_OK;
}

// The stream's cost-ordered table for single-view W x H renders, uint32: [0] = number of
// hand-out positions, [1, 1 + nb + kSplitExtra) = order (split blocks expanded), then nb costs.
// Set up on first use or a size change with the centre-out order and zero costs, copied on the
// stream (no host sync except when an old table of another size is freed).
constexpr int kSplitMaxK = 64, kSplitMaxF = 4;
constexpr size_t kSplitExtra = (size_t)kSplitMaxK * (kSplitMaxF - 1);
static unsigned* stream_order_table(po_tree* t, cudaStream_t s, int W, int H, const unsigned* centre, cudaError_t* err) {
    *err = cudaSuccess;
    const size_t nb = (size_t)((W + 15) / 16) * ((H + 15) / 16);
    const unsigned n_pos = (unsigned)nb;
    std::lock_guard<std::mutex> lk(t->work_mu);
    const int slot = t->slot_of(s);
    if (slot < 0) return nullptr;
    if ((int)t->stream_order.size() <= slot) t->stream_order.resize(slot + 1);
    po_tree::StreamOrder& so = t->stream_order[slot];
    if (so.d && so.W == W && so.H == H) return so.d;
    if (so.d) {
        if ((*err = cudaStreamSynchronize(s)) != cudaSuccess) return nullptr;   // the old table may be in use
        cudaFree(so.d);
        so.d = nullptr;
    }
    if ((*err = cudaMalloc(&so.d, (1 + 2 * nb + kSplitExtra) * sizeof(unsigned))) != cudaSuccess) {
        (void)cudaGetLastError();   // reported by the caller, not left for the next launch check
        so.d = nullptr;
        return nullptr;
    }
    // (a pageable source is staged before cudaMemcpyAsync returns)
    if ((*err = cudaMemcpyAsync(so.d, &n_pos, sizeof(unsigned), cudaMemcpyHostToDevice, s)) != cudaSuccess ||
        (*err = cudaMemcpyAsync(so.d + 1, centre, nb * sizeof(unsigned), cudaMemcpyDeviceToDevice, s)) != cudaSuccess ||
        (*err = cudaMemsetAsync(so.d + 1 + nb + kSplitExtra, 0, nb * sizeof(unsigned), s)) != cudaSuccess) {
        (void)cudaGetLastError();
        cudaFree(so.d);
        so.d = nullptr;
        return nullptr;
    }
    so.W = W;
    so.H = H;
    return so.d;
}

// (split_k, split_f) of cost-ordered renders: the costliest blocks rendered with fewer lanes per
// warp tile (DESIGN.md §6.1 v14); PO_SPLIT_K / PO_SPLIT_F override it in diagnostics builds.
static std::pair<int, int> split_cfg() {
    static const std::pair<int, int> cfg = [] {
        int k = 32, f = 2;
#ifdef PO_DIAG
        if (const char* e = getenv("PO_SPLIT_K")) k = atoi(e);
        if (const char* e = getenv("PO_SPLIT_F")) f = atoi(e);
#endif
        if (f != 1 && f != 2 && f != 4 && f != 8) f = 1;
        k = k < 0 ? 0 : (k > kSplitMaxK ? kSplitMaxK : k);
        if (f > 1 && (size_t)k * (f - 1) > kSplitExtra) k = (int)(kSplitExtra / (f - 1));   // table room
        return std::make_pair(f == 1 ? 0 : k, f);
    }();
    return cfg;
}

// Block hand-out order and launch of the persistent render kernel.  Single-view renders hand
// blocks out costliest first by the costs the previous single-view render of the same size on
// the same stream measured (temporal coherence of a moving camera; the first one uses the
// centre-out order); other launches use the centre-out order (DESIGN.md §6.1 v13).
// PO_RENDER_ORDER=centre keeps the centre-out order for every launch, =raster raster order.
static po_status render_scheduled(po_tree* t, const po_camera* cams, int n_cams, int W, int H,
                                  const po::RenderOpts& o, float* out, cudaStream_t s, const char* where,
                                  unsigned long long* timeline = nullptr, bool zip = false, bool raster = false) {
    static const bool centre_only = [] {
        const char* e = getenv("PO_RENDER_ORDER");
        return e && (std::strcmp(e, "centre") == 0 || std::strcmp(e, "raster") == 0);
    }();
    cudaError_t e = cudaSuccess;
    const unsigned* order = raster ? nullptr : block_order(t, W, H, s, &e, zip);
    if (e != cudaSuccess) return cuda_status(e, "block order");
    unsigned* work = t->work_for(s);
    if (!work) return fail(PO_ERR_UNSUPPORTED, "%s: more than %d distinct streams on one tree", where, po_tree::kWorkSlots);
    po::RenderOpts o2 = o;
    const size_t nb = (size_t)((W + 15) / 16) * ((H + 15) / 16);
    if (order != nullptr && !centre_only && n_cams == 1 && o.shard_count == 1 && nb <= 16384) {
        unsigned* tab = stream_order_table(t, s, W, H, order, &e);
        if (e != cudaSuccess) return cuda_status(e, "stream block order");
        if (tab) {
            order = tab + 1;
            o2.blk_cost = tab + 1 + nb + kSplitExtra;
            o2.split_k = split_cfg().first;
            o2.split_f = split_cfg().second;
            o2.zip_order = zip ? 1 : 0;
        }
    }
    return launched(po::launch_render(dev_tree(t), t->desc.sh_degree, t->desc.payload == PO_F16, cams, n_cams, W, H, o2,
                                      out, work, order, timeline, s),
                    where);
}

po_status po_render(const po_tree* t, const po_camera* cams, int32_t n_cams, int32_t W, int32_t H,
                    const po_render_opts* opts, float* out_rgb, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    if (po_status s = check_image(n_cams, W, H)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (n_cams == 0) return PO_OK;
    if (!cams || !out_rgb) return fail(PO_ERR_INVALID_ARG, "cams / out_rgb NULL");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    po_tree* tm = const_cast<po_tree*>(t);   // only scratch (work counters, block order) is mutated
    return render_scheduled(tm, cams, n_cams, W, H, o, out_rgb, (cudaStream_t)stream, "po_render");
}

po_status po_render_shard(const po_tree* t, const po_camera* cams, int32_t n_cams, int32_t W, int32_t H,
                          const po_render_opts* opts, int32_t shard_index, int32_t shard_count, float* out_rgb,
                          po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    if (po_status s = check_image(n_cams, W, H)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (shard_count < 1 || shard_count > 4096 || shard_index < 0 || shard_index >= shard_count)
        return fail(PO_ERR_INVALID_ARG, "need 0 <= shard_index < shard_count <= 4096");
    if (n_cams == 0) return PO_OK;
    if (!cams || !out_rgb) return fail(PO_ERR_INVALID_ARG, "cams / out_rgb NULL");
    o.shard_index = shard_index;
    o.shard_count = shard_count;
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    po_tree* tm = const_cast<po_tree*>(t);
    return render_scheduled(tm, cams, n_cams, W, H, o, out_rgb, (cudaStream_t)stream, "po_render_shard");
}

po_status po_render_host(const po_tree* tc, const po_camera* cams_host, int32_t n_cams, int32_t W, int32_t H,
                         const po_render_opts* opts, float* out_host, po_stream stream) {
    po_tree* t = const_cast<po_tree*>(tc);   // only the camera scratch is mutated
    if (po_status s = check_tree(t)) return s;
    if (po_status s = check_image(n_cams, W, H)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (n_cams == 0) return PO_OK;
    if (!cams_host || !out_host) return fail(PO_ERR_INVALID_ARG, "cams / out NULL");
    if (po_status s = check_cams_host(cams_host, n_cams)) return s;
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    // one host render per tree at a time: the camera, image and pipeline scratch are per tree
    // (the call synchronises its stream before returning, so this costs no overlap)
    std::lock_guard<std::mutex> host_lk(t->host_mu);
    cudaStream_t s = (cudaStream_t)stream;
    if (t->cam_cap < n_cams) {
        if (t->d_cams) cudaFree(t->d_cams);
        t->d_cams = nullptr;
        t->cam_cap = 0;
        cudaError_t e = cudaMalloc(&t->d_cams, sizeof(po_camera) * (size_t)n_cams);
        if (e != cudaSuccess) return cuda_status(e, "cudaMalloc(cams)");
        t->cam_cap = n_cams;
    }
    cudaError_t e = cudaSuccess;
    if (n_cams == 1) {   // one view travels in the kernel's parameters: no H2D copy on the stream
        o.cam_inline = 1;
        std::memcpy(o.cam, cams_host, sizeof(po_camera));
    } else {
        e = cudaMemcpyAsync(t->d_cams, cams_host, sizeof(po_camera) * (size_t)n_cams, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_status(e, "H2D cams");
    }
    const size_t out_bytes = (size_t)n_cams * W * H * 3 * sizeof(float);
    // A pinned (page-locked, device-mapped) output buffer is written by the kernel itself over
    // PCIe while it renders, so the image transfer overlaps the render instead of following
    // it; pageable buffers go through the device scratch image and one D2H copy.
    static const bool direct_ok = [] {
        const char* ev = getenv("PO_HOST_DIRECT");
        return !(ev && std::strcmp(ev, "0") == 0);
    }();
    float* direct = nullptr;
    if (direct_ok) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, out_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer != nullptr)
            direct = static_cast<float*>(pa.devicePointer);
        else
            (void)cudaGetLastError();   // pageable memory: not an error
    }
    // Multi-view renders into a pinned buffer whose transfer outlasts the render (c2: 200 views,
    // 1.5 GB): the copy engine moves data faster than SM stores into host memory (55.7 vs 47-50
    // GB/s, tools/micro/hostwrite.cu), so views are rendered in chunks into device buffers and
    // each chunk's D2H copy runs on a second stream while the next chunk renders.
    static const bool pipe_ok = [] {
        const char* ev = getenv("PO_HOST_PIPE");
        return !(ev && std::strcmp(ev, "0") == 0);
    }();
    if (direct && pipe_ok && n_cams >= 4 && out_bytes > ((size_t)12 << 20)) {
        const int chunk = n_cams >= 32 ? 16 : (n_cams + 1) / 2;   // views per render launch
        const size_t view_floats = (size_t)W * H * 3;
        const size_t cfloats = (size_t)chunk * view_floats;
        if (t->pipe_stream == nullptr) {
            if ((e = cudaStreamCreateWithFlags(&t->pipe_stream, cudaStreamNonBlocking)) != cudaSuccess)
                return cuda_status(e, "copy stream");
            for (cudaEvent_t& ev : t->pipe_ev)
                if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
                    return cuda_status(e, "copy events");
        }
        if (t->pipe_cap < 2 * cfloats) {
            if ((e = cudaStreamSynchronize(s)) != cudaSuccess || (e = cudaStreamSynchronize(t->pipe_stream)) != cudaSuccess)
                return cuda_status(e, "sync");
            if (t->d_pipe) cudaFree(t->d_pipe);
            t->d_pipe = nullptr;
            t->pipe_cap = 0;
            if ((e = cudaMalloc((void**)&t->d_pipe, 2 * cfloats * sizeof(float))) != cudaSuccess)
                return cuda_status(e, "cudaMalloc(chunk buffers)");
            t->pipe_cap = 2 * cfloats;
        }
        po_status st = PO_OK;
        for (int k = 0, v0 = 0; v0 < n_cams && st == PO_OK; ++k, v0 += chunk) {
            const int nv = std::min(chunk, n_cams - v0), b = k & 1;
            float* buf = t->d_pipe + (size_t)b * cfloats;
            if (k >= 2 && (e = cudaStreamWaitEvent(s, t->pipe_ev[2 + b], 0)) != cudaSuccess) {   // buffer copied out
                st = cuda_status(e, "wait copy");
                break;
            }
            st = render_scheduled(t, t->d_cams + v0, nv, W, H, o, buf, s, "po_render_host");
            if (st != PO_OK) break;
            if ((e = cudaEventRecord(t->pipe_ev[b], s)) != cudaSuccess ||
                (e = cudaStreamWaitEvent(t->pipe_stream, t->pipe_ev[b], 0)) != cudaSuccess ||
                (e = cudaMemcpyAsync(out_host + (size_t)v0 * view_floats, buf, (size_t)nv * view_floats * sizeof(float),
                                     cudaMemcpyDeviceToHost, t->pipe_stream)) != cudaSuccess ||
                (e = cudaEventRecord(t->pipe_ev[2 + b], t->pipe_stream)) != cudaSuccess)
                st = cuda_status(e, "chunk copy");
        }
        cudaError_t e1 = cudaStreamSynchronize(t->pipe_stream), e2 = cudaStreamSynchronize(s);
        if (st == PO_OK && e1 != cudaSuccess) st = cuda_status(e1, "sync");
        if (st == PO_OK && e2 != cudaSuccess) st = cuda_status(e2, "sync");
        return st;
    }
    // One large view into a pinned buffer: render into a device image in raster block order and let a
    // copy stream move each band of block rows as soon as its last tile is stored (the kernel
    // counts stored tiles per band; cuStreamWaitValue64 gates each band's D2H copy), so the
    // copy engine (55.7 GB/s) streams the image while the rest renders and only the last band's
    // copy follows the kernel.  Needs 64-bit stream memory operations; PO_HOST_BANDS=0 (or no
    // support) keeps the in-kernel stores below.
    using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
    static const WaitFn wait64 = []() -> WaitFn {
        const char* ev = getenv("PO_HOST_BANDS");
        if (ev && std::strcmp(ev, "0") == 0) return nullptr;
        void* fp = nullptr;
        void* ga = nullptr;
        cudaDriverEntryPointQueryResult q1, q2;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &fp, cudaEnableDefault, &q1) != cudaSuccess ||
            q1 != cudaDriverEntryPointSuccess ||
            cudaGetDriverEntryPoint("cuDeviceGetAttribute", &ga, cudaEnableDefault, &q2) != cudaSuccess ||
            q2 != cudaDriverEntryPointSuccess) {
            (void)cudaGetLastError();
            return nullptr;
        }
        int dev = 0, ok = 0;
        cudaGetDevice(&dev);
        using AttrFn = CUresult (*)(int*, CUdevice_attribute, CUdevice);
        if (reinterpret_cast<AttrFn>(ga)(&ok, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, dev) != CUDA_SUCCESS ||
            !ok)
            return nullptr;
        return reinterpret_cast<WaitFn>(fp);
    }();
    // Only for images above 12 MiB: a smaller image moves faster than it renders, and its last
    // bands (the costly centre rows finish last) would be copied after the kernel -- in-kernel
    // stores win there (c1 800x800: 3700 vs 2545 FPS end to end; c3 1920x1080: 1878 vs 1126).
    if (direct && n_cams == 1 && wait64 != nullptr && out_bytes > ((size_t)12 << 20)) {
        const int by_n = (H + 15) / 16, bx_n = (W + 15) / 16;
        const int band_rows = (by_n + 7) / 8;   // 8 bands
        const int nb = (by_n + band_rows - 1) / band_rows;
        if (t->pipe_stream == nullptr) {
            if ((e = cudaStreamCreateWithFlags(&t->pipe_stream, cudaStreamNonBlocking)) != cudaSuccess)
                return cuda_status(e, "copy stream");
            for (cudaEvent_t& ev : t->pipe_ev)
                if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
                    return cuda_status(e, "copy events");
        }
        if (t->d_band == nullptr || t->band_w != W || t->band_h != H) {   // counters restart at 0
            if ((e = cudaStreamSynchronize(s)) != cudaSuccess || (e = cudaStreamSynchronize(t->pipe_stream)) != cudaSuccess)
                return cuda_status(e, "sync");
            if (t->d_band) cudaFree(t->d_band);
            t->d_band = nullptr;
            if ((e = cudaMalloc((void**)&t->d_band, 8 * sizeof(unsigned long long))) != cudaSuccess)
                return cuda_status(e, "cudaMalloc(band counters)");
            if ((e = cudaMemset(t->d_band, 0, 8 * sizeof(unsigned long long))) != cudaSuccess)
                return cuda_status(e, "memset(band counters)");
            t->band_w = W;
            t->band_h = H;
            t->band_calls = 0;
        }
        if (t->img_cap < out_bytes) {
            if ((e = cudaStreamSynchronize(s)) != cudaSuccess || (e = cudaStreamSynchronize(t->pipe_stream)) != cudaSuccess)
                return cuda_status(e, "sync");
            if (t->d_img) cudaFree(t->d_img);
            t->d_img = nullptr;
            t->img_cap = 0;
            if ((e = cudaMalloc((void**)&t->d_img, out_bytes)) != cudaSuccess) return cuda_status(e, "cudaMalloc(image)");
            t->img_cap = out_bytes;
        }
        // the copies of the previous call on this tree are done with d_img before it is rewritten
        if ((e = cudaEventRecord(t->pipe_ev[2], t->pipe_stream)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(s, t->pipe_ev[2], 0)) != cudaSuccess)
            return cuda_status(e, "order");
        const unsigned long long call = ++t->band_calls;
        po::RenderOpts ob = o;
        ob.band_done = t->d_band;
        ob.band_rows = band_rows;
        po_status st = render_scheduled(t, t->d_cams, 1, W, H, ob, t->d_img, s, "po_render_host", nullptr, false, true);
        const size_t row_floats = (size_t)W * 3;
        for (int b = 0; b < nb && st == PO_OK; ++b) {
            const int br0 = b * band_rows, br1 = std::min(by_n, br0 + band_rows);
            const int r0 = br0 * 16, r1 = std::min(H, br1 * 16);
            const cuuint64_t target = (cuuint64_t)call * (cuuint64_t)bx_n * (br1 - br0) * 8;   // 8 tiles per block
            CUresult ce = wait64((CUstream)t->pipe_stream, (CUdeviceptr)(t->d_band + b), target, CU_STREAM_WAIT_VALUE_GEQ);
            if (ce != CUDA_SUCCESS) {
                st = fail(PO_ERR_CUDA, "cuStreamWaitValue64 failed (%d)", (int)ce);
                break;
            }
            if ((e = cudaMemcpyAsync(out_host + (size_t)r0 * row_floats, t->d_img + (size_t)r0 * row_floats,
                                     (size_t)(r1 - r0) * row_floats * sizeof(float), cudaMemcpyDeviceToHost,
                                     t->pipe_stream)) != cudaSuccess)
                st = cuda_status(e, "band copy");
        }
        cudaError_t e1 = cudaStreamSynchronize(t->pipe_stream), e2 = cudaStreamSynchronize(s);
        if (st == PO_OK && e1 != cudaSuccess) st = cuda_status(e1, "sync");
        if (st == PO_OK && e2 != cudaSuccess) st = cuda_status(e2, "sync");
        return st;
    }
    if (direct) {
        // Block order for in-kernel image stores over PCIe (GPU stores into mapped pinned memory
        // reach 47-50 GB/s, tools/micro/hostwrite.cu).  Centre-out hands the cheap border blocks
        // out last, so half the image is stored in a burst near the end of the render and the
        // PCIe backlog outlasts the kernel; zipping the order with its reverse spreads the stores
        // over the render.  That pays while the image moves faster than it renders (c1 800x800,
        // 7.7 MB: 3708 vs 3495 FPS end to end); when the transfer itself is the bound (c3
        // 1920x1080, 24.9 MB: 1268-1313 vs 1383-1419) centre-out measured better.  Threshold
        // 12 MiB per launch (~250 us at 50 GB/s, about one c1 render); PO_HOST_ORDER=centre|zip
        // overrides it.
        static const int host_order = [] {
            const char* ev = getenv("PO_HOST_ORDER");
            if (ev && std::strcmp(ev, "centre") == 0) return 0;
            if (ev && std::strcmp(ev, "zip") == 0) return 1;
            return -1;
        }();
        const bool zip = host_order >= 0 ? host_order == 1 : out_bytes <= ((size_t)12 << 20);
        po_status st = render_scheduled(t, t->d_cams, n_cams, W, H, o, direct, s, "po_render_host", nullptr, zip);
        e = cudaStreamSynchronize(s);
        if (st == PO_OK && e != cudaSuccess) st = cuda_status(e, "sync");
        return st;
    }
    if (t->img_cap < out_bytes) {   // grows once; later calls reuse it (no per-call allocation)
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_status(e, "sync");
        if (t->d_img) cudaFree(t->d_img);
        t->d_img = nullptr;
        t->img_cap = 0;
        e = cudaMalloc((void**)&t->d_img, out_bytes);
        if (e != cudaSuccess) return cuda_status(e, "cudaMalloc(image)");
        t->img_cap = out_bytes;
    }
    po_status st = render_scheduled(t, t->d_cams, n_cams, W, H, o, t->d_img, s, "po_render_host");
    if (st == PO_OK) {
        e = cudaMemcpyAsync(out_host, t->d_img, out_bytes, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) st = cuda_status(e, "D2H image");
    }
    e = cudaStreamSynchronize(s);
    if (st == PO_OK && e != cudaSuccess) st = cuda_status(e, "sync");
    return st;
}

po_status po_camera_rays(const po_camera* cams, int32_t n_cams, int32_t W, int32_t H, float* rays, int32_t device,
                         po_stream stream) {
    if (po_status s = check_image(n_cams, W, H)) return s;
    if (n_cams == 0) return PO_OK;
    if (!cams || !rays) return fail(PO_ERR_INVALID_ARG, "cams / rays NULL");
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    return launched(po::launch_camera_rays(cams, n_cams, W, H, rays, (cudaStream_t)stream), "po_camera_rays");
}

// po_segments -> launcher struct; n_expect < 0 skips the batch-size check (chunked backward)
static po_status check_segments(const po_segments* sg, int64_t n_expect, const void* aux, po::Segments* out) {
    *out = po::Segments{nullptr, nullptr, 0, 0};
    if (!sg) return PO_OK;
    if (!aux) return fail(PO_ERR_INVALID_ARG, "segments need aux (pass-1 / pass-2 pairing)");
    if ((!sg->records && sg->max_seg > 0) || !sg->count) return fail(PO_ERR_INVALID_ARG, "segments: NULL records / count");
    if (sg->max_seg < 0) return fail(PO_ERR_INVALID_ARG, "segments: max_seg < 0");
    if (((uintptr_t)sg->records & 15u) != 0) return fail(PO_ERR_INVALID_ARG, "segments: records not 16-byte aligned");
    if (sg->n_rays < 0 || (n_expect >= 0 && sg->n_rays != n_expect))
        return fail(PO_ERR_INVALID_ARG, "segments: n_rays %lld does not match the batch", (long long)sg->n_rays);
    *out = po::Segments{sg->records, sg->count, sg->n_rays, sg->max_seg};
    return PO_OK;
}

po_status po_render_rays(const po_tree* t, const float* rays, int64_t n, const po_render_opts* opts, float* out_rgb,
                         double* aux, uint32_t* leaf_span, const po_segments* segments, po_stream stream) {
    return po_render_rays_ordered(t, rays, n, opts, nullptr, out_rgb, aux, leaf_span, segments, stream);
}

po_status po_render_rays_ordered(const po_tree* t, const float* rays, int64_t n, const po_render_opts* opts,
                                 const int32_t* group_order, float* out_rgb, double* aux, uint32_t* leaf_span,
                                 const po_segments* segments, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (n > (int64_t)INT32_MAX * 32) return fail(PO_ERR_INVALID_ARG, "n too large for 32-ray groups");
    o.group_order = group_order;
    if (n < 0) return fail(PO_ERR_INVALID_ARG, "n < 0");
    if (leaf_span && !aux) return fail(PO_ERR_INVALID_ARG, "leaf_span needs aux (pass-1 mode)");
    if (leaf_span && ((uintptr_t)leaf_span & 7u) != 0) return fail(PO_ERR_INVALID_ARG, "leaf_span not 8-byte aligned");
    po::Segments sg;
    if (po_status s = check_segments(segments, n, aux, &sg)) return s;
    if (n == 0) return PO_OK;
    if (!rays || !out_rgb) return fail(PO_ERR_INVALID_ARG, "rays / out_rgb NULL");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    po_tree* tm = const_cast<po_tree*>(t);   // only the work counters are mutated
    unsigned* work = tm->work_for((cudaStream_t)stream);
    if (!work) return fail(PO_ERR_UNSUPPORTED, "more than %d distinct streams on one tree", po_tree::kWorkSlots);
    return launched(po::launch_render_rays(dev_tree(t), t->desc.sh_degree, t->desc.payload == PO_F16, rays, n, o,
                                           out_rgb, aux, leaf_span, sg, (cudaStream_t)stream, work),
                    "po_render_rays");
}

po_status po_backward_plan(po_tree* t, const uint32_t* leaf_span, int64_t n, int32_t K, const int64_t* leaf_bounds,
                           int32_t* perm, int64_t* chunk_ray_end, int64_t* leaf_end, int64_t* key_quantiles,
                           po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    if (n < 0 || n > (int64_t)INT32_MAX) return fail(PO_ERR_INVALID_ARG, "n outside [0, 2^31)");
    if (K < 1 || K > po::kMaxPlanChunks) return fail(PO_ERR_INVALID_ARG, "K outside [1, %d]", po::kMaxPlanChunks);
    if (!chunk_ray_end || (n > 0 && (!leaf_span || !perm))) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    if (t->n_leaves >= (int64_t)0xFFFFFFFFu) return fail(PO_ERR_UNSUPPORTED, "n_leaves >= 2^32");
    po::PlanBounds pb{};
    pb.K = K;
    for (int32_t j = 0; j < K; ++j) {
        pb.b[j] = leaf_bounds ? leaf_bounds[j] : t->n_leaves * (int64_t)(j + 1) / K;
        if (pb.b[j] < (j ? pb.b[j - 1] : 0) || pb.b[j] > t->n_leaves)
            return fail(PO_ERR_INVALID_ARG, "leaf_bounds not non-decreasing in [0, n_leaves]");
    }
    if (pb.b[K - 1] != t->n_leaves) return fail(PO_ERR_INVALID_ARG, "leaf_bounds[K-1] != n_leaves");
    if (leaf_end)
        for (int32_t j = 0; j < K; ++j) leaf_end[j] = pb.b[j];
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(chunk_ray_end, 0, sizeof(int64_t) * K, s);
        if (e == cudaSuccess && key_quantiles) {
            std::vector<int64_t> q((size_t)K, t->n_leaves);
            e = cudaMemcpyAsync(key_quantiles, q.data(), sizeof(int64_t) * K, cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);   // q is a stack buffer
        }
        return e == cudaSuccess ? PO_OK : cuda_status(e, "po_backward_plan (n = 0)");
    }
    // keys = lowest sigma~>0 leaf per ray (n_leaves when the ray has none), sorted stably
    // with the ray index as value: rays keep their relative order inside equal keys
    int end_bit = 1;
    while (end_bit < 32 && ((uint64_t)1 << end_bit) <= (uint64_t)t->n_leaves) ++end_bit;
    size_t cub_bytes = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)n, 0, end_bit, s);
    if (e != cudaSuccess) return cuda_status(e, "cub sizing");
    const size_t arr = ((size_t)n * 4 + 255) / 256 * 256;
    const size_t need = 3 * arr + cub_bytes;
    std::lock_guard<std::mutex> lk(t->plan_mu);
    if (t->plan_cap < need) {
        if (t->d_plan) cudaFree(t->d_plan);
        t->d_plan = nullptr;
        t->plan_cap = 0;
        e = cudaMalloc(&t->d_plan, need);
        if (e != cudaSuccess) return cuda_status(e, "cudaMalloc(plan scratch)");
        t->plan_cap = need;
    }
    char* base = static_cast<char*>(t->d_plan);
    uint32_t* keys_in = reinterpret_cast<uint32_t*>(base);
    uint32_t* keys_out = reinterpret_cast<uint32_t*>(base + arr);
    int32_t* idx_in = reinterpret_cast<int32_t*>(base + 2 * arr);
    void* tmp = base + 3 * arr;
    if ((e = po::launch_plan_keys(leaf_span, n, (uint32_t)t->n_leaves, keys_in, idx_in, s)) != cudaSuccess)
        return cuda_status(e, "plan keys");
    g_launches.fetch_add(1);
    e = cub::DeviceRadixSort::SortPairs(tmp, cub_bytes, keys_in, keys_out, idx_in, perm, (int)n, 0, end_bit, s);
    if (e != cudaSuccess) return cuda_status(e, "cub sort");
    return launched(po::launch_plan_ends(keys_out, n, t->n_leaves, pb, chunk_ray_end, key_quantiles, s),
                    "po_backward_plan");
}

po_status po_render_backward_chunk(const po_tree* t, const float* rays, const int32_t* perm,
                                   const int64_t* chunk_ray_end, int32_t chunk, const float* dL_dC, const double* aux,
                                   const po_segments* segments, const po_render_opts* opts, float* grad_sigma,
                                   float* grad_sh, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    po::Segments sg;
    if (po_status s = check_segments(segments, -1, aux, &sg)) return s;
    if (chunk < 0) return fail(PO_ERR_INVALID_ARG, "chunk < 0");
    if (!rays || !perm || !chunk_ray_end || !dL_dC || !grad_sigma || !grad_sh)
        return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    if (((uintptr_t)grad_sh & 15u) != 0) return fail(PO_ERR_INVALID_ARG, "grad_sh must be 16-byte aligned");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    po_tree* mt = const_cast<po_tree*>(t);   // work counters only
    unsigned* work = mt->work_for((cudaStream_t)stream);
    if (!work) return fail(PO_ERR_UNSUPPORTED, "more than %d distinct streams on one tree", po_tree::kWorkSlots);
    if (segments != nullptr && aux != nullptr) g_launches.fetch_add(1);   // + the replay kernel
    return launched(po::launch_backward_chunk(dev_tree(t), t->desc.sh_degree, t->desc.payload == PO_F16, rays, perm,
                                              chunk_ray_end, chunk, dL_dC, aux, sg, o, grad_sigma, grad_sh,
                                              work, (cudaStream_t)stream),
                    "po_render_backward_chunk");
}

po_status po_render_backward(const po_tree* t, const float* rays, int64_t n, const float* dL_dC, const double* aux,
                             const po_segments* segments, const po_render_opts* opts, float* grad_sigma,
                             float* grad_sh, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (n < 0) return fail(PO_ERR_INVALID_ARG, "n < 0");
    po::Segments sg;
    if (po_status s = check_segments(segments, n, aux, &sg)) return s;
    if (n == 0) return PO_OK;
    if (!rays || !dL_dC || !grad_sigma || !grad_sh) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    if (((uintptr_t)grad_sh & 15u) != 0) return fail(PO_ERR_INVALID_ARG, "grad_sh must be 16-byte aligned");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    if (segments != nullptr && aux != nullptr) g_launches.fetch_add(1);   // replay + overflow re-traversal
    return launched(po::launch_backward(dev_tree(t), t->desc.sh_degree, t->desc.payload == PO_F16, rays, n, dL_dC, aux,
                                        sg, o, grad_sigma, grad_sh, (cudaStream_t)stream),
                    "po_render_backward");
}

po_status po_render_backward_sgd(po_tree* t, const float* rays, int64_t n, const float* dL_dC, const double* aux,
                                 const po_segments* segments, const po_render_opts* opts, float lr,
                                 float* grad_sigma, float* grad_sh, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (t->desc.payload != PO_F32) return fail(PO_ERR_UNSUPPORTED, "po_render_backward_sgd needs an fp32 payload");
    if (!std::isfinite(lr)) return fail(PO_ERR_INVALID_ARG, "lr is not finite");
    if (n < 0) return fail(PO_ERR_INVALID_ARG, "n < 0");
    if (!segments || !aux) return fail(PO_ERR_INVALID_ARG, "po_render_backward_sgd needs aux and segments");
    po::Segments sg;
    if (po_status s = check_segments(segments, n, aux, &sg)) return s;
    if (n == 0) return PO_OK;
    if (!rays || !dL_dC || !grad_sigma || !grad_sh) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    if (((uintptr_t)grad_sh & 15u) != 0) return fail(PO_ERR_INVALID_ARG, "grad_sh must be 16-byte aligned");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    g_launches.fetch_add(2);   // overflow re-traversal + fused replay + gated SGD
    return launched(po::launch_backward_sgd(dev_tree(t), t->desc.sh_degree, rays, n, dL_dC, aux, sg, o, t->d_sigma,
                                            static_cast<float*>(t->d_sh), t->sh_row, t->n_leaves, lr, grad_sigma,
                                            grad_sh, t->sgd_flag(),
                                            (cudaStream_t)stream),
                    "po_render_backward_sgd");
}

static cudaError_t grow(void** p, size_t* cap, size_t need) {
    if (*cap >= need) return cudaSuccess;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(p, need);
    if (e == cudaSuccess) *cap = need;
    return e;
}

po_status po_render_backward_deterministic(const po_tree* tc, const float* rays, int64_t n, const float* dL_dC,
                                           const double* aux, const po_segments* segments, const po_render_opts* opts,
                                           float* grad_sigma, float* grad_sh, int32_t* n_overflow, po_stream stream) {
    po_tree* t = const_cast<po_tree*>(tc);   // scratch only
    if (po_status s = check_tree(t)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (n < 0 || n >= (int64_t)INT32_MAX) return fail(PO_ERR_INVALID_ARG, "n outside [0, 2^31 - 1)");
    if (!segments || !aux) return fail(PO_ERR_INVALID_ARG, "the deterministic backward needs segments and aux");
    po::Segments sg;
    if (po_status s = check_segments(segments, n, aux, &sg)) return s;
    if (!rays || !dL_dC || !grad_sigma || !grad_sh) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    if (((uintptr_t)grad_sh & 15u) != 0) return fail(PO_ERR_INVALID_ARG, "grad_sh must be 16-byte aligned");
    if (n * (int64_t)std::max(segments->max_seg, 1) >= (int64_t)INT32_MAX)
        return fail(PO_ERR_UNSUPPORTED, "n * max_seg >= 2^31 (32-bit segment slots)");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    if (n_overflow && (e = cudaMemsetAsync(n_overflow, 0, sizeof(int32_t), s)) != cudaSuccess)
        return cuda_status(e, "memset(n_overflow)");
    if (n == 0) return PO_OK;
    std::lock_guard<std::mutex> lk(t->det_mu);
    const po::DevTree dt = dev_tree(t);
    // 1-2: per-ray emitted counts and their exclusive scan (one host sync reads the total S)
    size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int32_t*)nullptr, (int32_t*)nullptr, (int)(n + 1), s);
    scan_bytes = (scan_bytes + 255) / 256 * 256;   // keeps the records after it 16-B aligned
    const size_t a1 = ((size_t)(n + 1) * 4 + 255) / 256 * 256;
    if ((e = grow(&t->d_det, &t->det_cap, 2 * a1 + scan_bytes)) != cudaSuccess) return cuda_status(e, "scratch");
    int32_t* cnt = static_cast<int32_t*>(t->d_det);
    int32_t* offs = reinterpret_cast<int32_t*>(static_cast<char*>(t->d_det) + a1);
    if ((e = po::launch_det_counts(rays, n, dL_dC, sg, cnt, n_overflow, s)) != cudaSuccess) return cuda_status(e, "counts");
    if ((e = cub::DeviceScan::ExclusiveSum(static_cast<char*>(t->d_det) + 2 * a1, scan_bytes, cnt, offs, (int)(n + 1),
                                           s)) != cudaSuccess)
        return cuda_status(e, "scan");
    int32_t S32 = 0;
    if ((e = cudaMemcpyAsync(&S32, offs + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
        return cuda_status(e, "segment total");
    const int64_t S = S32;
    // 3-5: emit, sort by leaf, reduce per leaf in slot order
    int end_bit = 1;
    while (end_bit < 32 && ((uint64_t)1 << end_bit) <= (uint64_t)t->n_leaves) ++end_bit;
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)std::max<int64_t>(S, 1), 0,
                                    end_bit, s);
    const size_t a4 = ((size_t)std::max<int64_t>(S, 1) * 4 + 255) / 256 * 256;
    const size_t need = 2 * a1 + scan_bytes + 5 * a4 + 4 * a4 + sort_bytes;
    if (t->det_cap < need) {   // keep cnt / offs: grow into a fresh block and copy offs over
        // 25 % headroom: batches of one scene vary by a few % in segment count, and every
        // regrowth frees (a device-wide sync) and reallocates hundreds of MB inside the step
        size_t got = need + need / 4;
        void* nb = nullptr;
        if ((e = cudaMalloc(&nb, got)) != cudaSuccess) {
            (void)cudaGetLastError();
            got = need;
            if ((e = cudaMalloc(&nb, got)) != cudaSuccess) return cuda_status(e, "scratch");
        }
        e = cudaMemcpyAsync(static_cast<char*>(nb) + a1, offs, (size_t)(n + 1) * 4, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(t->d_det);
        t->d_det = nb;
        t->det_cap = got;
        if (e != cudaSuccess) return cuda_status(e, "scratch copy");
        offs = reinterpret_cast<int32_t*>(static_cast<char*>(t->d_det) + a1);
    }
    char* b = static_cast<char*>(t->d_det) + 2 * a1 + scan_bytes;
    uint32_t* key = reinterpret_cast<uint32_t*>(b);
    uint32_t* val = reinterpret_cast<uint32_t*>(b + a4);
    uint32_t* skey = reinterpret_cast<uint32_t*>(b + 2 * a4);
    uint32_t* sval = reinterpret_cast<uint32_t*>(b + 3 * a4);
    int32_t* ray_of = reinterpret_cast<int32_t*>(b + 4 * a4);
    float4* contrib = reinterpret_cast<float4*>(b + 5 * a4);
    void* sort_tmp = b + 9 * a4;
    if ((e = po::launch_det_emit(dt, t->desc.sh_degree, rays, n, dL_dC, aux, sg, offs, key, val, contrib, ray_of, s)) !=
        cudaSuccess)
        return cuda_status(e, "emit");
    if (S > 0 &&
        (e = cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, key, skey, val, sval, (int)S, 0, end_bit, s)) !=
            cudaSuccess)
        return cuda_status(e, "sort");
    if ((e = po::launch_det_reduce(dt, t->desc.sh_degree, rays, skey, sval, S, contrib, ray_of, grad_sigma, grad_sh,
                                   s)) != cudaSuccess)
        return cuda_status(e, "reduce");
    g_launches.fetch_add(3);   // counts, emit, reduce (+ CUB's scan / sort kernels, library code)
    // rays whose segments overflowed max_seg: the re-traversal (atomic, not order-fixed)
    return launched(po::launch_backward(dt, t->desc.sh_degree, t->desc.payload == PO_F16, rays, n, dL_dC, aux, sg, o,
                                        grad_sigma, grad_sh, s, true),
                    "po_render_backward_deterministic");
}

po_status po_l2_loss_grad(const float* pred, const float* target, int64_t n, float* dL_dC, double* loss,
                          int32_t device, po_stream stream) {
    if (n < 0) return fail(PO_ERR_INVALID_ARG, "n < 0");
    if (n > 0 && (!pred || !target || !dL_dC)) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    return launched(po::launch_l2_loss(pred, target, n * 3, dL_dC, loss, (cudaStream_t)stream), "po_l2_loss_grad");
}

po_status po_tree_sgd_step_range(po_tree* t, float* grad_sigma, float* grad_sh, float lr, int64_t begin, int64_t end,
                                 int32_t flags, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    if (t->desc.payload != PO_F32) return fail(PO_ERR_UNSUPPORTED, "SGD needs an fp32 payload (P:973 trains in fp32)");
    if (!std::isfinite(lr)) return fail(PO_ERR_INVALID_ARG, "lr not finite");
    const int64_t total = t->n_leaves * (int64_t)(t->ne + 1);
    if (begin < 0 || end > total || begin > end)
        return fail(PO_ERR_INVALID_ARG, "range [%lld, %lld) outside [0, %lld)", (long long)begin, (long long)end,
                    (long long)total);
    if (end == begin) return PO_OK;
    if (!grad_sigma || !grad_sh) return fail(PO_ERR_INVALID_ARG, "NULL gradient");
    if (flags & ~PO_SGD_ZERO_GRAD) return fail(PO_ERR_INVALID_ARG, "unknown flags %d", flags);
    if (((uintptr_t)grad_sh & 15u) != 0) return fail(PO_ERR_INVALID_ARG, "grad_sh must be 16-byte aligned");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    return launched(po::launch_sgd(t->d_sigma, static_cast<float*>(t->d_sh), t->sh_row, t->ne, t->n_leaves, grad_sigma,
                                   grad_sh, lr, begin, end, (flags & PO_SGD_ZERO_GRAD) != 0, (cudaStream_t)stream),
                    "po_tree_sgd_step");
}

po_status po_tree_sgd_step(po_tree* t, const float* grad_sigma, const float* grad_sh, float lr, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    // flags = 0: the gradients are only read
    return po_tree_sgd_step_range(t, const_cast<float*>(grad_sigma), const_cast<float*>(grad_sh), lr, 0,
                                  t->n_leaves * (int64_t)(t->ne + 1), 0, stream);
}

po_status po_trace(const po_tree* t, const float* rays, int64_t n, const po_render_opts* opts, int32_t max_leaves,
                   int32_t* leaf_ids, int32_t* counts, int32_t* node_counts, int32_t flags, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (n < 0 || max_leaves < 0) return fail(PO_ERR_INVALID_ARG, "n < 0 or max_leaves < 0");
    if (n == 0) return PO_OK;
    if (!rays || (max_leaves > 0 && !leaf_ids)) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    if (flags & ~PO_TRACE_CLASSIC) return fail(PO_ERR_INVALID_ARG, "unknown flags %d", flags);
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    return launched(po::launch_trace(dev_tree(t), rays, n, o.gamma, max_leaves, max_leaves > 0 ? leaf_ids : nullptr,
                                     counts, node_counts, (flags & PO_TRACE_CLASSIC) != 0, (cudaStream_t)stream),
                    "po_trace");
}

po_status po_render_depth(const po_tree* t, const float* rays, int64_t n, const po_render_opts* opts, float* alpha,
                          float* depth, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (n < 0) return fail(PO_ERR_INVALID_ARG, "n < 0");
    if (n == 0) return PO_OK;
    if (!rays || !alpha || !depth) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    return launched(po::launch_render_depth(dev_tree(t), rays, n, o.gamma, alpha, depth, (cudaStream_t)stream),
                    "po_render_depth");
}

po_status po_leaf_max_alpha(const po_tree* t, const float* rays, int64_t n, const po_render_opts* opts,
                            float* max_alpha, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (n < 0) return fail(PO_ERR_INVALID_ARG, "n < 0");
    if (n == 0) return PO_OK;
    if (!rays || !max_alpha) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    return launched(po::launch_leaf_max_alpha(dev_tree(t), rays, n, o.gamma, max_alpha, (cudaStream_t)stream),
                    "po_leaf_max_alpha");
}

po_status po_render_timeline(const po_tree* t, const po_camera* cams, int32_t n_cams, int32_t W, int32_t H,
                             const po_render_opts* opts, float* out_rgb, unsigned long long* timeline,
                             po_stream stream) {
#ifndef PO_DIAG
    return fail(PO_ERR_UNSUPPORTED, "%s: diagnostics are built only with -DPO_DIAG", "po_render_timeline");
#else
    if (po_status s = check_tree(t)) return s;
    if (po_status s = check_image(n_cams, W, H)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (n_cams == 0) return PO_OK;
    if (!cams || !out_rgb || !timeline) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    return render_scheduled(const_cast<po_tree*>(t), cams, n_cams, W, H, o, out_rgb, (cudaStream_t)stream,
                            "po_render_timeline", timeline);
#endif
}

po_status po_set_block_order(po_tree* t, int32_t W, int32_t H, const uint32_t* order) {
#ifndef PO_DIAG
    (void)t, (void)W, (void)H, (void)order;
    return fail(PO_ERR_UNSUPPORTED, "%s: diagnostics are built only with -DPO_DIAG", "po_set_block_order");
#else
    if (po_status s = check_tree(t)) return s;
    if (po_status s = check_image(1, W, H)) return s;
    if (!order) return fail(PO_ERR_INVALID_ARG, "NULL order");
    const size_t nb = (size_t)((W + 15) / 16) * ((H + 15) / 16);
    std::vector<char> seen(nb, 0);
    for (size_t i = 0; i < nb; ++i) {
        if (order[i] >= nb || seen[order[i]]) return fail(PO_ERR_INVALID_ARG, "order is not a permutation");
        seen[order[i]] = 1;
    }
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    cudaError_t e = cudaSuccess;
    block_order(t, W, H, nullptr, &e);   // allocates the table for this size
    if (e != cudaSuccess) return cuda_status(e, "block order");
    std::lock_guard<std::mutex> lk(t->order_mu);
    if (!t->d_order) return fail(PO_ERR_UNSUPPORTED, "raster order (PO_RENDER_ORDER=raster)");
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cuda_status(e, "sync");
    if ((e = cudaMemcpy(t->d_order, order, nb * sizeof(unsigned), cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_status(e, "order copy");
    return PO_OK;
#endif
}

po_status po_ray_step_timing(const po_tree* t, const float* rays, int64_t n, const po_render_opts* opts,
                             int32_t max_steps, uint32_t* rec, int32_t* steps, po_stream stream) {
#ifndef PO_DIAG
    return fail(PO_ERR_UNSUPPORTED, "%s: diagnostics are built only with -DPO_DIAG", "po_ray_step_timing");
#else
    if (po_status s = check_tree(t)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (t->desc.sh_degree != 3 || t->desc.payload != PO_F32)
        return fail(PO_ERR_UNSUPPORTED, "po_ray_step_timing: SH-3 fp32 trees only");
    if (n < 0 || max_steps < 0) return fail(PO_ERR_INVALID_ARG, "n or max_steps < 0");
    if (n == 0) return PO_OK;
    if (!rays || !rec || !steps) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    return launched(po::launch_ray_step_timing(dev_tree(t), rays, n, o, max_steps, rec, steps, (cudaStream_t)stream),
                    "po_ray_step_timing");
#endif
}

po_status po_render_stats(const po_tree* t, const po_camera* cams, int32_t n_cams, int32_t W, int32_t H,
                          const po_render_opts* opts, unsigned long long* counters, po_stream stream) {
    if (po_status s = check_tree(t)) return s;
    if (po_status s = check_image(n_cams, W, H)) return s;
    po::RenderOpts o;
    if (po_status s = check_opts(opts, &o)) return s;
    if (n_cams == 0) return PO_OK;
    if (!cams || !counters) return fail(PO_ERR_INVALID_ARG, "NULL buffer");
    DeviceGuard g(t->desc.device);
    if (g.err != cudaSuccess) return cuda_status(g.err, "cudaSetDevice");
    return launched(po::launch_stats(dev_tree(t), cams, n_cams, W, H, o.gamma, counters, (cudaStream_t)stream),
                    "po_render_stats");
}

}  // extern "C"
