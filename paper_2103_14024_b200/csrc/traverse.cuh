// Device-side building blocks of the PlenOctree hot path (sm_100a).
//
//   ray setup + AABB clip ......... SURVEY §8(a) a1/a2, reading Q5/Q6
//   ordered octree descent ........ a3, PAPER P:424-433 ("skipping large voxels in one step
//                                   while also not missing small voxels")
//   SH basis, colour .............. a5, P:296-300 (Eq. 5), P:749-767 (App. B.1)
//   alpha / transmittance ......... a4/a6, P:238-243 (Eq. 1-2), P:435-437 (early stop)
//
// Traversal design (B200-first, not the paper's): the ray lives in integer leaf-grid
// coordinates (the cube is [0, 2^D)^3, leaf cells are unit cubes).  Every plane crossing
// is computed from scratch as t = (plane - o') * inv with an exactly representable
// integer plane, and consecutive segments share their boundary t.  The current cell
// is a triple of integers; after leaving a box through face `ax`, the neighbour cell is
// known exactly on that axis and by point location on the other two (clamped to the
// box).  The descent restarts at the deepest common ancestor, found with one clz of
// (old XOR new) cell coordinates, from a per-thread ancestor stack.  Empty coarse boxes
// are skipped in one step.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

namespace po {

constexpr uint32_t kTagEmpty = 0u, kTagInternal = 1u, kTagLeaf = 2u;
constexpr uint32_t kIdxMask = (1u << 30) - 1u;
constexpr int kMaxDepth = 15;
// The device child table keeps the ABI encoding (reading Q1): tag << 30 | index.

struct DevTree {
    const uint32_t* __restrict__ child;   // [n_nodes][8], tag << 30 | index (reading Q1)
    const float* __restrict__ sigma;      // [n_leaves]   sigma~
    const void* __restrict__ sh;          // [n_leaves][row] fp32 or fp16, rows 16-B aligned
    int32_t sh_row;                       // row stride in elements
    int32_t depth;
    float bmin[3];
    float scale;                          // 2^D / edge
    float odd_sign;                       // +1 (Condon-Shortley reading) or -1
    // NEXT f3, spherical Gaussians: B lobes (unit axis xyz, bandwidth) replacing
    // the SH basis when non-null (po_tree_set_sg_basis)
    const float4* __restrict__ sg;
    // kOptGrid cell index: one (E, F) pair per level-(D-1) cell, 2^(D-1) per axis, x-major;
    // null when not built.  E = tag << 30 | payload:
    //   tag 0: empty box, payload = its level (bits 0-7) | Chebyshev distance of the cell to
    //          the nearest occupied level-(D-1) cell, capped at 255 (bits 8-15)
    //                                                  tag 2: a depth-(D-1) leaf (its entry)
    //   tag 1: a depth-(D-1) node (child-table entry)  tag 3: a depth-(D-1) node whose leaves
    //   are consecutive in octant order: payload = 8-bit occupancy mask, F = its first leaf, so
    //   a leaf-level cell's entry is F + popc(mask below its octant) -- no child-table load
    //   0xFFFFFFFF: a leaf coarser than D-1 covers the cell (classic descent)
    const uint2* __restrict__ grid = nullptr;
    // rays are clipped to this box (leaf units, integral): the occupied cells' bounding box in
    // level-(D-1) cells when the index is built, else [0, 2^D]^3.  Leaves lie inside it, so
    // every leaf segment keeps its t values (its faces are the same planes)
    float clip_lo[3] = {0.f, 0.f, 0.f}, clip_hi[3] = {0.f, 0.f, 0.f};
};

struct RayState {
    float o[3];     // origin in grid units
    float dg[3];    // unit direction * scale (grid units per world unit)
    float inv[3];   // 1 / dg (world t per grid unit), +inf for a zero component
    float d[3];     // unit world direction (SH argument, reading Q15)
    float tnear, tfar;
};

// a1/a2: normalise d, move to grid units, slab-clip against [0, 2^D]^3.
// Unit direction exactly as ray_setup computes it (the stored-segment pass 2 needs the same
// SH basis as pass 1).  Scales by the largest component first so tiny / huge directions
// normalise without under- or overflow; false for a zero / denormal / inf / NaN direction.
__device__ __forceinline__ bool unit_direction(const float dir[3], float d[3]) {
    const float m = fmaxf(fabsf(dir[0]), fmaxf(fabsf(dir[1]), fabsf(dir[2])));
    if (!(m >= 1.17549435e-38f) || !(m < INFINITY)) return false;
    const float im = 1.0f / m;
    const float s0 = dir[0] * im, s1 = dir[1] * im, s2 = dir[2] * im;
    const float rn = im / sqrtf(s0 * s0 + s1 * s1 + s2 * s2);
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = dir[k] * rn;
    return true;
}

// clip = false: the whole cube [0, 2^D]^3 (the classic reference descent of k_trace / k_stats,
// whose node counts define SURVEY 8(d)'s algorithmic bytes); true: the occupied box clip_lo/hi.
__device__ __forceinline__ bool ray_setup(const DevTree& tr, const float o[3], const float dir[3], RayState& r,
                                          bool clip = true) {
    // a zero or non-finite direction renders the background
    if (!unit_direction(dir, r.d)) return false;
    const float G = (float)(1 << tr.depth);
    float tn = 0.f, tf = INFINITY;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        r.o[k] = (o[k] - tr.bmin[k]) * tr.scale;
        r.dg[k] = r.d[k] * tr.scale;
        const float lo = clip ? tr.clip_lo[k] : 0.f, hi = clip ? tr.clip_hi[k] : G;
        if (r.dg[k] != 0.f) {
            r.inv[k] = 1.0f / r.dg[k];
            float ta = (lo - r.o[k]) * r.inv[k];   // plane_t's expression
            float tb = (hi - r.o[k]) * r.inv[k];
            tn = fmaxf(tn, fminf(ta, tb));
            tf = fminf(tf, fmaxf(ta, tb));
        } else {
            r.inv[k] = INFINITY;
            if (!(r.o[k] >= lo && r.o[k] <= hi)) return false;
        }
    }
    r.tnear = tn;
    r.tfar = tf;
    return tf > tn;
}

// world t at which the ray crosses the integer plane `face` of axis k (the same expression in
// every kernel, so all of them walk identical boxes with identical t)
__device__ __forceinline__ float plane_t(const RayState& r, int k, int face) {
    return ((float)face - r.o[k]) * r.inv[k];
}

// Cell index on one axis of the point o' + t*dg, for a ray moving with slope dg:
// the cell the ray is about to traverse (ceil-1 when moving down).
__device__ __forceinline__ int cell_of(float o, float dg, float t) {
    float p = fmaf(t, dg, o);
    return dg < 0.f ? (int)ceilf(p) - 1 : (int)floorf(p);
}

// Per-thread ancestor stack in shared memory: slot L of thread t at base[L * kStackStride + t]
// (consecutive lanes hit consecutive banks; no local-memory traffic).
constexpr int kStackStride = 256;   // = threads per CTA of every kernel that traverses
struct SmemStack {
    uint32_t* base;
    __device__ __forceinline__ uint32_t& operator[](int L) const { return base[L * kStackStride]; }
};
#define PO_DECLARE_STACK(name)                                                        \
    __shared__ uint32_t name##_storage[(po::kMaxDepth + 1) * po::kStackStride];       \
    po::SmemStack name{name##_storage + threadIdx.x}

// a3: ordered descent.  Calls vis.on_node() for every internal node entered (root
// included) and vis.on_leaf(idx, t_in, t_out) for every positive-length leaf segment in
// ray order; traversal stops when on_leaf returns false (early stop) or the ray exits.
// Neighbour-step variants (compile time; DESIGN.md §6.1 logs the others that were measured
// slower and removed: leaf-step fast path, shared-memory / pipelined rows, macro-grid skip,
// child occupancy masks, 4x4x4 bricks, shared-memory upper levels):
//   kOptPlain = 0      the exit axis steps exactly, the other two are point-located with the
//                      "moving down onto an integral plane" correction and clamped into the box
//   kOptLean           every axis whose face is crossed at t_exit steps (an exact edge or corner
//                      crossing moves diagonally), the others take one F2I.FLOOR and the clamp
//   kOptProbeNoShade   (render only) measurement probe: traversal + T, no SH rows
constexpr int kOptPlain = 0;
constexpr int kOptProbeNoShade = 64;
constexpr int kOptLean = 128;
//   kOptGrid           (render experiment) boxes found through a dense level-(D-1) index:
//                      one index load (+ one child-entry load) per step, no stack
constexpr int kOptGrid = 8192;
// Default traversal of every kernel (render, render_rays, backward, trace, stats), so all
// entry points visit the same leaf segments with the same t values (po_render ==
// po_render_rays bitwise).  Lean measured +2-3% on c1 over the plain step.
constexpr int kOptDefault = kOptLean;
// The frame renderer additionally finds boxes through the level-(D-1) index when the tree has
// one (kOptGrid: same boxes, same t values, bit-identical images; DESIGN.md §6.1 v11).
constexpr int kRenderOptDefault = kOptDefault | kOptGrid;

// Optional visitor hook on_box(shift), called once per box the ray steps through (leaf or
// empty; shift = log2 of the box edge in leaf cells).  Only the statistics visitor has it.
template <class V, class = void>
struct HasOnBox : std::false_type {};
template <class V>
struct HasOnBox<V, std::void_t<decltype(std::declval<V&>().on_box(0))>> : std::true_type {};

template <int OPT = kOptDefault, class V>
__device__ __forceinline__ void traverse(const DevTree& tr, const RayState& r, V& vis, const SmemStack& stk) {
    const int D = tr.depth;
    const int G = 1 << D;
    float t = r.tnear;
    int c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = min(max(cell_of(r.o[k], r.dg[k], t), 0), G - 1);
    stk[0] = kTagInternal << 30;   // the root, node 0
    int L = 0;
    vis.on_node();
    if constexpr ((OPT & kOptGrid) != 0) {
        if (tr.grid != nullptr && D >= 1) {
            const int G2 = G >> 1;
            // the next box's index entry is loaded as soon as its cell is known, before this
            // box's leaf is shaded, so the entry's latency overlaps the SH-row loads and FMAs
            // (DESIGN.md §6.1 v16)
            uint2 EF = __ldg(tr.grid + (((size_t)(c[0] >> 1) * G2 + (c[1] >> 1)) * G2 + (c[2] >> 1)));
            while (true) {
                const uint32_t E = EF.x;
                uint32_t e;
                int shift;
                if (E == 0xFFFFFFFFu) {
                    break;   // a coarse leaf: not indexed (never in the benchmark trees); classic path below
                } else if ((E >> 30) == 3u) {   // packed depth-(D-1) node: the leaf entry without a load
                    const uint32_t oct = (uint32_t)(((c[0] & 1) << 2) | ((c[1] & 1) << 1) | (c[2] & 1));
                    e = ((E >> oct) & 1u) ? ((kTagLeaf << 30) | (EF.y + __popc(E & ((1u << oct) - 1u) & 0xFFu))) : 0u;
                    shift = 0;
                } else if ((E >> 30) == kTagInternal) {
                    e = __ldg(tr.child + ((E & kIdxMask) * 8u + (uint32_t)(((c[0] & 1) << 2) | ((c[1] & 1) << 1) | (c[2] & 1))));
                    shift = 0;
                } else if ((E >> 30) == kTagLeaf) {
                    e = E;
                    shift = 1;
                } else {
                    e = 0u;
                    shift = D - (int)(E & 0xFFu);   // the empty box's level (bits 8-15: Chebyshev distance)
                }
                const int size = 1 << shift;
                int lo[3], hi[3];
                float te[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    lo[k] = c[k] & ~(size - 1);
                    hi[k] = lo[k] + size;
                    te[k] = plane_t(r, k, (r.dg[k] >= 0.f) ? hi[k] : lo[k]);
                }
                float texit = fminf(fminf(te[0], te[1]), te[2]);
                // an empty cell at Chebyshev distance dc from the nearest occupied level-(D-1)
                // cell lies in an empty cube of (2 dc - 1)^3 such cells: leave that instead of
                // the octree box when it reaches further (leaves are still entered through their
                // own faces, so their segments keep the same t values)
                const int dc = (E >> 30) == 0u ? (int)((E >> 8) & 0xFFu) : 0;
                if (dc > 1) {
                    int lo2[3], hi2[3];
                    float te2[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const int cc = c[k] >> 1;
                        lo2[k] = max(2 * (cc - dc + 1), 0);
                        hi2[k] = min(2 * (cc + dc), G);
                        te2[k] = plane_t(r, k, (r.dg[k] >= 0.f) ? hi2[k] : lo2[k]);
                    }
                    const float tx2 = fminf(fminf(te2[0], te2[1]), te2[2]);
                    if (tx2 > texit) {
#pragma unroll
                        for (int k = 0; k < 3; ++k) {
                            lo[k] = lo2[k];
                            hi[k] = hi2[k];
                            te[k] = te2[k];
                        }
                        texit = tx2;
                    }
                }
                const float tout = fminf(texit, r.tfar);
                int nc[3];
                bool out = false;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const bool hit = te[k] == texit;
                    const int nex = (r.dg[k] > 0.f) ? hi[k] : lo[k] - 1;
                    const int ck = __float2int_rd(fmaf(texit, r.dg[k], r.o[k]));
                    nc[k] = hit ? nex : min(max(ck, lo[k]), hi[k] - 1);
                    out |= hit & ((unsigned)nex >= (unsigned)G);
                }
                const bool cont = (texit < r.tfar) && !out;
                uint2 EFn = make_uint2(0u, 0u);
                if (cont) EFn = __ldg(tr.grid + (((size_t)(nc[0] >> 1) * G2 + (nc[1] >> 1)) * G2 + (nc[2] >> 1)));
                if ((e >> 30) == kTagLeaf && tout > t) {
                    if (!vis.on_leaf(e & kIdxMask, t, tout)) return;
                }
                if (!cont) return;
                t = texit;
                c[0] = nc[0];
                c[1] = nc[1];
                c[2] = nc[2];
                EF = EFn;
            }
            L = 0;   // fall back from the current cell with a fresh descent
        }
    }
    while (true) {
        // stk[L] holds the entry word of the node at level L (the deepest common ancestor of
        // the previous and the current cell); descend to the box that contains cell c
        uint32_t ent = stk[L];
        uint32_t e;
        int shift;
        while (true) {
            shift = D - 1 - L;
            const int oct = (((c[0] >> shift) & 1) << 2) | (((c[1] >> shift) & 1) << 1) | ((c[2] >> shift) & 1);
            e = __ldg(tr.child + ((ent & kIdxMask) * 8u + (uint32_t)oct));
            if ((e >> 30) != kTagInternal) break;
            ent = e;
            ++L;
            stk[L] = ent;
            vis.on_node();
        }
        // the box of entry e: level L+1, 2^shift leaf cells per axis.  Exit t per axis,
        // branch-free: an axis with dg == 0 uses its upper face and inv = +inf, giving +inf
        // (or NaN when the origin sits exactly on that face), which fminf ignores.
        if constexpr (HasOnBox<V>::value) vis.on_box(shift);
        const int size = 1 << shift;
        int lo[3];
        float te[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            lo[k] = c[k] & ~(size - 1);
            const int face = (r.dg[k] >= 0.f) ? lo[k] + size : lo[k];
            te[k] = plane_t(r, k, face);
        }
        const float texit = fminf(fminf(te[0], te[1]), te[2]);
        const int ax = (te[0] == texit) ? 0 : ((te[1] == texit) ? 1 : 2);   // first minimal axis
        const float tout = fminf(texit, r.tfar);
        if ((e >> 30) == kTagLeaf && tout > t) {
            if (!vis.on_leaf(e & kIdxMask, t, tout)) return;
        }
        if (!(texit < r.tfar)) return;
        t = texit;
        int nc[3];
        bool out = false;
        if constexpr ((OPT & kOptLean) != 0) {
            // every axis whose face is crossed at texit steps (an exact edge or corner crossing
            // moves diagonally), the others are point-located with one F2I.FLOOR (an exactly
            // integral coordinate while moving down yields a zero-length box that the
            // `tout > t` test skips) and clamped into the box
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const bool hit = te[k] == texit;
                const int nex = (r.dg[k] > 0.f) ? lo[k] + size : lo[k] - 1;
                const int ck = __float2int_rd(fmaf(t, r.dg[k], r.o[k]));
                nc[k] = hit ? nex : min(max(ck, lo[k]), lo[k] + size - 1);
                out |= hit & ((unsigned)nex >= (unsigned)G);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                // cell the ray enters on axis k: floor(p), or p-1 when moving down and p is integral
                const float p = fmaf(t, r.dg[k], r.o[k]);
                const float f = floorf(p);
                const int ck = (int)f - (int)((r.dg[k] < 0.f) & (f == p));
                const int nex = (r.dg[k] > 0.f) ? lo[k] + size : lo[k] - 1;   // exact on the exit axis
                nc[k] = (k == ax) ? nex : min(max(ck, lo[k]), lo[k] + size - 1);
                out |= (k == ax) & ((unsigned)nex >= (unsigned)G);
            }
        }
        if (out) return;
        const int diff = (c[0] ^ nc[0]) | (c[1] ^ nc[1]) | (c[2] ^ nc[2]);
        L = D - 1 - (31 - __clz(diff));   // restart at the deepest common ancestor
        c[0] = nc[0];
        c[1] = nc[1];
        c[2] = nc[2];
    }
}

// ---------------------------------------------------------------------------------
// a5: real SH basis, l <= 3, Cartesian form of App. B.1 under the
// Condon-Shortley reading (Q16); odd-|m| functions are multiplied by odd_sign.
// ---------------------------------------------------------------------------------
template <int DEG>
struct ShDim {
    static constexpr int B = (DEG + 1) * (DEG + 1);
};

template <int DEG>
__device__ __forceinline__ void sh_basis(const float d[3], float odd, float* Y) {
    const float x = d[0], y = d[1], z = d[2];
    Y[0] = 0.28209479177387814f;
    if (DEG >= 1) {
        Y[1] = odd * 0.48860251190291992f * y;
        Y[2] = 0.48860251190291992f * z;
        Y[3] = odd * 0.48860251190291992f * x;
    }
    if (DEG >= 2) {
        const float xx = x * x, yy = y * y, zz = z * z;
        Y[4] = 1.0925484305920792f * x * y;
        Y[5] = odd * 1.0925484305920792f * y * z;
        Y[6] = 0.94617469575756008f * zz - 0.31539156525252005f;
        Y[7] = odd * 1.0925484305920792f * x * z;
        Y[8] = 0.54627421529603959f * (xx - yy);
        if (DEG >= 3) {
            Y[9] = odd * 0.59004358992664352f * y * (3.f * xx - yy);
            Y[10] = 2.8906114426405538f * x * y * z;
            Y[11] = odd * 0.45704579946446572f * y * (5.f * zz - 1.f);
            Y[12] = 0.37317633259011540f * z * (5.f * zz - 3.f);
            Y[13] = odd * 0.45704579946446572f * x * (5.f * zz - 1.f);
            Y[14] = 1.4453057213202769f * z * (xx - yy);
            Y[15] = odd * 0.59004358992664352f * x * (xx - 3.f * yy);
            if (DEG >= 4) {   // l = 4 (SH-25, the paper's T&T setting P:587-588), same sign convention
                const float x2y2 = xx - yy, z7m1 = 7.f * zz - 1.f, z7m3 = 7.f * zz - 3.f;
                Y[16] = 2.5033429417967046f * x * y * x2y2;
                Y[17] = odd * 1.7701307697799304f * y * z * (3.f * xx - yy);
                Y[18] = 0.94617469575756008f * x * y * z7m1;
                Y[19] = odd * 0.66904654355728917f * y * z * z7m3;
                Y[20] = 0.10578554691520430f * (zz * (35.f * zz - 30.f) + 3.f);
                Y[21] = odd * 0.66904654355728917f * x * z * z7m3;
                Y[22] = 0.47308734787878004f * x2y2 * z7m1;
                Y[23] = odd * 1.7701307697799304f * x * z * (xx - 3.f * yy);
                Y[24] = 0.62583573544917614f * (xx * (xx - 3.f * yy) - yy * (3.f * xx - yy));
            }
        }
    }
}

// The per-ray basis of the tree: SH (App. B.1) or, when the tree carries lobes, spherical
// Gaussians G_b(d) = exp(lambda_b (d . p_b - 1)), B = (DEG + 1)^2 of them.
template <int DEG>
__device__ __forceinline__ void ray_basis(const DevTree& tr, const float d[3], float* Y) {
    if (tr.sg != nullptr) {
        constexpr int B = ShDim<DEG>::B;
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const float4 p = __ldg(tr.sg + b);
            Y[b] = expf(p.w * (fmaf(d[0], p.x, fmaf(d[1], p.y, d[2] * p.z)) - 1.f));
        }
    } else {
        sh_basis<DEG>(d, tr.odd_sign, Y);
    }
}

// z_ch = sum_b k[b][ch] Y_b over one leaf row (basis-major, channel-minor), fixed order.
template <int DEG, bool F16>
__device__ __forceinline__ void sh_dot(const DevTree& tr, uint32_t idx, const float* Y, float z[3]) {
    constexpr int B = ShDim<DEG>::B;
    constexpr int NE = 3 * B;
    z[0] = z[1] = z[2] = 0.f;
    if (!F16) {
        const float4* row = reinterpret_cast<const float4*>(static_cast<const float*>(tr.sh) + (size_t)idx * tr.sh_row);
        constexpr int NV = (NE + 3) / 4;
        float4 v[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) v[j] = __ldg(row + j);
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const float vv[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int el = 4 * j + q;
                if (el < NE) z[el % 3] = fmaf(vv[q], Y[el / 3], z[el % 3]);
            }
        }
    } else {
        const uint4* row = reinterpret_cast<const uint4*>(static_cast<const __half*>(tr.sh) + (size_t)idx * tr.sh_row);
        constexpr int NV = (NE + 7) / 8;
        uint4 v[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) v[j] = __ldg(row + j);
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const uint32_t w4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                __half2 h2 = *reinterpret_cast<const __half2*>(&w4[q]);
                float2 f = __half22float2(h2);
                const int el0 = 8 * j + 2 * q, el1 = el0 + 1;
                if (el0 < NE) z[el0 % 3] = fmaf(f.x, Y[el0 / 3], z[el0 % 3]);
                if (el1 < NE) z[el1 % 3] = fmaf(f.y, Y[el1 / 3], z[el1 % 3]);
            }
        }
    }
}

// e^x as one MUFU.EX2 (flush-to-zero: results below 2^-126 become 0, harmless for T and colours)
__device__ __forceinline__ float exp_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__fmul_rn(x, 1.44269504088896341f)));
    return y;
}

__device__ __forceinline__ float sigmoidf_(float z) { return __fdividef(1.0f, 1.0f + exp_ftz(-z)); }

// a4: e = exp(-sigma delta), weight w = T (1 - e), T' = T e.  Explicit _rn intrinsics so
// every kernel that evaluates a leaf produces bit-identical w, T' (forward, trace,
// backward passes 1 and 2 must agree on termination and on the prefix sums).
struct Absorb {
    float e, w, Tn;
};
__device__ __forceinline__ Absorb absorb(float T, float sigma, float delta) {
    Absorb a;
    a.e = exp_ftz(-__fmul_rn(sigma, delta));
    a.w = __fmul_rn(T, __fsub_rn(1.0f, a.e));
    a.Tn = __fmul_rn(T, a.e);
    return a;
}

}  // namespace po
