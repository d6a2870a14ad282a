// =====================================================================================
//  PlenOctree CPU ORACLE  --  TEST INFRASTRUCTURE ONLY
// =====================================================================================
//  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
//  leg may load or call this library.  The product path (paper_2103_14024_b200/) never
//  does; it shares no code, header, table or constant with this file.
//
//  What it computes: the plain definition of PlenOctree volume rendering, in double
//  precision, in the paper's order and notation (PAPER.md = P:<line>):
//    * ray-voxel segments of the octree, in ray order            P:424-433 (§4.2 Rendering)
//    * real SH basis built from the complex SH definition         P:749-767 (App. B.1)
//    * colour c = S(sum_l sum_m k_l^m Y_l^m(d)), S = sigmoid      P:296-300 (Eq. 5)
//    * sigma = (sigma~)_+                                         P:959-963 (App. B.3)
//    * C = sum_i T_i (1 - exp(-sigma_i delta_i)) c_i + T_N c_N    P:238-243 (Eq. 1-2)
//    * early stop once T < gamma
//    * analytic derivatives dC/dc_i = w_i, dC/dsigma_i =
//      delta_i [c_i T_{i+1} - sum_{k>i} c_k w_k]
//      evaluated with DIRECT suffix sums (not the paper's two-pass "total minus prefix"
//      trick): this is the plain definition.
//  Readings where the paper is silent are DESIGN.md "Readings" Q1-Q32.
//
//  Parity pins (tests/test_oracle_*.py, run with -m "not gpu"): SH vs closed forms,
//  addition theorem, orthonormality and scipy; traversal brute force vs recursive
//  descent vs dense-grid DDA; Beer-Lambert / ln2 / weight-sum closed forms; central
//  finite differences of the oracle's own forward for the gradients.
// =====================================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

typedef struct {
    const uint32_t* child;   // [n_nodes][8], tag<<30 | index (reading Q1)
    int64_t n_nodes;
    const double* sigma;     // [n_leaves] sigma-tilde (the caller widens fp32/fp16 exactly)
    const double* sh;        // [n_leaves][B][3], or NULL when sh32 is given
    const float* sh32;       // [n_leaves][B][3] fp32 values (widened exactly when read), used if sh == NULL
    int64_t n_leaves;
    int32_t depth;           // D
    int32_t sh_degree;       // l_max
    int32_t sh_cs;           // 1: Condon-Shortley phase inside P_l^m (reading Q16 default)
    int32_t pad_;
    double bbox_min[3];
    double edge;
    // NEXT f3, spherical Gaussians: when sg_axes != NULL the B = (sh_degree+1)^2
    // per-channel basis functions are G_b(d) = exp(lambda_b (d . p_b - 1)) instead of SH
    const double* sg_axes;     // [B][3] lobe axes p_b (normalised here, reading Q36)
    const double* sg_lambda;   // [B] bandwidths lambda_b
} or_tree;

}  // extern "C"

namespace {

const double kPi = 3.14159265358979323846;

struct Seg {
    double t0, t1;
    int64_t leaf;
};

struct NodeHit {
    double t0;
};

// ------------------------------------------------------------------------------------
// App. B.1: complex SH  Y_l^m = sqrt((2l+1)/(4 pi) (l-m)!/(l+m)!) P_l^m(cos th) e^{i m ph},
// real SH = sqrt2 (-1)^m Im[Y_l^|m|] (m<0), Y_l^0 (m=0), sqrt2 (-1)^m Re[Y_l^m] (m>0).
// P_l^m by the textbook three-term recurrence in l.
// ------------------------------------------------------------------------------------
double factorial(int n) {
    double f = 1.0;
    for (int i = 2; i <= n; ++i) f *= i;
    return f;
}

double assoc_legendre(int l, int m, double x, int cs) {
    // P_m^m = (-1)^m (2m-1)!! (1-x^2)^{m/2}   (the (-1)^m is the Condon-Shortley phase)
    double somx2 = std::sqrt(std::max(0.0, 1.0 - x * x));
    double pmm = 1.0;
    for (int i = 1; i <= m; ++i) pmm *= (2.0 * i - 1.0) * somx2;
    if (cs && (m & 1)) pmm = -pmm;
    if (l == m) return pmm;
    double pmmp1 = x * (2.0 * m + 1.0) * pmm;   // P_{m+1}^m
    if (l == m + 1) return pmmp1;
    double pll = 0.0;
    for (int ll = m + 2; ll <= l; ++ll) {        // (l-m) P_l^m = (2l-1) x P_{l-1}^m - (l+m-1) P_{l-2}^m
        pll = ((2.0 * ll - 1.0) * x * pmmp1 - (ll + m - 1.0) * pmm) / (ll - m);
        pmm = pmmp1;
        pmmp1 = pll;
    }
    return pll;
}

void sh_basis(int lmax, int cs, const double* dir, double* Y) {
    double n = std::sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
    double x = dir[0] / n, y = dir[1] / n, z = dir[2] / n;
    double cos_th = std::max(-1.0, std::min(1.0, z));
    double phi = std::atan2(y, x);
    int b = 0;
    for (int l = 0; l <= lmax; ++l) {
        for (int m = -l; m <= l; ++m, ++b) {
            int am = m < 0 ? -m : m;
            double N = std::sqrt((2.0 * l + 1.0) / (4.0 * kPi) * factorial(l - am) / factorial(l + am));
            double P = assoc_legendre(l, am, cos_th, cs);
            double sgn = (am & 1) ? -1.0 : 1.0;   // (-1)^m
            if (m == 0)
                Y[b] = N * P;
            else if (m > 0)
                Y[b] = std::sqrt(2.0) * sgn * N * P * std::cos(am * phi);   // Re e^{i m phi}
            else
                Y[b] = std::sqrt(2.0) * sgn * N * P * std::sin(am * phi);   // Im e^{i |m| phi}
        }
    }
}

// ------------------------------------------------------------------------------------
// Geometry.  Box of cell c at level L: [bmin + edge*c/2^L, bmin + edge*(c+1)/2^L).
// Slab intersection with half-open cells (reading Q8: the global max face inclusive).
// ------------------------------------------------------------------------------------
struct Ray {
    double o[3], d[3];
};

inline void cell_box(const or_tree* T, int level, const int64_t c[3], double lo[3], double hi[3]) {
    double n = std::ldexp(1.0, level);
    for (int k = 0; k < 3; ++k) {
        lo[k] = T->bbox_min[k] + T->edge * ((double)c[k] / n);
        hi[k] = T->bbox_min[k] + T->edge * ((double)(c[k] + 1) / n);
    }
}

// Intersect ray with box, clipped to [tlo, thi].  Returns false if empty.
inline bool slab(const Ray& r, const double lo[3], const double hi[3], bool hi_inclusive[3],
                 double tlo, double thi, double* a, double* b) {
    double t0 = tlo, t1 = thi;
    for (int k = 0; k < 3; ++k) {
        if (r.d[k] != 0.0) {
            double ta = (lo[k] - r.o[k]) / r.d[k];
            double tb = (hi[k] - r.o[k]) / r.d[k];
            if (ta > tb) std::swap(ta, tb);
            t0 = std::max(t0, ta);
            t1 = std::min(t1, tb);
        } else {
            bool in = r.o[k] >= lo[k] && (r.o[k] < hi[k] || (hi_inclusive[k] && r.o[k] <= hi[k]));
            if (!in) return false;
        }
    }
    *a = t0;
    *b = t1;
    return t1 > t0;
}

struct Ctx {
    const or_tree* T;
    Ray r;
    double root_hi[3];
    std::vector<Seg> segs;
    std::vector<NodeHit> nodes;
};

// recursive ordered descent.  Children whose box meets the ray's
// interval in positive length are visited in order of entry t.
void descend(Ctx& cx, int64_t node, int level, const int64_t cell[3], double tlo, double thi) {
    const or_tree* T = cx.T;
    cx.nodes.push_back({tlo});
    struct Cand { double a, b; int o; };
    Cand cand[8];
    int nc = 0;
    for (int o = 0; o < 8; ++o) {
        uint32_t e = T->child[node * 8 + o];
        if ((e >> 30) == 0) continue;
        int64_t c[3] = {cell[0] * 2 + ((o >> 2) & 1), cell[1] * 2 + ((o >> 1) & 1), cell[2] * 2 + (o & 1)};
        double lo[3], hi[3];
        cell_box(T, level + 1, c, lo, hi);
        bool inc[3];
        for (int k = 0; k < 3; ++k) inc[k] = hi[k] == cx.root_hi[k];
        double a, b;
        if (slab(cx.r, lo, hi, inc, tlo, thi, &a, &b)) cand[nc++] = {a, b, o};
    }
    std::sort(cand, cand + nc, [](const Cand& p, const Cand& q) { return p.a < q.a || (p.a == q.a && p.o < q.o); });
    for (int i = 0; i < nc; ++i) {
        uint32_t e = T->child[node * 8 + cand[i].o];
        uint32_t tag = e >> 30, idx = e & 0x3FFFFFFFu;
        int o = cand[i].o;
        int64_t c[3] = {cell[0] * 2 + ((o >> 2) & 1), cell[1] * 2 + ((o >> 1) & 1), cell[2] * 2 + (o & 1)};
        if (tag == 2)
            cx.segs.push_back({cand[i].a, cand[i].b, (int64_t)idx});
        else if (tag == 1)
            descend(cx, idx, level + 1, c, cand[i].a, cand[i].b);
    }
}

// Clip to the bbox (reading Q6: t_near = max(0, entry), t_far = exit).
bool clip_root(const or_tree* T, const Ray& r, double* tn, double* tf) {
    double lo[3], hi[3];
    int64_t c0[3] = {0, 0, 0};
    cell_box(T, 0, c0, lo, hi);
    bool inc[3] = {true, true, true};
    return slab(r, lo, hi, inc, 0.0, INFINITY, tn, tf);
}

// Brute force over all leaves (checks the recursive descent on tiny trees).
struct LeafBox {
    double lo[3], hi[3];
    bool inc[3];
    int64_t leaf;
};

void collect_leaf_boxes(const or_tree* T, int64_t node, int level, const int64_t cell[3], std::vector<LeafBox>& out) {
    double rlo[3], rhi[3];
    int64_t c0[3] = {0, 0, 0};
    cell_box(T, 0, c0, rlo, rhi);
    for (int o = 0; o < 8; ++o) {
        uint32_t e = T->child[node * 8 + o];
        uint32_t tag = e >> 30, idx = e & 0x3FFFFFFFu;
        int64_t c[3] = {cell[0] * 2 + ((o >> 2) & 1), cell[1] * 2 + ((o >> 1) & 1), cell[2] * 2 + (o & 1)};
        if (tag == 1) collect_leaf_boxes(T, idx, level + 1, c, out);
        if (tag == 2) {
            LeafBox lb;
            cell_box(T, level + 1, c, lb.lo, lb.hi);
            for (int k = 0; k < 3; ++k) lb.inc[k] = lb.hi[k] == rhi[k];
            lb.leaf = idx;
            out.push_back(lb);
        }
    }
}

void segments(const or_tree* T, const Ray& r, int mode, const std::vector<LeafBox>* boxes, Ctx& cx, double* tn,
              double* tf, bool* hit) {
    cx.T = T;
    cx.r = r;
    cx.segs.clear();
    cx.nodes.clear();
    int64_t c0[3] = {0, 0, 0};
    double lo[3];
    cell_box(T, 0, c0, lo, cx.root_hi);
    *hit = clip_root(T, r, tn, tf);
    if (!*hit) return;
    if (mode == 0) {
        descend(cx, 0, 0, c0, *tn, *tf);
    } else {
        for (const LeafBox& lb : *boxes) {
            double a, b;
            bool inc[3] = {lb.inc[0], lb.inc[1], lb.inc[2]};
            if (slab(r, lb.lo, lb.hi, inc, *tn, *tf, &a, &b)) cx.segs.push_back({a, b, lb.leaf});
        }
        std::sort(cx.segs.begin(), cx.segs.end(), [](const Seg& p, const Seg& q) { return p.t0 < q.t0; });
    }
}

inline double sigmoid(double z) { return 1.0 / (1.0 + std::exp(-z)); }

// Eq. (5): c_ch = S(sum_b k_{b,ch} Y_b)
// Spherical Gaussian basis: G(d; p, lambda) = e^{lambda (d . p - 1)}, p a unit axis.
void sg_basis(int B, const double* axes, const double* lambda, const double* dir, double* G) {
    for (int b = 0; b < B; ++b) {
        const double* p = axes + 3 * b;
        double n = std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
        double dp = (dir[0] * p[0] + dir[1] * p[1] + dir[2] * p[2]) / n;
        G[b] = std::exp(lambda[b] * (dp - 1.0));
    }
}

// the per-ray basis of the tree: SH (App. B.1) or SG
void ray_basis(const or_tree* T, const double* dir, double* Y) {
    if (T->sg_axes) {
        const int B = (T->sh_degree + 1) * (T->sh_degree + 1);
        sg_basis(B, T->sg_axes, T->sg_lambda, dir, Y);
    } else {
        sh_basis(T->sh_degree, T->sh_cs, dir, Y);
    }
}

inline void leaf_color(const or_tree* T, int64_t leaf, const double* Y, int B, double c[3]) {
    const int64_t off = leaf * (int64_t)B * 3;
    for (int ch = 0; ch < 3; ++ch) {
        double z = 0.0;
        for (int b = 0; b < B; ++b) {
            const double k = T->sh ? T->sh[off + b * 3 + ch] : (double)T->sh32[off + b * 3 + ch];
            z += k * Y[b];
        }
        c[ch] = sigmoid(z);
    }
}

struct Comp {
    double rgb[3];
    double T;
    int nproc;
    bool terminated;
};

// Eq. (1)-(2) with background and early stop (reading Q11).
Comp composite(const or_tree* T, const std::vector<Seg>& segs, const double* Y, int B, double gamma, const double* bg) {
    Comp r{{0, 0, 0}, 1.0, 0, false};
    double Tr = 1.0;
    for (const Seg& s : segs) {
        double sig = std::max((double)T->sigma[s.leaf], 0.0);   // sigma = (sigma~)_+
        double delta = s.t1 - s.t0;
        double alpha = -std::expm1(-sig * delta);               // 1 - exp(-sigma delta)
        double c[3];
        leaf_color(T, s.leaf, Y, B, c);
        for (int ch = 0; ch < 3; ++ch) r.rgb[ch] += Tr * alpha * c[ch];
        Tr = Tr * std::exp(-sig * delta);
        r.nproc++;
        if (Tr < gamma) {
            r.terminated = true;
            break;
        }
    }
    for (int ch = 0; ch < 3; ++ch) r.rgb[ch] += Tr * bg[ch];
    r.T = Tr;
    return r;
}

inline Ray make_ray(const double* p) {
    Ray r;
    double n = std::sqrt(p[3] * p[3] + p[4] * p[4] + p[5] * p[5]);
    for (int k = 0; k < 3; ++k) {
        r.o[k] = p[k];
        r.d[k] = p[3 + k] / n;
    }
    return r;
}

int set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) return nthreads;
    return omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}

}  // namespace

extern "C" {

int or_sh_basis(int lmax, int cs, const double* dir, double* Y) {
    if (lmax < 0 || lmax > 10) return 1;
    sh_basis(lmax, cs, dir, Y);
    return 0;
}

int or_sg_basis(int B, const double* axes, const double* lambda, int64_t n, const double* dirs, double* G) {
    if (B < 1) return 1;
    for (int64_t i = 0; i < n; ++i) sg_basis(B, axes, lambda, dirs + i * 3, G + i * B);
    return 0;
}

// Batched form: dirs [n][3] -> Y [n][(lmax+1)^2]
int or_sh_basis_n(int lmax, int cs, int64_t n, const double* dirs, double* Y) {
    if (lmax < 0 || lmax > 10) return 1;
    int B = (lmax + 1) * (lmax + 1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) sh_basis(lmax, cs, dirs + i * 3, Y + i * B);
    return 0;
}

// Pinhole camera, pixel centres, OpenGL axes (reading Q5).  cam = c2w[3][4], fx, fy, cx, cy.
void or_camera_rays(const float* cam, int W, int H, double* rays) {
    for (int j = 0; j < H; ++j)
        for (int i = 0; i < W; ++i) {
            double dc[3] = {((double)i + 0.5 - cam[14]) / cam[12], -((double)j + 0.5 - cam[15]) / cam[13], -1.0};
            double d[3];
            for (int k = 0; k < 3; ++k) d[k] = cam[k * 4 + 0] * dc[0] + cam[k * 4 + 1] * dc[1] + cam[k * 4 + 2] * dc[2];
            double n = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            double* out = rays + ((int64_t)j * W + i) * 6;
            for (int k = 0; k < 3; ++k) {
                out[k] = cam[k * 4 + 3];
                out[3 + k] = d[k] / n;
            }
        }
}

// All positive-length leaf segments of one ray in t order (no early stop).
// mode 0 = recursive descent, 1 = brute force over all leaves.  Returns the count
// (may exceed max_seg; only the first max_seg are written).
int64_t or_trace_ray(const or_tree* T, const double* ray, int mode, int64_t max_seg, int64_t* leaf, double* t_in,
                     double* t_out, double* t_near_far) {
    std::vector<LeafBox> boxes;
    if (mode == 1) {
        int64_t c0[3] = {0, 0, 0};
        collect_leaf_boxes(T, 0, 0, c0, boxes);
    }
    Ctx cx;
    double tn = 0, tf = 0;
    bool hit;
    segments(T, make_ray(ray), mode, &boxes, cx, &tn, &tf, &hit);
    if (t_near_far) {
        t_near_far[0] = hit ? tn : NAN;
        t_near_far[1] = hit ? tf : NAN;
    }
    int64_t n = (int64_t)cx.segs.size();
    for (int64_t i = 0; i < n && i < max_seg; ++i) {
        leaf[i] = cx.segs[i].leaf;
        t_in[i] = cx.segs[i].t0;
        t_out[i] = cx.segs[i].t1;
    }
    return n;
}

// Forward render of n rays ([n][6] = o, d; d is normalised here).
// Outputs: rgb [n][3], T_final [n], n_proc [n] (leaves composited), optional
// leaf_ids [n][max_leaves] (visited sequence, -1 padded), nodes_met [n] (internal
// nodes, root included, whose box the processed interval meets).
int or_render(const or_tree* T, const double* rays, int64_t n, double gamma, const double* bg, int mode, double* rgb,
              double* T_final, int32_t* n_proc, int32_t max_leaves, int32_t* leaf_ids, int32_t* nodes_met,
              int nthreads) {
    int B = (T->sh_degree + 1) * (T->sh_degree + 1);
    std::vector<LeafBox> boxes;
    if (mode == 1) {
        int64_t c0[3] = {0, 0, 0};
        collect_leaf_boxes(T, 0, 0, c0, boxes);
    }
    int nt = set_threads(nthreads);
#pragma omp parallel num_threads(nt)
    {
        Ctx cx;
        std::vector<double> Y(B);
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            Ray r = make_ray(rays + i * 6);
            double tn, tf;
            bool hit;
            segments(T, r, mode, &boxes, cx, &tn, &tf, &hit);
            ray_basis(T, r.d, Y.data());
            Comp c = composite(T, cx.segs, Y.data(), B, gamma, bg);
            for (int ch = 0; ch < 3; ++ch) rgb[i * 3 + ch] = c.rgb[ch];
            if (T_final) T_final[i] = c.T;
            if (n_proc) n_proc[i] = c.nproc;
            if (leaf_ids) {
                for (int j = 0; j < max_leaves; ++j) leaf_ids[i * max_leaves + j] = j < c.nproc ? (int32_t)cx.segs[j].leaf : -1;
            }
            if (nodes_met) {
                int cnt = 0;
                if (hit) {
                    double lim = (c.terminated && c.nproc > 0) ? cx.segs[c.nproc - 1].t0 : INFINITY;
                    for (const NodeHit& nh : cx.nodes) cnt += nh.t0 <= lim;
                }
                nodes_met[i] = cnt;
            }
        }
    }
    return 0;
}

// Analytic backward with direct suffix sums in double.
// grad_sigma [n_leaves], grad_sh [n_leaves][B][3] are ACCUMULATED (+=).  If non-NULL,
// sigma_scale / sh_scale accumulate the magnitude of what was summed into each component
// (|delta| sum_ch |g| (|c T| + |S|) and |g w c (1-c) Y|): the natural yardstick for the rounding
// error of any implementation that forms and sums those terms in finite precision.
int or_backward(const or_tree* T, const double* rays, int64_t n, double gamma, const double* bg, const double* dL_dC,
                double* grad_sigma, double* grad_sh, int nthreads, double* sigma_scale, double* sh_scale) {
    int B = (T->sh_degree + 1) * (T->sh_degree + 1);
    int nt = set_threads(nthreads);
#pragma omp parallel num_threads(nt)
    {
        Ctx cx;
        std::vector<double> Y(B);
        std::vector<double> Ti, w, col, S;
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            Ray r = make_ray(rays + i * 6);
            double tn, tf;
            bool hit;
            segments(T, r, 0, nullptr, cx, &tn, &tf, &hit);
            if (!hit) continue;
            ray_basis(T, r.d, Y.data());
            // forward quantities up to termination: M processed segments, T_0..T_M
            Ti.assign(1, 1.0);
            w.clear();
            col.clear();
            int M = 0;
            for (const Seg& s : cx.segs) {
                double sig = std::max((double)T->sigma[s.leaf], 0.0);
                double delta = s.t1 - s.t0;
                double c[3];
                leaf_color(T, s.leaf, Y.data(), B, c);
                double Tnext = Ti.back() * std::exp(-sig * delta);
                w.push_back(Ti.back() * -std::expm1(-sig * delta));   // w_i = T_i (1 - e^{-sigma delta})
                for (int ch = 0; ch < 3; ++ch) col.push_back(c[ch]);
                Ti.push_back(Tnext);
                ++M;
                if (Tnext < gamma) break;
            }
            // S_i = sum_{k=i+1}^{M} c_k w_k  with w_M = T_M, c_M = background
            S.assign((size_t)(M + 1) * 3, 0.0);
            for (int ch = 0; ch < 3; ++ch) S[(size_t)M * 3 + ch] = 0.0;
            double acc[3] = {Ti[M] * bg[0], Ti[M] * bg[1], Ti[M] * bg[2]};
            for (int k = M - 1; k >= 0; --k) {
                for (int ch = 0; ch < 3; ++ch) S[(size_t)k * 3 + ch] = acc[ch];
                for (int ch = 0; ch < 3; ++ch) acc[ch] += col[(size_t)k * 3 + ch] * w[k];
            }
            const double* g = dL_dC + i * 3;
            for (int k = 0; k < M; ++k) {
                int64_t leaf = cx.segs[k].leaf;
                double st = (double)T->sigma[leaf];
                double delta = cx.segs[k].t1 - cx.segs[k].t0;
                if (st > 0.0) {   // ReLU gate: zero for sigma~ <= 0 (reading Q21)
                    double gs = 0.0, mag = 0.0;
                    for (int ch = 0; ch < 3; ++ch) {
                        gs += g[ch] * (col[(size_t)k * 3 + ch] * Ti[k + 1] - S[(size_t)k * 3 + ch]);
                        mag += std::fabs(g[ch]) * (std::fabs(col[(size_t)k * 3 + ch] * Ti[k + 1]) +
                                                   std::fabs(S[(size_t)k * 3 + ch]));
                    }
                    gs *= delta;
#pragma omp atomic
                    grad_sigma[leaf] += gs;
                    if (sigma_scale) {
#pragma omp atomic
                        sigma_scale[leaf] += std::fabs(delta) * mag;
                    }
                }
                for (int ch = 0; ch < 3; ++ch) {
                    double c = col[(size_t)k * 3 + ch];
                    double gz = g[ch] * w[k] * c * (1.0 - c);   // dC/dc = w, dc/dz = c(1-c)
                    if (gz == 0.0) continue;
                    for (int b = 0; b < B; ++b) {
#pragma omp atomic
                        grad_sh[(leaf * B + b) * 3 + ch] += gz * Y[b];
                        if (sh_scale) {
#pragma omp atomic
                            sh_scale[(leaf * B + b) * 3 + ch] += std::fabs(gz * Y[b]);
                        }
                    }
                }
            }
        }
    }
    return 0;
}

// NEXT f4 ("render the depth map"; alpha maps P:468): per ray, over the segments
// composited up to termination (Eq. 1-2 weights w_i = T_i (1 - exp(-sigma_i delta_i))):
//   alpha = 1 - T_stop,   depth = sum_i w_i (t_in,i + t_out,i) / 2     (reading Q34)
// t in world units from the ray origin along the unit direction; the background adds 0.
int or_render_depth(const or_tree* T, const double* rays, int64_t n, double gamma, double* alpha, double* depth,
                    int nthreads) {
    int nt = set_threads(nthreads);
#pragma omp parallel num_threads(nt)
    {
        Ctx cx;
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            Ray r = make_ray(rays + i * 6);
            double tn, tf;
            bool hit;
            segments(T, r, 0, nullptr, cx, &tn, &tf, &hit);
            double Tr = 1.0, D = 0.0;
            if (hit) {
                for (const Seg& s : cx.segs) {
                    double sig = std::max((double)T->sigma[s.leaf], 0.0);
                    double delta = s.t1 - s.t0;
                    double w = Tr * -std::expm1(-sig * delta);
                    D += w * 0.5 * (s.t0 + s.t1);
                    Tr = Tr * std::exp(-sig * delta);
                    if (Tr < gamma) break;
                }
            }
            alpha[i] = 1.0 - Tr;
            depth[i] = D;
        }
    }
    return 0;
}

// NEXT f1, visibility filtering: "keeping track of the maximum ray weight
// 1 - exp(-sigma_i delta_i) at each voxel" over the leaves each ray composites before it
// terminates (reading Q33).  max_alpha [n_leaves] is max-accumulated (caller initialises).
int or_leaf_max_alpha(const or_tree* T, const double* rays, int64_t n, double gamma, double* max_alpha,
                      int nthreads) {
    int nt = set_threads(nthreads);
    std::vector<std::vector<double>> part((size_t)nt);
#pragma omp parallel num_threads(nt)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        std::vector<double>& mine = part[(size_t)tid];
        mine.assign((size_t)T->n_leaves, 0.0);
        Ctx cx;
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            Ray r = make_ray(rays + i * 6);
            double tn, tf;
            bool hit;
            segments(T, r, 0, nullptr, cx, &tn, &tf, &hit);
            if (!hit) continue;
            double Tr = 1.0;
            for (const Seg& s : cx.segs) {
                double sig = std::max((double)T->sigma[s.leaf], 0.0);
                double delta = s.t1 - s.t0;
                double a = -std::expm1(-sig * delta);   // 1 - exp(-sigma delta)
                mine[(size_t)s.leaf] = std::max(mine[(size_t)s.leaf], a);
                Tr = Tr * std::exp(-sig * delta);
                if (Tr < gamma) break;
            }
        }
    }
    for (const std::vector<double>& v : part)
        for (size_t j = 0; j < v.size(); ++j) max_alpha[j] = std::max(max_alpha[j], v[j]);
    return 0;
}

// Tie tags (reading Q27).  A ray is a tie when an implementation that evaluates the
// same definition in floating point with unit roundoff `eps` (2^-24 for fp32) may legitimately
// produce a different visited-leaf sequence or stop at a different segment.  Such an
// implementation computes a plane crossing t = (p - o_k)/d_k with an absolute error of at most
//   e(t) = 2 eps |o_k - b_k| / |d_k| + 12 eps t      (world units; o rounded into grid units,
//                                                    one subtraction, one reciprocal, products)
// -- the oracle evaluates the bound in double for every crossing it uses.
//   bit0: two consecutive crossings (level-D planes on any axis, t_near, t_far) inside
//         [t_near, t_far], up to the stop, whose order is not determined (gap <= e_a + e_b),
//         where a LEAF touches the crossing point (probes straddling both planes): only then can
//         a different order change the visited leaves;
//   bit1: a processed segment no longer than the error of its two ends;
//   bit2: some T_{i+1} within its error band of gamma up to the stop;
//   bit3: the origin (inside the box) within its rounding error of a level-D plane.
// The band is the optical-depth error sum_k sigma_k (e(t_in,k) + e(t_out,k)) + 10 eps per
// segment, plus 2 (e_a + e_b) sigma_max for every bit-0 crossing pair (a sliver leaf that may be
// entered or skipped).  C = sum_i T_i alpha_i c_i + T_N c_N with colours in [0, 1] moves by at
// most |d tau| when one segment's optical depth tau moves by d tau, so
//   bound = band + [bit2] gamma (1 + band)
// bounds |C_impl - C_oracle| of the ray beyond the implementation's own rounding (optional
// output; the GPU tests assert it on every excluded ray).
namespace {
struct Crossing {
    double t, e;
};

// entry of the tree at point q (0 = empty / outside): plain walk down the child table
uint32_t entry_at(const or_tree* T, const double q[3]) {
    double u[3];
    for (int k = 0; k < 3; ++k) {
        u[k] = (q[k] - T->bbox_min[k]) / T->edge;
        if (!(u[k] >= 0.0 && u[k] < 1.0)) return 0u;
    }
    int64_t node = 0;
    for (int level = 0; level < 62; ++level) {
        double n = std::ldexp(1.0, level + 1);
        int oct = 0;
        for (int k = 0; k < 3; ++k) oct |= (int)((int64_t)std::floor(u[k] * n) & 1) << (2 - k);
        uint32_t e = T->child[node * 8 + oct];
        if ((e >> 30) != 1u) return e;
        node = e & 0x3FFFFFFFu;
    }
    return 0u;
}
}  // namespace

int or_tie_flags(const or_tree* T, const double* rays, int64_t n, double gamma, double eps, uint8_t* flags,
                 double* bound, int nthreads) {
    int nt = set_threads(nthreads);
    int64_t G = (int64_t)1 << T->depth;
#pragma omp parallel num_threads(nt)
    {
        Ctx cx;
        std::vector<Crossing> cs;
        struct Tie {
            double t, dtau;
        };
        std::vector<Tie> ties;
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            Ray r = make_ray(rays + i * 6);
            double tn, tf;
            bool hit;
            segments(T, r, 0, nullptr, cx, &tn, &tf, &hit);
            uint8_t f = 0;
            double bnd = 0.0;
            if (hit) {
                double slope[3];   // |o_k - b_k| / |d_k|: the crossing error per axis
                for (int k = 0; k < 3; ++k)
                    slope[k] = r.d[k] != 0.0 ? std::fabs(r.o[k] - T->bbox_min[k]) / std::fabs(r.d[k]) : 0.0;
                auto err = [&](int k, double t) { return 2.0 * eps * slope[k] + 12.0 * eps * t; };
                cs.clear();
                double e_tn = 0.0, e_tf = 0.0;   // t_near / t_far: the bbox face that sets them
                for (int k = 0; k < 3; ++k) {
                    if (r.d[k] == 0.0) continue;
                    for (int64_t j = 0; j <= G; ++j) {
                        double plane = T->bbox_min[k] + T->edge * ((double)j / (double)G);
                        double t = (plane - r.o[k]) / r.d[k];
                        if (t == tn && tn > 0.0) e_tn = std::max(e_tn, err(k, t));
                        if (t == tf) e_tf = std::max(e_tf, err(k, t));
                        if (t > tn && t < tf) cs.push_back({t, err(k, t)});
                    }
                }
                cs.push_back({tn, e_tn});
                cs.push_back({tf, e_tf});
                std::sort(cs.begin(), cs.end(), [](const Crossing& a, const Crossing& b) { return a.t < b.t; });
                auto e_of = [&](double t) {   // error of a segment end: the crossing with that exact t
                    auto it = std::lower_bound(cs.begin(), cs.end(), t,
                                               [](const Crossing& a, double v) { return a.t < v; });
                    double e = 0.0;
                    for (; it != cs.end() && it->t == t; ++it) e = std::max(e, it->e);
                    return e;
                };
                // undetermined crossing orders where a leaf touches the crossing point
                ties.clear();
                for (size_t a = 1; a < cs.size(); ++a) {
                    const Crossing& p = cs[a - 1];
                    const Crossing& q = cs[a];
                    double tol = p.e + q.e;
                    if (q.t - p.t > tol) continue;
                    double tm = 0.5 * (p.t + q.t), h = 3.0 * tol + 1e-12 * T->edge;
                    bool leaf = false;
                    double smax = 0.0;
                    for (int c = 0; c < 8; ++c) {
                        double pt[3];
                        for (int k = 0; k < 3; ++k) pt[k] = r.o[k] + tm * r.d[k] + (((c >> k) & 1) ? h : -h);
                        uint32_t e = entry_at(T, pt);
                        if ((e >> 30) == 2u) {
                            leaf = true;
                            smax = std::max(smax, (double)T->sigma[e & 0x3FFFFFFFu]);
                        }
                    }
                    if (leaf) ties.push_back({tm, 2.0 * tol * smax});
                }
                // forward up to the stop: bits 1 and 2, the band, and the stop itself
                double Tr = 1.0, band = 0.0, t_stop = tf;
                size_t ti = 0;
                bool near_gamma = false;
                for (const Seg& s : cx.segs) {
                    double ea = e_of(s.t0), eb = e_of(s.t1);
                    if (s.t1 - s.t0 <= ea + eb) f |= 2;
                    double sig = std::max((double)T->sigma[s.leaf], 0.0);
                    Tr *= std::exp(-sig * (s.t1 - s.t0));
                    band += sig * (ea + eb) + 10.0 * eps;
                    for (; ti < ties.size() && ties[ti].t <= s.t1 + eb; ++ti) {
                        band += ties[ti].dtau;
                        f |= 1;
                    }
                    if (gamma > 0 && std::fabs(Tr - gamma) <= band * std::max(Tr, gamma)) near_gamma = true;
                    if (Tr < gamma) {
                        t_stop = s.t1 + eb;
                        break;
                    }
                }
                for (; ti < ties.size() && ties[ti].t <= t_stop; ++ti) {   // ties after the last segment
                    band += ties[ti].dtau;
                    f |= 1;
                }
                if (near_gamma) f |= 4;
                bnd = band + (near_gamma ? gamma * (1.0 + band) : 0.0);
                if (tn == 0.0) {
                    for (int k = 0; k < 3; ++k) {
                        double u = (r.o[k] - T->bbox_min[k]) / T->edge * (double)G;
                        double dist = std::fabs(u - std::round(u)) * T->edge / (double)G;
                        if (dist <= 4.0 * eps * (std::fabs(r.o[k] - T->bbox_min[k]) + T->edge)) f |= 8;
                    }
                }
            }
            flags[i] = f;
            if (bound) bound[i] = bnd;
        }
    }
    return 0;
}

}  // extern "C"
