/* Plain-C use of libplenoct through include/plenoct.h only (no CUDA headers, no PyTorch):
 * a uniform depth-2 PlenOctree (64 leaves, sigma~ = 1.5, SH degree 0), one 64x64 view rendered
 * into a host image with po_render_host, every pixel checked against the closed form of a
 * constant medium: C = S(k Y00) (1 - T) + T bg with T = exp(-sigma chord) (Eq. 1-2, P:238-243;
 * Y00 = 1 / (2 sqrt(pi)), App. B.1).  Prints "OK" and returns 0 on success.
 * Build:  gcc render_uniform.c -I../include -L../paper_2103_14024_b200 -lplenoct -lm */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "plenoct.h"

static double slab_chord(const double o[3], const double d[3]) {
    double tn = 0.0, tf = INFINITY;
    for (int k = 0; k < 3; ++k) {
        if (d[k] == 0.0) {
            if (o[k] < -1.0 || o[k] > 1.0) return 0.0;
            continue;
        }
        double a = (-1.0 - o[k]) / d[k], b = (1.0 - o[k]) / d[k];
        if (a > b) { double t = a; a = b; b = t; }
        if (a > tn) tn = a;
        if (b < tf) tf = b;
    }
    return tf > tn ? tf - tn : 0.0;
}

int main(void) {
    enum { W = 64, H = 64, NN = 9, NL = 64 };
    uint32_t child[NN * 8];
    for (int o = 0; o < 8; ++o) child[o] = (1u << 30) | (uint32_t)(1 + o);          /* root -> nodes 1..8 */
    for (int n = 1; n < NN; ++n)
        for (int o = 0; o < 8; ++o) child[n * 8 + o] = (2u << 30) | (uint32_t)((n - 1) * 8 + o);   /* leaves */
    float sigma[NL], sh[NL * 3];
    const float k = 0.8f;
    for (int i = 0; i < NL; ++i) {
        sigma[i] = 1.5f;
        sh[3 * i] = sh[3 * i + 1] = sh[3 * i + 2] = k;
    }
    po_tree_desc desc = {{-1.f, -1.f, -1.f}, 2.f, 2, 0, PO_F32, PO_SH_CS, 0, 0};
    po_tree* tree = NULL;
    if (po_tree_create(&desc, child, NN, sigma, sh, NL, &tree) != PO_OK) {
        fprintf(stderr, "po_tree_create: %s\n", po_last_error());
        return 1;
    }
    int64_t nn = 0, nl = 0;
    int32_t row = 0;
    if (po_tree_info(tree, &nn, &nl, &row) != PO_OK || nn != NN || nl != NL) return 2;
    /* camera at (0.1, -0.2, 3) looking down -z (OpenGL axes, reading Q5) */
    po_camera cam = {{{1.f, 0.f, 0.f, 0.1f}, {0.f, 1.f, 0.f, -0.2f}, {0.f, 0.f, 1.f, 3.f}}, 48.f, 48.f, 32.f, 32.f};
    po_render_opts opts = {0.0f, {1.f, 1.f, 1.f}};   /* gamma 0: no early stop, white background */
    static float img[H * W * 3];
    if (po_render_host(tree, &cam, 1, W, H, &opts, img, NULL) != PO_OK) {
        fprintf(stderr, "po_render_host: %s\n", po_last_error());
        return 3;
    }
    const double c = 1.0 / (1.0 + exp(-(double)k * 0.28209479177387814));
    double worst = 0.0;
    for (int j = 0; j < H; ++j)
        for (int i = 0; i < W; ++i) {
            const double o[3] = {0.1, -0.2, 3.0};
            double d[3] = {(i + 0.5 - 32.0) / 48.0, -((j + 0.5 - 32.0) / 48.0), -1.0};
            const double nd = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            for (int q = 0; q < 3; ++q) d[q] /= nd;
            const double T = exp(-(double)sigma[0] * slab_chord(o, d));
            const double want = c * (1.0 - T) + T;
            for (int ch = 0; ch < 3; ++ch) {
                const double err = fabs(img[(j * W + i) * 3 + ch] - want);
                if (err > worst) worst = err;
            }
        }
    /* an invalid call reports an error status and a message instead of crashing */
    po_render_opts bad = {2.f, {1.f, 1.f, 1.f}};
    const int bad_ok = po_render_host(tree, &cam, 1, W, H, &bad, img, NULL) == PO_ERR_INVALID_ARG &&
                       po_last_error()[0] != '\0';
    po_tree_destroy(tree);
    printf("libplenoct %s: max |C - closed form| = %.3e\n", po_version(), worst);
    if (worst > 2e-5 || !bad_ok) return 4;
    printf("OK\n");
    return 0;
}
