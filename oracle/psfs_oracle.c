/*
 * psfs_oracle.c -- plain, slow, obviously-correct CPU oracle of the PSFS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path
 * (paper_1311_6811_b200/csrc/), and the CUDA path never calls it.
 *
 * Citation keys: P:n = PAPER.md line n (arXiv 1311.6811, "Digitize Your Body and
 * Action in 3-D at Over 10 FPS"), S:n = SPEC.md line n, R#n = reading n of the
 * DESIGN.md "Readings" table (where the paper is silent or garbled).
 *
 * Arithmetic: double precision everywhere, EXCEPT the voxel->pixel projection
 * (oracle_project_pinned), whose FP32 operation sequence is pinned by the
 * specification in DESIGN.md (R#11, R#16): nearest-pixel sampling is
 * discontinuous, so both sides evaluate the same correctly-rounded float ops.
 * Build with -O2 -ffp-contract=off and without -ffast-math so that every
 * float/double operation below is one IEEE-754 correctly-rounded operation.
 *
 * Parity status of each function is recorded in DESIGN.md ("Oracle pins");
 * every function here is pinned by tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "psfs_oracle.h"

/* ------------------------------------------------------------------------ */
/* Stage 1: silhouette likelihood map, Eq (1)-(2), and per-view likelihoods,  */
/* Eq (5)-(9).                                                                */
/* ------------------------------------------------------------------------ */

/* ln N(x | mu, s): one channel of the single Gaussian background model
 * P(I | F=0) ~ N(I | mu, sigma).  sigma is a standard deviation, per
 * channel, channels independent (R#2, R#3). */
static double ln_gauss(double x, double mu, double s)
{
    const double z = (x - mu) / s;
    return -0.5 * z * z - log(s) - 0.5 * log(2.0 * M_PI);
}

/* ln U(I): uniform foreground density over the 8-bit RGB cube, (1/256)^3
 * ("the foreground obeys a uniform distribution"; R#4). */
static double ln_uniform_rgb(void) { return -3.0 * log(256.0); }

void oracle_pixel(const uint8_t I[3], const float mu[3], const float sigma[3],
                  double sigma_floor, double p_occ,
                  double *slm_out, double *lnp1_out, double *lnp0_out)
{
    /* Eq (1): P(F=1|I) = P(I|F=1)P(F=1) / sum_{F in {0,1}} P(I|F)P(F)  (
     * the garbled "sum_{F=0}" is read as the sum over F in {0,1}, R#1), with
     * P(F=1) = P(F=0) = 0.5, P(I|F=1) = U, P(I|F=0) = N.
     * Evaluated in log space to avoid underflow of the density product (R#16). */
    double ln_g = 0.0; /* ln P(I|F=0) = sum_ch ln N(I_ch | mu_ch, sigma'_ch) */
    for (int ch = 0; ch < 3; ++ch) {
        double s = (double)sigma[ch];
        if (s < sigma_floor) s = sigma_floor; /* sigma floor (R#6) */
        ln_g += ln_gauss((double)I[ch], (double)mu[ch], s);
    }
    const double ln_fg = ln_uniform_rgb() + log(0.5); /* ln P(I|F=1)P(F=1) */
    const double ln_bg = ln_g + log(0.5);             /* ln P(I|F=0)P(F=0) */
    /* SLM = fg/(fg+bg) = 1/(1+exp(ln_bg-ln_fg));  1-SLM = 1/(1+exp(ln_fg-ln_bg)).
     * Both are formed as logistic functions so that neither loses precision by
     * cancellation (Eq 2). */
    const double dd = ln_bg - ln_fg;
    const double slm = 1.0 / (1.0 + exp(dd));
    const double one_minus_slm = 1.0 / (1.0 + exp(-dd));

    /* Eq (5): P(S|V) = sum_O P(S|O,V) P(O),  P(O=1) = p_occ (R#7).
     * Eq (6): P(S|O=0,V=0) = 1 - SLM;  Eq (7)-(9): the other three = SLM. */
    const double p_o1 = p_occ, p_o0 = 1.0 - p_occ;
    const double p_s_v1 = p_o0 * slm /* Eq 8 */ + p_o1 * slm /* Eq 9 */;
    const double p_s_v0 = p_o0 * one_minus_slm /* Eq 6 */ + p_o1 * slm /* Eq 7 */;

    if (slm_out) *slm_out = slm;
    if (lnp1_out) *lnp1_out = log(p_s_v1);
    if (lnp0_out) *lnp0_out = log(p_s_v0);
}

/* Per-view likelihood pair for a hand-set SLM value (used for out-of-view
 * views, SLM = 1/2 (R#12), and by the closed-form pins). Eq (5)-(9). */
void oracle_view_likelihood(double slm, double p_occ, double *lnp1, double *lnp0)
{
    const double p_o1 = p_occ, p_o0 = 1.0 - p_occ;
    *lnp1 = log(p_o0 * slm + p_o1 * slm);
    *lnp0 = log(p_o0 * (1.0 - slm) + p_o1 * slm);
}

void oracle_slm_image(int W, int H, const uint8_t *img, const float *mu, const float *sigma,
                      double sigma_floor, double p_occ, double *slm, double *lnp1, double *lnp0,
                      int nthreads)
{
    const int64_t n = (int64_t)W * H;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t p = 0; p < n; ++p) {
        oracle_pixel(img + 3 * p, mu + 3 * p, sigma + 3 * p, sigma_floor, p_occ,
                     slm ? slm + p : NULL, lnp1 ? lnp1 + p : NULL, lnp0 ? lnp0 + p : NULL);
    }
    (void)nthreads;
}

/* ------------------------------------------------------------------------ */
/* Voxel -> pixel projection ("the pixel ... is the projection of voxel V_i", */
/* P:91; nearest pixel, R#10; pixel centres at integers, round half up, R#11). */
/* ------------------------------------------------------------------------ */

/* O4: fold the lattice->world map T (voxel centre = origin + spacing*(idx+1/2),
 * S:181, R#13) and the +1/2 pixel shift S (round-half-up = floor(x/w + 1/2))
 * into one 3x4 float matrix A = S * P * T, computed in double in a fixed
 * order, each entry rounded once to float. */
void oracle_precompose(const double P[12], const double origin[3], double spacing, float A[12])
{
    double Q[3][4];
    for (int c = 0; c < 4; ++c) {
        Q[0][c] = P[0 * 4 + c] + 0.5 * P[2 * 4 + c];
        Q[1][c] = P[1 * 4 + c] + 0.5 * P[2 * 4 + c];
        Q[2][c] = P[2 * 4 + c];
    }
    double cen[3];
    for (int a = 0; a < 3; ++a) cen[a] = origin[a] + 0.5 * spacing;
    for (int r = 0; r < 3; ++r) {
        A[r * 4 + 0] = (float)(spacing * Q[r][0]);
        A[r * 4 + 1] = (float)(spacing * Q[r][1]);
        A[r * 4 + 2] = (float)(spacing * Q[r][2]);
        A[r * 4 + 3] = (float)(((Q[r][0] * cen[0] + Q[r][1] * cen[1]) + Q[r][2] * cen[2]) + Q[r][3]);
    }
}

/* O5: pinned FP32 projection of lattice point (i,j,k).  Returns 1 and the
 * pixel if the voxel centre is in view (in front of the camera, w > 0, and
 * inside the image, R#12), else 0.  Every operation is one correctly
 * rounded float op: three fmaf chains, one reciprocal, two products, floor. */
int oracle_project_pinned(const float A[12], int W, int H, int i, int j, int k,
                          int *px, int *py)
{
    const float fi = (float)i, fj = (float)j, fk = (float)k;
    const float x = fmaf(A[2], fk, fmaf(A[1], fj, fmaf(A[0], fi, A[3])));
    const float y = fmaf(A[6], fk, fmaf(A[5], fj, fmaf(A[4], fi, A[7])));
    const float w = fmaf(A[10], fk, fmaf(A[9], fj, fmaf(A[8], fi, A[11])));
    if (!(w > 0.0f)) return 0;
    const float rr = 1.0f / w;
    const float u = x * rr;
    const float v = y * rr;
    if (!(u >= 0.0f && u < (float)W && v >= 0.0f && v < (float)H)) return 0;
    *px = (int)floorf(u);
    *py = (int)floorf(v);
    return 1;
}

/* The same projection evaluated exactly in double from the unrounded camera
 * matrix and voxel centre: pixel = floor(x/w + 1/2).  Used only for the
 * pinned-vs-exact disagreement diagnostic (SURVEY §8(c) diagnostic (i)). */
int oracle_project_exact(const double P[12], const double origin[3], double spacing,
                         int W, int H, int i, int j, int k, int *px, int *py)
{
    const double X = origin[0] + spacing * (i + 0.5);
    const double Y = origin[1] + spacing * (j + 0.5);
    const double Z = origin[2] + spacing * (k + 0.5);
    const double x = P[0] * X + P[1] * Y + P[2] * Z + P[3];
    const double y = P[4] * X + P[5] * Y + P[6] * Z + P[7];
    const double w = P[8] * X + P[9] * Y + P[10] * Z + P[11];
    if (!(w > 0.0)) return 0;
    const double u = x / w + 0.5, v = y / w + 0.5;
    if (!(u >= 0.0 && u < (double)W && v >= 0.0 && v < (double)H)) return 0;
    *px = (int)floor(u);
    *py = (int)floor(v);
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Stage 2: occupancy posterior, Eq (3)-(4), and thresholding.        */
/* ------------------------------------------------------------------------ */

static double posterior_from_logs(double a1, double a0)
{
    /* Eq (3): P(V=1|S) = e^a1 / (e^a1 + e^a0), a_v = ln P({S}|V=v) + ln P(V=v). */
    const double m = a1 > a0 ? a1 : a0;
    const double e1 = exp(a1 - m), e0 = exp(a0 - m);
    return e1 / (e1 + e0);
}

/* One voxel, given per-camera (lnP(S|V=1), lnP(S|V=0)) images. */
static void fuse_voxel(const oracle_rig *rig, const double *const *lnp1,
                       const double *const *lnp0, double p_vox, int i, int j, int k,
                       double *L, double *post)
{
    /* Eq (4): ln P({S}_n | V) = sum_k ln P(S_k | V), cameras in order 0..n-1. */
    double s1 = 0.0, s0 = 0.0;
    double h1, h0; /* out-of-view view: SLM = 1/2, uninformative (R#12) */
    oracle_view_likelihood(0.5, rig->p_occ, &h1, &h0);
    for (int c = 0; c < rig->ncam; ++c) {
        int px, py;
        if (oracle_project_pinned(rig->A + 12 * c, rig->W[c], rig->H[c], i, j, k, &px, &py)) {
            const int64_t p = (int64_t)py * rig->W[c] + px;
            s1 += lnp1[c][p];
            s0 += lnp0[c][p];
        } else {
            s1 += h1;
            s0 += h0;
        }
    }
    /* Eq (3) with the voxel prior P(V=1) = p_vox (R#8). */
    const double a1 = s1 + log(p_vox), a0 = s0 + log(1.0 - p_vox);
    *L = a1 - a0; /* log-odds of the posterior (R#18) */
    *post = posterior_from_logs(a1, a0);
}

void oracle_fuse(const oracle_rig *rig, const oracle_grid *g, const double *const *lnp1,
                 const double *const *lnp0, double p_vox, double tau, int k0, int k1,
                 double *L_out, double *post_out, uint32_t *bits_out, int nthreads)
{
    /* bits_out (if given) must be zeroed by the caller; bits are OR-ed in. */
    const int64_t plane = (int64_t)g->xlen * g->ylen;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int k = k0; k < k1; ++k) {
        for (int j = 0; j < g->ylen; ++j) {
            for (int i = 0; i < g->xlen; ++i) {
                double L, post;
                fuse_voxel(rig, lnp1, lnp0, p_vox, i, j, k, &L, &post);
                const int64_t v = (int64_t)i + (int64_t)g->xlen * (j + (int64_t)g->ylen * k);
                const int64_t o = v - plane * k0; /* outputs are slab-relative */
                if (L_out) L_out[o] = L;
                if (post_out) post_out[o] = post;
                if (bits_out) {
                    /* thresholding: occupied iff posterior > tau (R#14);
                     * word v>>5, bit v&31, LSB first, x-fastest (R#19) */
                    const uint32_t m = 1u << (o & 31);
                    uint32_t *wp = bits_out + (o >> 5);
                    if (post > tau) {
#ifdef _OPENMP
#pragma omp atomic
#endif
                        *wp |= m;
                    }
                }
            }
        }
    }
    (void)nthreads;
}

/* Sampled mode for grids too large to evaluate whole: for each listed voxel,
 * evaluate every view's Eq (1)-(9) terms directly from the frame and the
 * background model at the projected pixel, then Eq (3)-(4).  Same arithmetic
 * as oracle_slm_image + oracle_fuse, voxel by voxel. */
void oracle_fuse_sample(const oracle_rig *rig, const oracle_grid *g,
                        const uint8_t *const *frames, const float *const *mu,
                        const float *const *sigma, double sigma_floor, double p_vox,
                        int64_t nsample, const int64_t *vox, double *L_out, double *post_out,
                        int nthreads)
{
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t s = 0; s < nsample; ++s) {
        const int64_t v = vox[s];
        const int i = (int)(v % g->xlen);
        const int j = (int)((v / g->xlen) % g->ylen);
        const int k = (int)(v / ((int64_t)g->xlen * g->ylen));
        double s1 = 0.0, s0 = 0.0, h1, h0;
        oracle_view_likelihood(0.5, rig->p_occ, &h1, &h0);
        for (int c = 0; c < rig->ncam; ++c) {
            int px, py;
            if (oracle_project_pinned(rig->A + 12 * c, rig->W[c], rig->H[c], i, j, k, &px, &py)) {
                const int64_t p = (int64_t)py * rig->W[c] + px;
                double l1, l0;
                oracle_pixel(frames[c] + 3 * p, mu[c] + 3 * p, sigma[c] + 3 * p, sigma_floor,
                             rig->p_occ, NULL, &l1, &l0);
                s1 += l1;
                s0 += l0;
            } else {
                s1 += h1;
                s0 += h0;
            }
        }
        const double a1 = s1 + log(p_vox), a0 = s0 + log(1.0 - p_vox);
        L_out[s] = a1 - a0;
        if (post_out) post_out[s] = posterior_from_logs(a1, a0);
    }
    (void)nthreads;
}

/* Diagnostic (i): number of (voxel, camera) pairs, over slices [k0,k1), whose
 * (in-view, px, py) differ between the pinned FP32 and the exact double
 * projection. */
int64_t oracle_projection_flips(const oracle_rig *rig, const double *P, const oracle_grid *g,
                                int k0, int k1, int nthreads)
{
    int64_t flips = 0;
#ifdef _OPENMP
#pragma omp parallel for reduction(+ : flips) schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int k = k0; k < k1; ++k)
        for (int j = 0; j < g->ylen; ++j)
            for (int i = 0; i < g->xlen; ++i)
                for (int c = 0; c < rig->ncam; ++c) {
                    int a = -1, b = -1, x = -1, y = -1;
                    const int in1 = oracle_project_pinned(rig->A + 12 * c, rig->W[c], rig->H[c],
                                                          i, j, k, &a, &b);
                    const int in2 = oracle_project_exact(P + 12 * c, g->origin, g->spacing,
                                                         rig->W[c], rig->H[c], i, j, k, &x, &y);
                    if (in1 != in2 || (in1 && (a != x || b != y))) ++flips;
                }
    (void)nthreads;
    return flips;
}

void oracle_project_pinned_batch(const float A[12], int W, int H, int64_t n, const int32_t *ijk,
                                  int32_t *out /* n*3: inview, px, py */)
{
    for (int64_t s = 0; s < n; ++s) {
        int px = -1, py = -1;
        out[3 * s] = oracle_project_pinned(A, W, H, ijk[3 * s], ijk[3 * s + 1], ijk[3 * s + 2], &px, &py);
        out[3 * s + 1] = px;
        out[3 * s + 2] = py;
    }
}

/* ------------------------------------------------------------------------ */
/* NEXT-2: inner-voxel removal ("remove voxels inside human body and   */
/* get the surface voxels", "Remove inner voxel").           */
/* ------------------------------------------------------------------------ */

static int occupied(const uint32_t *bits, const oracle_grid *g, int i, int j, int k)
{
    /* outside the volume counts as unoccupied */
    if (i < 0 || j < 0 || k < 0 || i >= g->xlen || j >= g->ylen || k >= g->zlen) return 0;
    const int64_t v = (int64_t)i + (int64_t)g->xlen * (j + (int64_t)g->ylen * k);
    return (int)((bits[v >> 5] >> (v & 31)) & 1u);
}

/* Surface voxels of slices [k0,k1): occupied voxels with at least one
 * unoccupied 6-neighbour.  Writes their linear indices in increasing order
 * (up to `capacity`) and returns how many there are. */
int64_t oracle_surface(const uint32_t *bits, const oracle_grid *g, int k0, int k1,
                       int64_t *out, int64_t capacity)
{
    int64_t n = 0;
    for (int k = k0; k < k1; ++k)
        for (int j = 0; j < g->ylen; ++j)
            for (int i = 0; i < g->xlen; ++i) {
                if (!occupied(bits, g, i, j, k)) continue;
                const int inner = occupied(bits, g, i - 1, j, k) && occupied(bits, g, i + 1, j, k) &&
                                  occupied(bits, g, i, j - 1, k) && occupied(bits, g, i, j + 1, k) &&
                                  occupied(bits, g, i, j, k - 1) && occupied(bits, g, i, j, k + 1);
                if (inner) continue;
                if (n < capacity) out[n] = (int64_t)i + (int64_t)g->xlen * (j + (int64_t)g->ylen * k);
                ++n;
            }
    return n;
}

/* ------------------------------------------------------------------------ */
/* NEXT-1: probability filtering + thresholding, merged ("we filter the */
/* probability of voxels ... and then perform a thresholding process";        */
/* P:269-271): 3x3x3 box average of the posterior with zero */
/* padding outside the volume, then occupied := smoothed > tau.               */
/* ------------------------------------------------------------------------ */
void oracle_smooth_threshold(const double *post, const oracle_grid *g, double tau, double *smoothed,
                             uint32_t *bits_out)
{
    /* bits_out (if given) must be zeroed by the caller */
    for (int k = 0; k < g->zlen; ++k)
        for (int j = 0; j < g->ylen; ++j)
            for (int i = 0; i < g->xlen; ++i) {
                double acc = 0.0;
                for (int dk = -1; dk <= 1; ++dk)
                    for (int dj = -1; dj <= 1; ++dj)
                        for (int di = -1; di <= 1; ++di) {
                            const int a = i + di, b = j + dj, c = k + dk;
                            if (a < 0 || b < 0 || c < 0 || a >= g->xlen || b >= g->ylen || c >= g->zlen)
                                continue; /* zero padding */
                            acc += post[(int64_t)a + (int64_t)g->xlen * (b + (int64_t)g->ylen * c)];
                        }
                const double sm = acc / 27.0;
                const int64_t v = (int64_t)i + (int64_t)g->xlen * (j + (int64_t)g->ylen * k);
                if (smoothed) smoothed[v] = sm;
                if (bits_out && sm > tau) bits_out[v >> 5] |= 1u << (v & 31);
            }
}

/* ------------------------------------------------------------------------ */
/* NEXT-4: voxel colour ("the color rendering is also an iterative      */
/* process of all voxels", "Voxel color calculation",        */
/* P:303-307).  For each listed voxel: over the cameras whose      */
/* pinned nearest pixel is in view (R#10-R#12) and whose SLM there (Eq 1-2)    */
/* exceeds slm_gate (default 1/2; R#24), the arithmetic mean of the     */
/* 8-bit RGB at that pixel (R#23); no occlusion test.  count = number */
/* of qualifying views (0: colour unset, rgb = 0).  margin = the smallest      */
/* |SLM - slm_gate| over the in-view cameras (the parity band).               */
/* ------------------------------------------------------------------------ */
void oracle_color(const oracle_rig *rig, const oracle_grid *g, const uint8_t *const *frames,
                  const float *const *mu, const float *const *sigma, double sigma_floor,
                  double slm_gate, int64_t n, const int64_t *vox, double *rgb_out,
                  int32_t *count_out, double *margin_out)
{
    for (int64_t s = 0; s < n; ++s) {
        const int64_t v = vox[s];
        const int i = (int)(v % g->xlen);
        const int j = (int)((v / g->xlen) % g->ylen);
        const int k = (int)(v / ((int64_t)g->xlen * g->ylen));
        double sum[3] = {0.0, 0.0, 0.0}, margin = INFINITY;
        int32_t cnt = 0;
        for (int c = 0; c < rig->ncam; ++c) {
            int px, py;
            if (!oracle_project_pinned(rig->A + 12 * c, rig->W[c], rig->H[c], i, j, k, &px, &py))
                continue;
            const int64_t p = (int64_t)py * rig->W[c] + px;
            const uint8_t *I = frames[c] + 3 * p;
            double slm;
            oracle_pixel(I, mu[c] + 3 * p, sigma[c] + 3 * p, sigma_floor, rig->p_occ, &slm, NULL,
                         NULL);
            if (fabs(slm - slm_gate) < margin) margin = fabs(slm - slm_gate);
            if (slm > slm_gate) {
                for (int ch = 0; ch < 3; ++ch) sum[ch] += (double)I[ch];
                ++cnt;
            }
        }
        for (int ch = 0; ch < 3; ++ch) rgb_out[3 * s + ch] = cnt ? sum[ch] / cnt : 0.0;
        count_out[s] = cnt;
        if (margin_out) margin_out[s] = margin;
    }
}

/* ------------------------------------------------------------------------ */
/* NEXT-3: background-model training (the paper assumes mu, sigma   */
/* exist).  Per pixel and channel over n frames: the sample mean and    */
/* the population standard deviation, sigma clamped up to the floor   */
/* (R#6).  Two passes in double.                                       */
/* ------------------------------------------------------------------------ */
void oracle_train_background_elems(int n, int64_t nelem, const uint8_t *const *frames,
                                   double sigma_floor, double *mean_out, double *sigma_out)
{
    for (int64_t e = 0; e < nelem; ++e) {
        double sum = 0.0;
        for (int f = 0; f < n; ++f) sum += (double)frames[f][e];
        const double mean = sum / n;
        double ss = 0.0;
        for (int f = 0; f < n; ++f) {
            const double dv = (double)frames[f][e] - mean;
            ss += dv * dv;
        }
        double sd = sqrt(ss / n);
        if (sd < sigma_floor) sd = sigma_floor;
        mean_out[e] = mean;
        sigma_out[e] = sd;
    }
}

/* RGB frames: 3 elements per pixel. */
void oracle_train_background(int n, int64_t npx, const uint8_t *const *frames, double sigma_floor,
                             double *mean_out, double *sigma_out)
{
    oracle_train_background_elems(n, 3 * npx, frames, sigma_floor, mean_out, sigma_out);
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* NEXT-3 boundary variants (R#25-R#27).    */
/* ------------------------------------------------------------------------ */

/* Grayscale input (and any channel count nch): Eq (1)-(2) with the single
 * Gaussian of P:77 over nch independent 8-bit channels and the uniform
 * foreground density over the 8-bit cube of that dimension, U = 256^-nch
 * (S:134 fixes 256^-3 for RGB; grayscale is nch = 1, U = 256^-1, R#25), then
 * Eq (5)-(9) as oracle_pixel.  For nch = 3 this is oracle_pixel term for term
 * (tested bit for bit). */
void oracle_pixel_nch(int nch, const uint8_t *I, const float *mu, const float *sigma,
                      double sigma_floor, double p_occ,
                      double *slm_out, double *lnp1_out, double *lnp0_out)
{
    double ln_g = 0.0; /* ln P(I|F=0) = sum_ch ln N(I_ch | mu_ch, sigma'_ch) */
    for (int ch = 0; ch < nch; ++ch) {
        double s = (double)sigma[ch];
        if (s < sigma_floor) s = sigma_floor; /* sigma floor (R#6) */
        ln_g += ln_gauss((double)I[ch], (double)mu[ch], s);
    }
    const double ln_u = -(double)nch * log(256.0);   /* ln U, U = 256^-nch (R#25) */
    const double ln_fg = ln_u + log(0.5);             /* ln P(I|F=1)P(F=1) */
    const double ln_bg = ln_g + log(0.5);             /* ln P(I|F=0)P(F=0) */
    const double dd = ln_bg - ln_fg;
    const double slm = 1.0 / (1.0 + exp(dd));
    const double one_minus_slm = 1.0 / (1.0 + exp(-dd));
    const double p_o1 = p_occ, p_o0 = 1.0 - p_occ;
    const double p_s_v1 = p_o0 * slm /* Eq 8 */ + p_o1 * slm /* Eq 9 */;
    const double p_s_v0 = p_o0 * one_minus_slm /* Eq 6 */ + p_o1 * slm /* Eq 7 */;
    if (slm_out) *slm_out = slm;
    if (lnp1_out) *lnp1_out = log(p_s_v1);
    if (lnp0_out) *lnp0_out = log(p_s_v0);
}

void oracle_slm_image_nch(int nch, int64_t n, const uint8_t *img, const float *mu,
                          const float *sigma, double sigma_floor, double p_occ, double *slm,
                          double *lnp1, double *lnp0, int nthreads)
{
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t p = 0; p < n; ++p) {
        oracle_pixel_nch(nch, img + (int64_t)nch * p, mu + (int64_t)nch * p, sigma + (int64_t)nch * p,
                         sigma_floor, p_occ, slm ? slm + p : NULL, lnp1 ? lnp1 + p : NULL,
                         lnp0 ? lnp0 + p : NULL);
    }
    (void)nthreads;
}

/* The pinned projection's continuous coordinates: the float operations of
 * oracle_project_pinned, returning u = RN(x'/w), v = RN(y'/w) (the +1/2 of
 * round-half-up folded in, so u - 1/2 is the voxel centre's continuous pixel
 * x coordinate, pixel centres at integers, R#11) and the same in-view
 * decision (w > 0 and the nearest pixel inside the image, R#12, R#26). */
int oracle_project_pinned_uv(const float A[12], int W, int H, int i, int j, int k,
                             float *u_out, float *v_out)
{
    const float fi = (float)i, fj = (float)j, fk = (float)k;
    const float x = fmaf(A[2], fk, fmaf(A[1], fj, fmaf(A[0], fi, A[3])));
    const float y = fmaf(A[6], fk, fmaf(A[5], fj, fmaf(A[4], fi, A[7])));
    const float w = fmaf(A[10], fk, fmaf(A[9], fj, fmaf(A[8], fi, A[11])));
    if (!(w > 0.0f)) return 0;
    const float rr = 1.0f / w;
    const float u = x * rr;
    const float v = y * rr;
    if (!(u >= 0.0f && u < (float)W && v >= 0.0f && v < (float)H)) return 0;
    *u_out = u;
    *v_out = v;
    return 1;
}

static int clampi(int a, int lo, int hi) { return a < lo ? lo : (a > hi ? hi : a); }

/* Bilinear sample of a W x H double image at the continuous pixel position
 * (x, y) (pixel centres at integers): the four pixel centres around it,
 * x0 = floor(x), y0 = floor(y), weights (1-fx)(1-fy), fx(1-fy), (1-fx)fy, fx fy
 * with fx = x - x0, fy = y - y0; neighbour indices clamped to the image
 * ("bilinear SLM sampling at continuous projections, clamped at image
 * borders"; R#26). */
double oracle_bilinear(const double *img, int W, int H, double x, double y)
{
    const double x0 = floor(x), y0 = floor(y);
    const double fx = x - x0, fy = y - y0;
    const int xa = clampi((int)x0, 0, W - 1), xb = clampi((int)x0 + 1, 0, W - 1);
    const int ya = clampi((int)y0, 0, H - 1), yb = clampi((int)y0 + 1, 0, H - 1);
    const double s00 = img[(int64_t)ya * W + xa], s10 = img[(int64_t)ya * W + xb];
    const double s01 = img[(int64_t)yb * W + xa], s11 = img[(int64_t)yb * W + xb];
    return (1.0 - fx) * (1.0 - fy) * s00 + fx * (1.0 - fy) * s10 + (1.0 - fx) * fy * s01 +
           fx * fy * s11;
}

/* Eq (3)-(4) + threshold with the bilinear SLM sample of
 * every in-view camera (R#26): SLM_s = oracle_bilinear(SLM_c, u - 1/2,
 * v - 1/2), then the per-view likelihoods of Eq (5)-(9) of that value
 * (oracle_view_likelihood); out-of-view views contribute SLM = 1/2 (R#12).
 * slm: per camera W x H double SLM images (oracle_slm_image). */
void oracle_fuse_bilinear(const oracle_rig *rig, const oracle_grid *g, const double *const *slm,
                          double p_vox, double tau, int k0, int k1, double *L_out,
                          double *post_out, uint32_t *bits_out, int nthreads)
{
    const int64_t plane = (int64_t)g->xlen * g->ylen;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int k = k0; k < k1; ++k) {
        for (int j = 0; j < g->ylen; ++j) {
            for (int i = 0; i < g->xlen; ++i) {
                double s1 = 0.0, s0 = 0.0, h1, h0;
                oracle_view_likelihood(0.5, rig->p_occ, &h1, &h0);
                for (int c = 0; c < rig->ncam; ++c) {
                    float u, v;
                    if (oracle_project_pinned_uv(rig->A + 12 * c, rig->W[c], rig->H[c], i, j, k, &u, &v)) {
                        const double s = oracle_bilinear(slm[c], rig->W[c], rig->H[c],
                                                         (double)u - 0.5, (double)v - 0.5);
                        double l1, l0;
                        oracle_view_likelihood(s, rig->p_occ, &l1, &l0);
                        s1 += l1;
                        s0 += l0;
                    } else {
                        s1 += h1;
                        s0 += h0;
                    }
                }
                const double a1 = s1 + log(p_vox), a0 = s0 + log(1.0 - p_vox);
                const int64_t v = (int64_t)i + (int64_t)g->xlen * (j + (int64_t)g->ylen * k);
                const int64_t o = v - plane * k0;
                const double post = posterior_from_logs(a1, a0);
                if (L_out) L_out[o] = a1 - a0;
                if (post_out) post_out[o] = post;
                if (bits_out && post > tau) {
#ifdef _OPENMP
#pragma omp atomic
#endif
                    bits_out[o >> 5] |= 1u << (o & 31);
                }
            }
        }
    }
    (void)nthreads;
}
