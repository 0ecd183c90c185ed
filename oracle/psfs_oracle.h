/* psfs_oracle.h -- the CPU oracle's own declarations (TEST INFRASTRUCTURE ONLY).
 * Not shared with include/psfs.h or with the CUDA path. */
#ifndef PSFS_ORACLE_H
#define PSFS_ORACLE_H
#include <stdint.h>

typedef struct {
    double origin[3]; /* mm */
    double spacing;   /* mm */
    int xlen, ylen, zlen;
} oracle_grid;

typedef struct {
    int ncam;
    const float *A;  /* ncam*12 pre-composed matrices (oracle_precompose) */
    const int *W;    /* ncam */
    const int *H;    /* ncam */
    double p_occ;    /* P(O=1) */
} oracle_rig;

void oracle_pixel(const uint8_t I[3], const float mu[3], const float sigma[3], double sigma_floor,
                  double p_occ, double *slm, double *lnp1, double *lnp0);
void oracle_view_likelihood(double slm, double p_occ, double *lnp1, double *lnp0);
void oracle_slm_image(int W, int H, const uint8_t *img, const float *mu, const float *sigma,
                      double sigma_floor, double p_occ, double *slm, double *lnp1, double *lnp0,
                      int nthreads);
void oracle_precompose(const double P[12], const double origin[3], double spacing, float A[12]);
int oracle_project_pinned(const float A[12], int W, int H, int i, int j, int k, int *px, int *py);
int oracle_project_exact(const double P[12], const double origin[3], double spacing, int W, int H,
                         int i, int j, int k, int *px, int *py);
void oracle_fuse(const oracle_rig *rig, const oracle_grid *g, const double *const *lnp1,
                 const double *const *lnp0, double p_vox, double tau, int k0, int k1,
                 double *L_out, double *post_out, uint32_t *bits_out, int nthreads);
void oracle_fuse_sample(const oracle_rig *rig, const oracle_grid *g, const uint8_t *const *frames,
                        const float *const *mu, const float *const *sigma, double sigma_floor,
                        double p_vox, int64_t nsample, const int64_t *vox, double *L_out,
                        double *post_out, int nthreads);
int64_t oracle_projection_flips(const oracle_rig *rig, const double *P, const oracle_grid *g,
                                int k0, int k1, int nthreads);
void oracle_project_pinned_batch(const float A[12], int W, int H, int64_t n, const int32_t *ijk,
                                  int32_t *out);
int64_t oracle_surface(const uint32_t *bits, const oracle_grid *g, int k0, int k1, int64_t *out,
                       int64_t capacity);
void oracle_smooth_threshold(const double *post, const oracle_grid *g, double tau, double *smoothed,
                             uint32_t *bits_out);
void oracle_color(const oracle_rig *rig, const oracle_grid *g, const uint8_t *const *frames,
                  const float *const *mu, const float *const *sigma, double sigma_floor,
                  double slm_gate, int64_t n, const int64_t *vox, double *rgb_out,
                  int32_t *count_out, double *margin_out);
void oracle_train_background(int n, int64_t npx, const uint8_t *const *frames, double sigma_floor,
                             double *mean_out, double *sigma_out);
void oracle_train_background_elems(int n, int64_t nelem, const uint8_t *const *frames,
                                   double sigma_floor, double *mean_out, double *sigma_out);
/* NEXT-3 variants */
void oracle_pixel_nch(int nch, const uint8_t *I, const float *mu, const float *sigma,
                      double sigma_floor, double p_occ, double *slm, double *lnp1, double *lnp0);
void oracle_slm_image_nch(int nch, int64_t n, const uint8_t *img, const float *mu,
                          const float *sigma, double sigma_floor, double p_occ, double *slm,
                          double *lnp1, double *lnp0, int nthreads);
int oracle_project_pinned_uv(const float A[12], int W, int H, int i, int j, int k, float *u,
                             float *v);
double oracle_bilinear(const double *img, int W, int H, double x, double y);
void oracle_fuse_bilinear(const oracle_rig *rig, const oracle_grid *g, const double *const *slm,
                          double p_vox, double tau, int k0, int k1, double *L_out,
                          double *post_out, uint32_t *bits_out, int nthreads);
int oracle_max_threads(void);

#endif
