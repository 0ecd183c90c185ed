// psfs_next3.cu -- sm_100a kernels of the NEXT-3 boundary variants (SURVEY.md
// 8(f) rank 3; R#25-R#27):
//
//   k_s1x       stage 1 for grayscale input (one 8-bit channel, U = 256^-1, R#25)
//               and for bilinear sampling (the float SLM of Eq 1-2 instead of the
//               fused view term).  One thread per region-of-interest pixel, all F
//               frames of the pass; the background model record is read once per
//               pass.  Grayscale reuses the RGB arithmetic: channels 1 and 2 of a
//               grayscale model record hold mu = 0, sigma' = 1 and the kernel feeds
//               them I = 0, so they add exactly 0 to d.
//   k_voxel_bl  stage 2 with the bilinear SLM sample (clamped at image
//               borders, R#26): per voxel and camera the pinned projection's
//               (u, v), the four pixel centres around (u - 1/2, v - 1/2), the
//               interpolated SLM, the per-view term of Eq 5-9 of that value
//               rounded to Q11.20 and summed exactly in int32 (Eq 3-4), threshold
//                and warp-ballot bit words.
//
// Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n, R#n = DESIGN.md
// reading n.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "psfs_internal.h"
#include "psfs_device.cuh"

namespace psfs {

// SLM = 1 / (1 + e^d), d = D 2^-20 (Eq 1-2).  E = e^-|d| = 2^y with
// y = -|d| log2(e) split in double as n + r (|r| <= 1/2), 2^r from the MUFU ex2
// (relative error ~2^-22) and 2^n by exponent construction (0 below 2^-126);
// SLM = E / (1 + E) for d >= 0, 1 / (1 + E) otherwise.  Relative error of the
// float SLM <= ~4e-7.
__device__ __forceinline__ float slm_from_D(double D)
{
    const double y = -fabs(D) * (1.4426950408889634 / kQ);
    const double n = rint(y);
    const float r = (float)(y - n);
    const int ni = (int)n;
    const float E = ni < -126 ? 0.0f : ex2_approx(r) * __int_as_float((ni + 127) << 23);
    const float inv = __frcp_rn(1.0f + E);
    return D >= 0.0 ? E * inv : inv;
}

// D = 2^20 d of pixel_term (psfs_device.cuh), without the Eq 5-9 fold.
__device__ __forceinline__ double pixel_D(const PixelModel &m, uint32_t r, uint32_t gr, uint32_t b)
{
    double D = m.H;
    D = fma(-fma(m.cf[0], u8_to_double(r), m.g[0]), u8_to_double(r), D);
    D = fma(-fma(m.cf[1], u8_to_double(gr), m.g[1]), u8_to_double(gr), D);
    D = fma(-fma(m.cf[2], u8_to_double(b), m.g[2]), u8_to_double(b), D);
    return D;
}

template <int F>
__device__ __forceinline__ void store_words(int32_t *dst, const int32_t (&q)[F])
{
    if constexpr (F >= 4) {
#pragma unroll
        for (int k = 0; k < F / 4; ++k)
            reinterpret_cast<int4 *>(dst)[k] = make_int4(q[4 * k], q[4 * k + 1], q[4 * k + 2], q[4 * k + 3]);
    } else if constexpr (F == 2) {
        *reinterpret_cast<int2 *>(dst) = make_int2(q[0], q[1]);
    } else {
        *dst = q[0];
    }
}

// Stage 1 of the NEXT-3 variants.  NCH: bytes per pixel of the frames (1 or 3);
// SLM: store the float SLM (bilinear sampling) instead of the Q11.20 term.
// Output record of pixel (row, col): p.terms + (toff + row tstride + col) tf + f.
template <int F, int NCH, bool SLM>
__global__ void __launch_bounds__(256) k_s1x(const __grid_constant__ S1Params p)
{
    const int c = blockIdx.y;
    const int r0 = p.cam[c].r0, c0 = p.cam[c].c0;
    const int ncol = p.cam[c].c1 - c0;
    const int npx = ncol * (p.cam[c].r1 - r0);
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= npx) return;
    const int rr = q / ncol, cc = q - rr * ncol;
    const int64_t pix = (int64_t)(r0 + rr) * p.cam[c].W + c0 + cc;
    const int64_t gt = p.cam[c].toff + (int64_t)(r0 + rr) * p.cam[c].tstride + c0 + cc;
    const ModelPx *mp = p.model + p.cam[c].off + pix;
    const float4 ma = __ldg(reinterpret_cast<const float4 *>(mp));
    const float4 mb = __ldg(reinterpret_cast<const float4 *>(mp) + 1);
    uint32_t b[F][3];
#pragma unroll
    for (int f = 0; f < F; ++f) {
        const uint8_t *src = p.frames[f][c] + pix * NCH;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) b[f][ch] = ch < NCH ? (uint32_t)__ldg(src + ch) : 0u;
    }
    const float mu[3] = {ma.x, ma.y, ma.z};
    const float sg[3] = {ma.w, mb.x, mb.y};
    const double K = __hiloint2double(__float_as_int(mb.w), __float_as_int(mb.z));
    const PixelModel m = pixel_model(mu, sg, K);
    int32_t out[F];
    if constexpr (SLM) {
#pragma unroll
        for (int f = 0; f < F; ++f) out[f] = __float_as_int(slm_from_D(pixel_D(m, b[f][0], b[f][1], b[f][2])));
    } else {
        const double dlo = (p.ln_1mpo - p.ln_po) * kQ;
        const double lnpo = p.ln_po * kQ;
#pragma unroll
        for (int f = 0; f < F; ++f) out[f] = pixel_term(m, b[f][0], b[f][1], b[f][2], dlo, lnpo);
    }
    store_words<F>(p.terms + gt * p.tf, out);
}

template <int F, int NCH, bool SLM>
static cudaError_t launch_s1x_t(const S1Params &p, int max_px, cudaStream_t s)
{
    dim3 grid((max_px + 255) / 256, p.ncam);
    k_s1x<F, NCH, SLM><<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

template <int NCH, bool SLM>
static cudaError_t launch_s1x_f(const S1Params &p, int F, int max_px, cudaStream_t s)
{
    switch (F) {
    case 1: return launch_s1x_t<1, NCH, SLM>(p, max_px, s);
    case 2: return launch_s1x_t<2, NCH, SLM>(p, max_px, s);
    case 4: return launch_s1x_t<4, NCH, SLM>(p, max_px, s);
    case 8: return launch_s1x_t<8, NCH, SLM>(p, max_px, s);
    case 16: return launch_s1x_t<16, NCH, SLM>(p, max_px, s);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_s1x(const S1Params &p_in, int F, int nch, bool slm, int max_px, cudaStream_t s)
{
    if (max_px <= 0) return cudaSuccess;
    S1Params p = p_in;
    p.tf = F;
    p.halves = 1;
    if (nch == 1) return slm ? launch_s1x_f<1, true>(p, F, max_px, s) : launch_s1x_f<1, false>(p, F, max_px, s);
    if (nch == 3) return slm ? launch_s1x_f<3, true>(p, F, max_px, s) : launch_s1x_f<3, false>(p, F, max_px, s);
    return cudaErrorInvalidValue;
}

// One pixel's F-frame SLM record (F * 4 bytes, F * 4-byte aligned) as vector loads.
template <int F>
__device__ __forceinline__ void load_rec(const float *src, float (&v)[F])
{
    if constexpr (F == 8) {
        uint32_t w[8];
        asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
                       "=r"(w[7])
                     : "l"(src));
#pragma unroll
        for (int f = 0; f < 8; ++f) v[f] = __uint_as_float(w[f]);
    } else if constexpr (F == 4) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(src));
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else if constexpr (F == 2) {
        const float2 a = __ldg(reinterpret_cast<const float2 *>(src));
        v[0] = a.x; v[1] = a.y;
    } else {
        v[0] = __ldg(src);
    }
}

// Stage 2 with bilinear SLM sampling.  A warp is 32 consecutive voxels of the
// slab (x-fastest), i.e. one bitmask word: slabs start on word boundaries
// (psfs_create), so lane 0 stores the ballot word.  Per camera: the pinned
// projection of the voxel centre (the +1/2 of round-half-up folded into A_c);
// out of view (R#12) adds 0; else x = u - 1/2, y = v - 1/2 (exact in float for
// u >= 1/2; below, x0 = -1 and both neighbours clamp to column 0, so fx is
// irrelevant), x0 = floor(x), fx = x - x0 (exact), neighbours clamped to the
// image; per frame the SLM sample (three weighted pairs), t = ln s - ln((1 - p_O) +
// (2 p_O - 1) s) (Eq 5-9) as log2 differences (MUFU lg2), q = rint(t 2^20).
template <int F>
__global__ void __launch_bounds__(256) k_voxel_bl(const __grid_constant__ VParams p)
{
    const int64_t plane = (int64_t)p.xlen * p.ylen;
    const int64_t nslab = plane * (p.k1 - p.k0);
    const int64_t nitems = (nslab + 31) / 32;
    const int lane = threadIdx.x & 31;
    const float *T = reinterpret_cast<const float *>(p.terms);
    constexpr float kLn2Q = 0.6931471805599453f * 1048576.0f;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t wi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nitems; wi += wstride) {
        const int64_t o = wi * 32 + lane;  // slab-relative voxel
        const bool valid = o < nslab;
        const int64_t v = o + plane * p.k0;
        const int i = (int)(v % p.xlen);
        const int64_t rest = v / p.xlen;
        const int j = (int)(rest % p.ylen);
        const int k = (int)(rest / p.ylen);
        const float fi = (float)i, fj = (float)j, fk = (float)k;
        int32_t S[F];
#pragma unroll
        for (int f = 0; f < F; ++f) S[f] = 0;
        for (int c = 0; valid && c < p.ncam; ++c) {
            const float *A = p.cam[c].A;
            const float x = __fmaf_rn(A[2], fk, __fmaf_rn(A[1], fj, __fmaf_rn(A[0], fi, A[3])));
            const float y = __fmaf_rn(A[6], fk, __fmaf_rn(A[5], fj, __fmaf_rn(A[4], fi, A[7])));
            const float w = __fmaf_rn(A[10], fk, __fmaf_rn(A[9], fj, __fmaf_rn(A[8], fi, A[11])));
            const float rr = p.fast_rcp ? rcp_rn_fast(w) : __frcp_rn(w);
            const float u = __fmul_rn(x, rr), vv = __fmul_rn(y, rr);
            const int W = p.cam[c].W, H = p.cam[c].H;
            if (!(w > 0.0f && u >= 0.0f && u < (float)W && vv >= 0.0f && vv < (float)H)) continue;
            const float xs = __fsub_rn(u, 0.5f), ys = __fsub_rn(vv, 0.5f);
            const float x0f = floorf(xs), y0f = floorf(ys);
            const float fx = __fsub_rn(xs, x0f), fy = __fsub_rn(ys, y0f);
            const int x0 = (int)x0f, y0 = (int)y0f;
            const int xa = max(x0, 0), xb = min(x0 + 1, W - 1);
            const int ya = max(y0, 0), yb = min(y0 + 1, H - 1);
            const int64_t ra = (int64_t)p.cam[c].toff + (int64_t)ya * p.cam[c].Wp;
            const int64_t rb = (int64_t)p.cam[c].toff + (int64_t)yb * p.cam[c].Wp;
            float s00[F], s10[F], s01[F], s11[F];
            load_rec<F>(T + (ra + xa) * F, s00);
            load_rec<F>(T + (ra + xb) * F, s10);
            load_rec<F>(T + (rb + xa) * F, s01);
            load_rec<F>(T + (rb + xb) * F, s11);
            // weight form (1 - fx) a + fx b: every product and sum is of non-negative
            // values, so the sample keeps a few ulps of relative precision (the lerp
            // a + fx (b - a) loses it where SLM jumps from ~1 to ~1e-4 and the sample
            // is small: ~3e-5 in t, measured)
            const float wx = 1.0f - fx, wy = 1.0f - fy;
#pragma unroll
            for (int f = 0; f < F; ++f) {
                const float a0 = __fmaf_rn(fx, s10[f], __fmul_rn(wx, s00[f]));
                const float a1 = __fmaf_rn(fx, s11[f], __fmul_rn(wx, s01[f]));
                const float s = __fmaf_rn(fy, a1, __fmul_rn(wy, a0));
                const float l = lg2_approx(s) - lg2_approx(__fmaf_rn(p.bl_b, s, p.bl_a));
                S[f] += __float2int_rn(l * kLn2Q);
            }
        }
        const int64_t word = (plane * p.k0 + wi * 32) >> 5;
#pragma unroll
        for (int f = 0; f < F; ++f) {
            const unsigned m = __ballot_sync(0xffffffffu, valid && S[f] > p.Tq);
            if (p.lo_base && valid)
                p.lo_base[f * p.lo_stride + o] = p.lo_raw ? __int_as_float(S[f]) : logodds_of(S[f], p.logit_pv);
            if (lane == 0) {
                if (p.npeer == 0) {
                    if (p.bits_base) p.bits_base[f * p.bits_stride + word] = m;
                } else {
                    for (int r = 0; r < p.npeer; ++r) peer_store_word(&p.peer[r][f * p.peer_fstride + word], m, p.peer_mc);
                }
            }
        }
    }
}

cudaError_t launch_voxel_bl(const VParams &p, int F, cudaStream_t s)
{
    const int64_t nslab = (int64_t)p.xlen * p.ylen * (p.k1 - p.k0);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((nslab + 255) / 256, 148 * 8));
    switch (F) {
    case 1: k_voxel_bl<1><<<blocks, 256, 0, s>>>(p); break;
    case 2: k_voxel_bl<2><<<blocks, 256, 0, s>>>(p); break;
    case 4: k_voxel_bl<4><<<blocks, 256, 0, s>>>(p); break;
    case 8: k_voxel_bl<8><<<blocks, 256, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace psfs
