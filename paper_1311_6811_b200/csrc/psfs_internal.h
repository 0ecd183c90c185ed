// psfs_internal.h -- shared between the host runtime (psfs_api.cu) and the
// sm_100a kernels (psfs_kernels.cu).  Not part of the public ABI (include/psfs.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace psfs {

constexpr int kMaxCam = 64;  // == PSFS_MAX_CAMERAS
constexpr int kMaxF = 16;    // == PSFS_MAX_BATCH
constexpr int kQBits = 20;   // Q11.20 fixed point for the per-view term t
constexpr int kMaxPeers = 8; // == PSFS_MAX_PEERS

// Background model of one pixel as stored on the device (set once by
// psfs_set_background; K filled by k_prep_model): 32 bytes, so a row segment of
// the model is one contiguous block (one bulk copy) and a warp's 32 records are
// 1 KB of coalesced loads.
struct ModelPx {
    float mu[3];  // mean per channel
    float sg[3];  // sigma' = max(sigma, sigma_floor) per channel (R#6)
    double K;     // 24 ln 2 - 1.5 ln(2 pi) - ln(sg0 sg1 sg2)
};
static_assert(sizeof(ModelPx) == 32, "ModelPx must be 32 bytes");

// Stage 1 (per-pixel term) launch description.
struct S1Cam {
    int32_t W, H;
    int32_t r0, r1, c0, c1;  // region of interest, half-open (c0, c1 multiples of 16 on the TMA path)
    int64_t off;             // first pixel of this camera in the concatenated pixel space (model)
    int64_t toff;            // first pixel of this camera's term image
    int32_t tstride;         // term image row stride in pixels (W + 1: padded, or W for debug)
    int32_t seg_begin;       // TMA path: first segment index of this camera
    int32_t segs_per_row;    // TMA path: ceil((c1 - c0) / kSeg)
    int32_t q_begin;         // pipelined path: first ROI pixel index of this camera
    int32_t ch_begin;        // async path: first 32-pixel row chunk of this camera
    int32_t ch_per_row;      // async path: ceil((c1 - c0) / 32)
    int32_t pad_[3];
};

constexpr int kSeg = 512;  // pixels per TMA segment (one row chunk) = consumer threads per block

struct S1Params {
    S1Cam cam[kMaxCam];
    const uint8_t *frames[kMaxF][kMaxCam];  // [f][c] device pointers, H*W*3 RGB
    const struct ModelPx *model;            // total_px records (AoS, 32 B each)
    int32_t *terms;                         // (toff + p) * tf + f, 32-B aligned
    int64_t total_px;
    double ln_po;    // ln p_O
    double ln_1mpo;  // ln (1 - p_O)
    double c0;       // -1.5 ln(2 pi) - ln U = 24 ln 2 - 1.5 ln(2 pi)
    int32_t ncam;
    int32_t nseg;    // TMA path: total segments over all cameras
    int32_t nq;      // pipelined path: total ROI pixels over all cameras
    int32_t nchunk;  // async path: 32-pixel row chunks over all cameras
    int32_t tf;      // frames per term record (the pass's F: 1..16)
    int32_t halves;  // 2: a 16-frame pass run as two 8-frame halves (path 0/4 only)
    int32_t n4;      // path 6: 4-pixel groups over all cameras (cam[c].pad_[0] = camera c's first)
    int32_t n2;      // path 6 with 2-pixel threads: 2-pixel groups (cam[c].pad_[1] = camera c's first)
    // per-row spans (nullable): row entry i = (camera | row << 8, first column),
    // span_pre[i] = 4-pixel groups before entry i, span_chunk[k] = the entry of
    // group 256 k; when set, n4 counts the spans' groups
    const int32_t *span_info, *span_pre, *span_chunk;
    int32_t span_rows;
    int64_t fstride;  // > 0: frames[f][c] == frames[0][c] + f * fstride for every f, c (path 6 addresses by arithmetic)
};

// Stage 2 (voxel) launch description.
// Term images are stored padded to (W+1) x (H+1) pixels: the extra column W and
// row H are all-zero terms (t = 0, the out-of-view contribution, R#12), so an
// out-of-view projection is clamped into the pad instead of branched on.
struct VCam {
    float A[12];    // pre-composed pinned projection matrix, row-major 3x4
    int32_t W, H;
    uint32_t toff;  // first pixel of this camera's padded term image (< 2^28)
    uint32_t Wp;    // padded row stride W + 1
};

struct VParams {
    VCam cam[kMaxCam];
    const int32_t *terms;
    uint32_t *bits[kMaxF];   // full-grid word arrays (nullable)
    float *logodds[kMaxF];   // slab arrays (nullable)
    int32_t xlen, ylen, k0, k1;
    int32_t ncam;
    int32_t Tq;              // occupied iff S > Tq
    int32_t byte_aligned;    // xlen % 8 == 0: each warp row is one whole byte
    int32_t fast_rcp;        // every w over the grid is <= 0 or in [2^-60, 2^60]
    double logit_pv;
    unsigned long long *tile_counter;  // persistent scheduling: monotone per handle
    long long tile_base;               // counter value at this launch's start
    int32_t ntiles;
    int32_t ty;                        // y sub-tiles per warp (1 or 4): tile = 32 x 8ty columns
    int32_t kz;                        // z-slices per tile
    int32_t max_blocks_per_sm;         // 0: fill the SMs (occupancy); > 0: cap (overlap)
    int32_t carve;                     // bits-only early exit (no log-odds output)
    int32_t q_max;                     // largest possible term: rint(-ln p_O 2^20)
    // fused z-slab exchange: npeer > 0 stores every bitmask byte into each rank's
    // buffer, frame f of this group at peer[r] + f * peer_fstride (bits[] unused)
    int32_t npeer;
    uint32_t *peer[kMaxPeers];
    int64_t peer_fstride;
    // the same outputs as base + frame * stride (a lane-dependent frame index
    // into bits[] / logodds[] would put those arrays in local memory)
    uint32_t *bits_base;       // bits[0] (nullable)
    int64_t bits_stride;       // words per frame
    float *lo_base;            // logodds[0] (nullable)
    int64_t lo_stride;         // floats per frame
    int32_t word_rows;         // xlen % 32 == 0: a 32-wide tile row is one bitmask word
    float bl_a, bl_b;          // bilinear sampling (k_voxel_bl): 1 - p_O, 2 p_O - 1
    int32_t lo_pairs;          // k_voxel16: x-adjacent log-odds as 8-byte stores (xlen, lo_stride even, 8-B base)
    int32_t lo_raw;            // lo_base receives the int32 sums S instead of float log-odds (NEXT-1)
    int32_t peer_mc;           // peer[0] is a multicast (NVLS) mapping: multimem stores / reductions
};

// ---- coarse passes (bits-only calls) -------------------
// Stage 1 stores, per pixel and frame, an 8-bit code c + bias of the Q11.20 term
// q with c 2^sh <= q <= c 2^sh + wc (c from an FP32 evaluation of t, widened by
// its error bound); the 32 frames of a pass share one 32-byte record.  Stage 2
// sums codes, decides every voxel-frame whose bounds lie on one side of T_q, and
// recomputes the rest exactly (the same per-pixel arithmetic as k_likelihood).
constexpr int kMaxFC = 64;       // frames per coarse pass (one byte each per record)
constexpr int kMaxFramePtrs = 2048;  // frames x cameras of one coarse pass (kernel-parameter table)

struct S1CParams {
    S1Cam cam[kMaxCam];                      // ROI, model / code offsets (tstride = row stride)
    const uint8_t *frames[kMaxFramePtrs];  // [f * ncam + c], f < nf
    const struct ModelPx *model;
    uint8_t *codes;      // (toff + p) * rec + f
    int32_t rec;         // bytes per code record: 32 (passes of <= 32 frames), 64 (<= 64), 1 (debug, nf = 1)
    int32_t ncam, nf;    // frames in this pass (1..32)
    int32_t quarters;    // ceil(nf / 8): 8-frame parts in adjacent blocks
    int32_t x4;          // 4 pixels per thread (W % 4, ROI columns % 4, frames 4-byte aligned)
    int32_t persistent;  // x4: persistent blocks, all quarters per thread (k_likelihood_c8p)
    int32_t n4;          // x4: 4-pixel groups over all cameras (cam[c].pad_[0] = camera c's first)
    double lr;           // ln(1 - p_O) - ln p_O
    float s;             // 2^(20 - sh)
    float zoff;          // (-ln p_O - eps) s + bias
    const int32_t *span_info, *span_pre, *span_chunk;  // per-row spans (as S1Params), nullable
    int32_t span_rows;
    int64_t fstride;     // > 0: frames[f * ncam + c] == frames[c] + f * fstride for every f, c (address arithmetic
                         // instead of a pointer-table load per frame); 0: use the table
};

struct VCCam {
    float A[12];    // pinned matrix (as VCam)
    int32_t W, H;
    uint32_t toff;  // padded code image offset (pixels)
    uint32_t Wp;    // W + 1
    int64_t off;    // model record offset (fix-up)
};

struct VCParams {
    VCCam cam[kMaxCam];
    const uint8_t *frames[kMaxFramePtrs];  // [f * ncam + c]; fix-up: the exact terms are recomputed
    const struct ModelPx *model;
    const uint8_t *codes;     // 32- or 64-byte records (rec)
    int32_t rec;
    uint32_t K0, K1;          // packed 16-bit thresholds: field >= K1 -> bit 1; K0 <= field < K1 -> exact
    int32_t Tq;
    int32_t ncam, nf;
    int32_t xlen, ylen, k0, k1;
    int32_t fast_rcp;
    double dlo, lnpo;         // exact path constants (k_likelihood): (ln(1-p_O) - ln p_O) 2^20, ln p_O 2^20
    unsigned long long *tile_counter;
    long long tile_base;
    int32_t ntiles, kz;
    // k_voxel_c8w: tiles [0, nbig) are kz deep over slices [k0, kzb); the rest are
    // one slice deep over [kzb, k1) (a finer tail for the persistent grid's last wave)
    int32_t nbig, kzb;
    uint32_t *bits_base;      // frame f at bits_base + f * bits_stride (nullable when npeer > 0)
    int64_t bits_stride;
    int32_t npeer;
    uint32_t *peer[kMaxPeers];
    int64_t peer_fstride;
    unsigned long long *fix_count;  // nullable: voxel-frames resolved exactly
    // undecided voxel-frames: (v << 6 | frame) appended at fix_list[*fix_head], then
    // k_fixup_c8 sums them exactly and patches the bits; beyond fix_cap the lane
    // resolves them in place (slow, correct)
    unsigned long long *fix_list;
    unsigned long long *fix_head;  // [0] entries, [1] k_fixup_c8 blocks done (reset by its last block)
    uint64_t fix_cap;
    int32_t peer_mc;          // peer[0] is a multicast (NVLS) mapping: multimem stores / reductions
    // tail-drained fix-up (non-null tile_flag): entries are stored + 1 (0 = not yet
    // written); a voxel block publishes tile_flag[tile] = pass_id once the tile's
    // words are flushed and counts itself in fix_head[3] when it has no tiles left;
    // k_fixup_c8 then needs no grid-wide wait: it claims entries (fix_head[2]) as
    // the voxel grid's last tiles run, waits only for the entry's own tile, and
    // zeroes the slots it consumed
    uint32_t *tile_flag;
    uint32_t pass_id;
    int32_t vox_blocks;       // blocks of the voxel launch (producers)
    int32_t ntx, nty;         // tile grid (the fix-up maps a voxel to its tile)
    int32_t max_blocks_per_sm; // 0: fill the SMs (occupancy); > 0: cap (room for a concurrent stage 1)
};

cudaError_t launch_likelihood_coarse(const S1CParams &p, int max_roi_px, cudaStream_t s);

// Pad records of the padded term / code images.  A buffer's record size changes
// with the pass (terms: 4F bytes, F = 1..16; codes: 32 or 64 bytes), and the pad
// records of one size overlap pixel records of another, so the host runtime
// rewrites them (k_fill_pads) whenever a buffer is about to be used with a
// record size other than its last one.
struct PadParams {
    uint32_t *buf;
    uint32_t toff[kMaxCam];          // first padded pixel of camera c
    int32_t W[kMaxCam], H[kMaxCam];
    int32_t first[kMaxCam + 1];      // pad pixels of camera c: [first[c], first[c+1]), W + H + 1 each
    int32_t ncam;
    int32_t rec_words;               // 32-bit words per record
    uint32_t fill;                   // 0 (terms) or bias * 0x01010101 (codes)
};
cudaError_t launch_fill_pads(const PadParams &p, cudaStream_t s);

// psfs_reconstruct_host upload through mapped pinned memory: warps copy the ROI
// rows of every (frame, camera) image of a group from host to the staging buffer.
struct H2DParams {
    const uint8_t *src[kMaxFramePtrs];    // [j * ncam + c]: device-usable addresses of the host images
    int32_t fidx[kMaxFC];                 // staging frame slot of compacted frame j
    uint8_t *dst;                         // staging: frame slot f, camera c at dst + f * img_bytes + off[c] * 3
    int64_t img_bytes;
    int64_t off[kMaxCam];
    int32_t W[kMaxCam], r0[kMaxCam], c0[kMaxCam], ncol[kMaxCam];
    int32_t task_begin[kMaxCam + 1];      // row tasks of camera c in one frame: [task_begin[c], task_begin[c+1])
    int32_t nf, ncam;
    int32_t bpp;      // bytes per pixel (3 RGB, 1 grayscale)
    // per-row spans (nullable): one task per (frame, row entry) uploading the
    // span's columns [cs, cs + 4 groups) instead of the rectangle's row
    const int32_t *span_info, *span_pre;
    int32_t span_rows;
    int32_t aligned;  // 16: every image and staging image 16-byte aligned with a whole number of
                      // 16-byte chunks (chunked copy); 4: every row segment 4-byte aligned; 1: bytes
};
cudaError_t launch_h2d_rows(const H2DParams &p, int nsm, cudaStream_t s);
cudaError_t launch_voxel_coarse(const VCParams &p, cudaStream_t s, int *nblocks);
cudaError_t launch_fixup_coarse(const VCParams &p, cudaStream_t s);

// NEXT-4 voxel colour (psfs_color): per camera the pinned matrix, the image and
// the model records of its pixels.
struct ColorCam {
    float A[12];
    int32_t W, H;
    int64_t off;              // first model record of this camera
    const uint8_t *frame;     // H*W*3 RGB (device)
};

struct ColorParams {
    ColorCam cam[kMaxCam];
    const struct ModelPx *model;
    const int64_t *indices;   // linear voxel indices (device)
    const int64_t *count;     // device: number of valid indices (min with capacity)
    int64_t capacity;
    float *rgb;               // n x 3 (device)
    int32_t *nviews;          // n (device, nullable)
    double d_gate;            // a view qualifies iff d < d_gate (SLM > gate)
    int32_t ncam, xlen, ylen, zlen;
};

// Device-side barrier of a fused exchange: flags[r] = rank r's flag array
// (kMaxPeers uint64 slots, mapped in this process); this rank writes `epoch`
// into slot `rank` of every rank's array, then waits for all `world` slots of
// its own array to reach `epoch` (err = 1 after a ~10 s timeout).
struct PeerBarrier {
    unsigned long long *flags[kMaxPeers];
    int32_t rank, world;
    unsigned long long epoch;
    int *err;
};

// Launchers (psfs_kernels.cu).  Return the cudaError_t of the launch.
cudaError_t launch_likelihood(const S1Params &p, int F, int max_roi_px, int path, cudaStream_t s);
// NEXT-3 (psfs_next3.cu): stage 1 for nch-byte pixels (1 grayscale, 3 RGB), storing
// the Q11.20 term (slm = false) or the float SLM (slm = true, bilinear sampling);
// F in {1, 2, 4, 8, 16}.  Stage 2 with bilinear SLM samples, F in {1, 2, 4, 8}.
cudaError_t launch_s1x(const S1Params &p, int F, int nch, bool slm, int max_roi_px, cudaStream_t s);
cudaError_t launch_voxel_bl(const VParams &p, int F, cudaStream_t s);
cudaError_t launch_prep_model(ModelPx *model, int64_t begin, int64_t n, double c0, cudaStream_t s);
// NEXT-3 background training (psfs_train_background): up to kMaxTrain frame
// pointers travel in the kernel parameters (no device table, no sync).
constexpr int kMaxTrain = 512;  // == PSFS_MAX_TRAIN_FRAMES
struct TrainParams {
    const uint8_t *frames[kMaxTrain];
    int32_t n;
    int64_t nelem;     // 3 * W * H
    float floor_f;
    int32_t nch;       // channels per pixel (3 RGB, 1 grayscale)
    float *mean, *sigma;
    ModelPx *model;    // non-null: install (mu, sigma') into these records
};
cudaError_t launch_train(const TrainParams &p, cudaStream_t s);
cudaError_t launch_voxel(const VParams &p, int F, cudaStream_t s, int *nblocks);
// NEXT-1 from the exact int32 sums (k_box_sums): posterior P = 1 / (1 + e^-L),
// L = S 2^-20 + logit p_V, 3x3x3 zero-padded box average, occupied := > tau.
// sums: nf frames of the slab [k0, k1) (frame stride nslab); halo_lo / halo_hi:
// slices k0 - 1 / k1 of the neighbouring slabs (frame stride xlen * ylen), NULL
// at the volume's own boundary (zero padding); outputs per frame: smoothed
// (slab, nullable), bits (full-grid words, slab words written, nullable).
struct BoxSumsParams {
    const int32_t *sums;
    const int32_t *halo_lo, *halo_hi;
    float *smoothed;
    uint32_t *bits;
    int64_t sums_stride, halo_stride, smoothed_stride, bits_stride;
    int32_t xlen, ylen, zlen, k0, k1, nf;
    double logit_pv;
    float tau;
};
cudaError_t launch_box_sums(const BoxSumsParams &p, cudaStream_t s);
// Fill words [w0, w1) of nf frames (frame stride fstride) through a multicast
// (NVLS) mapping: every replica receives the value (multimem.st).
cudaError_t launch_mc_fill(uint32_t *mc, int64_t fstride, int64_t w0, int64_t w1, int nf, uint32_t value,
                           cudaStream_t s);
int voxel_tiles(int xlen, int ylen, int k0, int k1, int ty, int kz);
#ifndef PSFS_EXP_BOXZ
#define PSFS_EXP_BOXZ 0  // 1: k_box_sums_z (z-streaming planes) instead of the in-memory halo box
#endif
#ifndef PSFS_EXP_BOXSZ
// output slices per k_box_sums block (in-memory halo box (32+2) x (8+2) x (BOXSZ+2): <= 10, one thread
// per right-edge element; k_box_sums_z: any depth)
#define PSFS_EXP_BOXSZ 8
#endif
// coarse stage-2 tiles: 32 x rows x kz, rows = coarse_tile_rows(rec) (the wide
// kernel's warps per block for 64-byte records, 8 otherwise)
#ifndef PSFS_EXP_C8W_NW
#define PSFS_EXP_C8W_NW 8  // warps per k_voxel_c8w block (4 or 8)
#endif
int coarse_tile_rows(int rec);
int coarse_voxel_tiles(int xlen, int ylen, int k0, int k1, int kz, int rec);
cudaError_t launch_surface(const uint32_t *bits, uint32_t *surf, int64_t *idx, int64_t capacity,
                           int64_t *count, long long *block_scratch, int xlen, int ylen, int zlen,
                           int k0, int k1, cudaStream_t s, int *launches);
int surface_blocks(int xlen, int ylen, int k0, int k1);
cudaError_t launch_smooth(const float *logodds, float *P, float *smoothed, uint32_t *bits, int xlen,
                          int ylen, int zlen, float tau, cudaStream_t s);
cudaError_t launch_peer_barrier(const PeerBarrier &b, cudaStream_t s);
cudaError_t launch_color(const ColorParams &p, cudaStream_t s);
cudaError_t launch_gather_probe(const void *tab, uint32_t lines_mask, int blocks, int iters, int G, int *out,
                                cudaStream_t s);
cudaError_t launch_l1_probe(const void *buf, int blocks, int iters, int *out, cudaStream_t s);
cudaError_t launch_rcp_check(uint32_t lo_bits, uint32_t hi_bits, unsigned long long *bad,
                             cudaStream_t s);

}  // namespace psfs
