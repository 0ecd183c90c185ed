/*
 * psfs.h -- C ABI of the B200-native probabilistic shape-from-silhouette (PSFS)
 * hot path of arXiv 1311.6811 ("Digitize Your Body and Action in 3-D at Over
 * 10 FPS"), section 2.2.2.
 *
 * Citation keys: P:n = PAPER.md line n; S:n = SPEC.md line n; R#n = reading n
 * in DESIGN.md ("Readings of the paper").
 *
 * What the library computes ("given a set of images ... calculate the
 * silhouette likelihood maps ... estimate the posterior probability
 * representing occupancy of each voxel"):
 *
 *   stage 1, per pixel p of camera r (Eq 1-2, and Eq 5-9):
 *     d   = sum_ch ln N(I_ch | mu_ch, sigma'_ch) - ln U,  U = 256^-3   (R#2-R#4)
 *     SLM = 1 / (1 + e^d)
 *     t   = ln P(S|V=1) - ln P(S|V=0)
 *         = ln SLM - ln((1-p_O)(1-SLM) + p_O SLM)
 *         = -logaddexp(ln p_O, ln(1-p_O) + d)
 *     stored as the fixed-point integer q = rint(t * 2^20)            (R#16)
 *   stage 2, per voxel (i,j,k) (Eq 3-4; threshold P:111):
 *     for each camera, project the voxel centre to its nearest pixel (
 *     pinned FP32 arithmetic, R#10-R#13); out-of-view views contribute t = 0
 *     (SLM = 1/2, R#12);  S = sum of the in-view q;
 *     log-odds L = S * 2^-20 + logit(p_V);   occupied <=> L > logit(tau)
 *     (<=> posterior > tau, R#14), bit v = i + xlen (j + ylen k) of a uint32
 *     word array, word v >> 5, bit v & 31, LSB first (R#19).
 *
 * Conventions for every call:
 *   - Return value: PSFS_OK (0) or a positive PSFS_E* code.  No exception or
 *     abort ever crosses the ABI.  psfs_last_error(h) gives detail text.
 *   - Ownership: the caller owns every buffer it passes.  psfs_set_* copy their
 *     HOST inputs into library-owned device memory and return after the copy.
 *   - psfs_reconstruct* are asynchronous on the given CUDA stream (a
 *     cudaStream_t passed as void*, NULL = the legacy default stream): inputs
 *     must stay valid and outputs must not be read until the stream reaches
 *     that point.  Calls that enqueue work on the same handle must use one
 *     stream at a time (the handle owns one term buffer).
 *   - A handle is bound to one CUDA device and is not thread-safe.
 */
#ifndef PSFS_H
#define PSFS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PSFS_OK = 0,
    PSFS_EINVAL = 1,      /* NULL where required; both outputs NULL; non-finite or
                             out-of-range values (priors or tau not in (0,1), spacing
                             <= 0, sizes <= 0); fixed-point headroom exceeded
                             (ncam * max|t| * 2^20 >= 2^31); unaligned pointers   */
    PSFS_EDEGENERATE = 2, /* camera 3x3 block singular, or W/H <= 0      */
    PSFS_EDIM = 3,        /* background size != camera size                */
    PSFS_ECOUNT = 4,      /* some camera has no background model yet      */
    PSFS_ESTATE = 5,      /* call order violated (cameras before backgrounds ...)  */
    PSFS_ECUDA = 6,       /* a CUDA runtime call or kernel launch failed           */
    PSFS_ENOMEM = 7,      /* device allocation failed                              */
    PSFS_ELIMIT = 8,      /* more cameras / frames than this build supports        */
    PSFS_ETIMEOUT = 9     /* a peer rank did not reach the exchange barrier        */
};

#define PSFS_MAX_CAMERAS 64 /* per handle                                  */
#define PSFS_MAX_BATCH 16   /* frames fused into one stage-1/stage-2 pass  */
#define PSFS_MAX_PEERS 8    /* ranks of one fused peer exchange (one node) */
#define PSFS_MAX_TRAIN_FRAMES 512 /* frames of one psfs_train_background call */
#define PSFS_IPC_HANDLE_BYTES 64 /* size of one exported peer buffer handle */
#define PSFS_MC_HANDLE_BYTES 64  /* size of the exported multicast object handle (fabric handle) */
#define PSFS_SAMPLE_NEAREST 0  /* the pixel nearest the projected voxel centre (R#10) */
#define PSFS_SAMPLE_BILINEAR 1 /* bilinear SLM sample, clamped at the borders (R#26) */

typedef struct psfs_handle psfs_handle; /* opaque, library-owned */

/* Volume of interest ("xlen ... ylen ... zlen").
 * Voxel (i,j,k) centre = origin + spacing * (idx + 1/2) in mm (R#13). */
typedef struct {
    double origin[3];
    double spacing;
    int32_t xlen, ylen, zlen;
} psfs_grid;

/* Model constants.  psfs_default_params() fills the defaults below. */
typedef struct {
    double occlusion_prior; /* P(O=1), Eq 5: 0.5; in (0,1)           (R#7)  */
    double voxel_prior;     /* P(V=1), Eq 3: 0.5; in (0,1)                 (R#8)  */
    double threshold;       /* tau: occupied iff posterior > tau, 0.5      (R#14) */
    double sigma_floor;     /* sigma' = max(sigma, floor), 1.0 grey level  (R#6)  */
} psfs_params;

/* Placement of this handle in a z-slab partition of the grid (DESIGN.md
 * "Multi-GPU").  world = 1: the handle computes the whole grid.  world > 1:
 * the handle computes slices [k0, k1) with k0 = rank*zlen/world; requires
 * zlen % world == 0 and xlen*ylen*(zlen/world) % 32 == 0 so every slab is a
 * whole number of bitmask words.  The bitmask exchange (all-gather) between
 * ranks is either the caller's (NCCL through torch.distributed in the Python
 * layer) or fused into stage 2 (psfs_peer_alloc / psfs_peer_open /
 * psfs_reconstruct_peer below). */
typedef struct {
    int32_t device; /* CUDA device ordinal the handle allocates on            */
    int32_t rank;   /* 0 <= rank < world                                       */
    int32_t world;  /* >= 1                                                    */
} psfs_dist;

void psfs_default_params(psfs_params *out);

/* Create a handle.  dist may be NULL (device = current device, world = 1).
 * Errors: PSFS_EINVAL (NULL grid/out, bad sizes or params, slab not
 * word-aligned), PSFS_ECUDA. */
int psfs_create(const psfs_grid *grid, const psfs_params *params, const psfs_dist *dist,
                psfs_handle **out);

/* Set the calibrated cameras.  P: HOST, ncam*12 doubles, camera c's
 * row-major 3x4 matrix mapping homogeneous world mm to homogeneous pixels with
 * pixel centres at integer coordinates; width/height: HOST, ncam each.  The
 * library pre-composes A_c = S P_c T in double and rounds it once to float
 * (DESIGN.md "Pinned projection").  Resets every background model.
 * Errors: PSFS_EINVAL, PSFS_ELIMIT (ncam > PSFS_MAX_CAMERAS), PSFS_EDEGENERATE,
 * PSFS_ENOMEM, PSFS_ECUDA. */
int psfs_set_cameras(psfs_handle *h, int32_t ncam, const double *P, const int32_t *width,
                     const int32_t *height);

/* NEXT-3 boundary variants, any time after psfs_create:
 * channels = 3: 8-bit RGB frames (default; U = 256^-3); channels = 1:
 * 8-bit grayscale frames, H*W bytes per image, single-channel background
 * models, U = 256^-1 (R#25).  Changing the channel count discards every
 * background model (set or train them again before reconstructing).
 * sampling = PSFS_SAMPLE_NEAREST (default, the hot path) or
 * PSFS_SAMPLE_BILINEAR: each in-view camera contributes the per-view term of
 * Eq 5-9 evaluated at the bilinear interpolation of its SLM image
 * (Eq 1-2) around the projected voxel centre, neighbours clamped to the image
 * (R#26); the in-view rule is the nearest-pixel one (R#12).  Coarse
 * passes apply only to RGB nearest-pixel handles; other combinations take the
 * exact path (bilinear: groups of <= 8 frames).  psfs_color needs RGB.
 * Errors: PSFS_EINVAL (other values). */
int psfs_set_input(psfs_handle *h, int32_t channels, int32_t sampling);

/* Set camera `cam`'s single-Gaussian background model: mean and sigma
 * (a standard deviation per channel, R#2), HOST, height*width*channels floats
 * each (channels of psfs_set_input, default 3), row-major, channel-interleaved
 * (the frame layout).  sigma is clamped to
 * sigma_floor (R#6).  Errors: PSFS_ESTATE (no cameras), PSFS_EINVAL (cam out
 * of range, NULL, non-finite values), PSFS_EDIM (width/height differ from the
 * camera's), PSFS_ECUDA. */
int psfs_set_background(psfs_handle *h, int32_t cam, int32_t width, int32_t height,
                        const float *mean, const float *sigma);

/* NEXT-3, background-model training (the paper assumes the single
 * Gaussian of P:77 exists): camera `cam`'s per-pixel, per-channel sample mean
 * and population standard deviation over nframes background frames, sigma
 * clamped up to sigma_floor (R#6).  frames: HOST array of nframes
 * DEVICE pointers, each an H_c*W_c*channels uint8 image.  mean / sigma:
 * DEVICE, nullable, H_c*W_c*channels float (sigma after the clamp).  install != 0 makes the
 * result camera cam's background model, exactly as psfs_set_background with
 * these float values would, without a host round trip.  Asynchronous on
 * cuda_stream.  Errors: PSFS_ESTATE (no cameras), PSFS_EINVAL (cam out of
 * range, nframes <= 0 = EmptyInput of S:104, NULL frame, no output),
 * PSFS_ELIMIT (nframes > PSFS_MAX_TRAIN_FRAMES), PSFS_ECUDA. */
int psfs_train_background(psfs_handle *h, int32_t cam, int32_t nframes,
                          const uint8_t *const *frames, float *mean, float *sigma, int32_t install,
                          void *cuda_stream);

/* Reconstruct one frame set.  frames: HOST array of ncam DEVICE pointers, each
 * an H_c*W_c*3 uint8 RGB image (row-major, channel-interleaved; H_c*W_c bytes
 * for a grayscale handle, psfs_set_input).
 * logodds: DEVICE, nullable, float per voxel of this handle's slab
 * (xlen*ylen*(k1-k0), x-fastest, slab-relative).  bits: DEVICE, nullable,
 * ceil(xlen*ylen*zlen/32) uint32 words for the FULL grid; this handle writes
 * the words of its own slab only.  At least one output must be non-NULL.
 * Errors: PSFS_EINVAL, PSFS_ESTATE, PSFS_ECOUNT, PSFS_ECUDA. */
int psfs_reconstruct(psfs_handle *h, const uint8_t *const *frames, float *logodds, uint32_t *bits,
                     void *cuda_stream);

/* Reconstruct nframes frame sets in one call (frame-batched: the background
 * model is read once per group of up to PSFS_MAX_BATCH frames and every voxel
 * projection is computed once per group).  frames: HOST array of nframes*ncam
 * DEVICE pointers, frame-major (frames[f*ncam + c]).  logodds: nullable,
 * nframes consecutive slab arrays; bits: nullable, nframes consecutive
 * full-grid word arrays.  Same errors as psfs_reconstruct. */
int psfs_reconstruct_batch(psfs_handle *h, int32_t nframes, const uint8_t *const *frames,
                           float *logodds, uint32_t *bits, void *cuda_stream);

/* End-to-end variant with HOST buffers (the paper's non-blocking transfers on
 * several command queues): frames: HOST array of nframes*ncam HOST
 * pointers (page-locked memory gives real overlap), frame-major; logodds /
 * bits: nullable HOST outputs laid out as in psfs_reconstruct_batch.  The
 * library copies each group of frames -- only the region-of-interest rectangle
 * of each image, the pixels stage 1 reads (psfs_debug_roi) -- into its own
 * device staging buffers on
 * an internal copy stream, computes on cuda_stream, and copies the results back
 * on a second copy stream, double-buffered so group g+1's upload and group
 * g-1's download overlap group g's kernels (and a call's upload the previous
 * call's kernels).  Asynchronous: the host frames are read from the time of the
 * call on (they must not be the destination of copies still pending on
 * cuda_stream); host outputs are valid once cuda_stream has reached the end of
 * the call (synchronize it).
 * Same errors as psfs_reconstruct_batch, plus PSFS_ENOMEM for the staging. */
int psfs_reconstruct_host(psfs_handle *h, int32_t nframes, const uint8_t *const *frames,
                          float *logodds, uint32_t *bits, void *cuda_stream);

/* NEXT-2, inner-voxel removal ("remove voxels inside human body and get
 * the surface voxels"): the occupied voxels of this handle's
 * slab with at least one unoccupied 6-neighbour, voxels outside the volume
 * counting as unoccupied.  bits: DEVICE, the FULL grid's words (after the
 * all-gather in a z-slab partition).  surface_bits: DEVICE, nullable, full-grid
 * words; the slab's words are written.  indices: DEVICE, nullable, up to
 * `capacity` int64 linear voxel indices in increasing order.  count: DEVICE,
 * one int64, the exact number of surface voxels of the slab (also when it
 * exceeds capacity).  Asynchronous on cuda_stream.
 * Errors: PSFS_EINVAL, PSFS_ENOMEM, PSFS_ECUDA. */
int psfs_surface(psfs_handle *h, const uint32_t *bits, uint32_t *surface_bits, int64_t *indices,
                 int64_t capacity, int64_t *count, void *cuda_stream);

/* NEXT-1, probability filtering + thresholding merged ("we filter the
 * probability of voxels ... and then perform a thresholding process";
 * P:269-271): posterior P = 1/(1 + e^-L) from the log-odds,
 * 3x3x3 box average with zero padding outside the volume, occupied :=
 * smoothed > tau (the handle's threshold).  logodds: DEVICE, the whole grid
 * (x-fastest floats, e.g. psfs_reconstruct's output); smoothed: DEVICE,
 * nullable, nvox floats; bits: DEVICE, nullable, full-grid words.  World-1
 * handles only (a z-slab would need a one-slice halo from its neighbours).
 * Errors: PSFS_EINVAL, PSFS_ENOMEM, PSFS_ECUDA. */
int psfs_smooth_threshold(psfs_handle *h, const float *logodds, float *smoothed, uint32_t *bits,
                          void *cuda_stream);

/* NEXT-1 merged with reconstruction, from the exact sums (no float log-odds or
 * posterior volume in between; "merging this procedure will
 * significantly improve GPU computing efficiency").  S = sum of the in-view
 * Q11.20 terms (Eq 3-4), L = S 2^-20 + logit p_V, P = 1/(1 + e^-L), then the
 * 3x3x3 zero-padded box average and smoothed > tau as psfs_smooth_threshold.
 *
 * psfs_reconstruct_sums: both stages of the exact path with the int32 sums as
 *   the per-voxel output: sums DEVICE, nframes x (this handle's slab, x-fastest)
 *   int32; bits (nullable) the unsmoothed bitmask as psfs_reconstruct_batch.
 * psfs_smooth_sums: the smoothing of nframes such slabs.  A z-slab handle
 *   (psfs_dist world > 1) needs the neighbouring slabs' boundary slices:
 *   halo_lo = slice k0 - 1 (required when k0 > 0), halo_hi = slice k1 (required
 *   when k1 < zlen), DEVICE, nframes x xlen*ylen int32 each (the caller moves
 *   them between ranks: NCCL send/recv in parallel.py); slices past the volume
 *   are the zero padding.  smoothed (nullable): nframes x slab floats; bits
 *   (nullable): nframes full-grid word arrays, this slab's words written.
 * psfs_reconstruct_smoothed: world-1 handles: both in one call per frame group,
 *   the sums in library scratch (kMaxF frames of the slab).
 * All asynchronous on cuda_stream.  Errors: PSFS_EINVAL (NULL / missing halo /
 * world != 1 for psfs_reconstruct_smoothed), PSFS_ESTATE, PSFS_ECOUNT,
 * PSFS_ENOMEM, PSFS_ECUDA. */
int psfs_reconstruct_sums(psfs_handle *h, int32_t nframes, const uint8_t *const *frames, int32_t *sums,
                          uint32_t *bits, void *cuda_stream);
int psfs_smooth_sums(psfs_handle *h, int32_t nframes, const int32_t *sums, const int32_t *halo_lo,
                     const int32_t *halo_hi, float *smoothed, uint32_t *bits, void *cuda_stream);
int psfs_reconstruct_smoothed(psfs_handle *h, int32_t nframes, const uint8_t *const *frames, float *smoothed,
                              uint32_t *bits, void *cuda_stream);

void psfs_destroy(psfs_handle *h);

const char *psfs_status_string(int status);
const char *psfs_last_error(const psfs_handle *h);

/* ---- introspection (tests, planner) ------------------------------------ */

/* This handle's slab [k0, k1). */
int psfs_slab(const psfs_handle *h, int32_t *k0, int32_t *k1);

/* The pre-composed float matrices A_c (HOST out, ncam*12). */
int psfs_debug_matrices(const psfs_handle *h, float *out);

/* Stage 1 only, for one frame set over whole images: writes q (int32 Q11.20)
 * for every pixel, cameras concatenated in order (DEVICE out, sum_c W_c*H_c).
 * Asynchronous on cuda_stream. */
int psfs_debug_terms(psfs_handle *h, const uint8_t *const *frames, int32_t *terms_out,
                     void *cuda_stream);

/* The stage-1 work of one frame set: the pixels of the per-row spans of the
 * region of interest (the columns each row's slab hull covers, 4-aligned), or
 * of the rectangles where spans do not apply (psfs_debug_roi).  HOST out.
 * Errors: PSFS_EINVAL, PSFS_ESTATE (no cameras). */
int psfs_roi_pixels(const psfs_handle *h, int64_t *pixels);

/* Per-camera stage-1 region of interest the planner computed for this
 * handle's slab: HOST out, ncam*4 int32 (row0, row1, col0, col1), half-open;
 * every pixel a voxel of the slab can project to lies inside it. */
int psfs_debug_roi(const psfs_handle *h, int32_t *out);

/* Enable/disable the ROI restriction of stage 1 (default on). */
int psfs_set_roi_enabled(psfs_handle *h, int32_t enabled);  /* 2: rectangles without per-row spans */

/* Stage-1 kernel of the exact path: 0 = one pixel per thread; 1 = TMA
 * bulk-copy ring (needs every W % 16 == 0 and 16-byte aligned frames); 2 =
 * software-pipelined persistent kernel; 3 = four pixels per thread (W % 4,
 * 4-byte aligned frames); 4 = warp-row coalesced image loads with shuffles (W %
 * 32, 4-byte aligned); 5 = cp.async ring per warp; 6 = persistent four pixels
 * per thread, whole pass per thread (W % 4, 4-byte aligned frames; default).
 * A path whose requirement fails falls back to 0.  All give bit-identical terms
 * (DESIGN.md §8 has the measurements that made 6 the default). */
int psfs_set_stage1_path(psfs_handle *h, int32_t path);

/* Bits-only early exit (default off): when a call requests no log-odds, a
 * warp stops adding cameras once every one of its voxels and frames satisfies
 * S + (cameras left) * q_max <= T_q, q_max = rint(-ln p_O 2^20) + 1 bounding
 * every term -- the occupancy bit is then provably 0 and the bitmask is
 * identical to the full sum's.  Ignored when log-odds are requested. */
int psfs_set_carve(psfs_handle *h, int32_t enabled);

/* Coarse passes for bits-only calls (the threshold of
 * P:111 / R#14 needs only the sign of L - logit tau).  When a reconstruct call
 * requests no log-odds, stage 1 stores an 8-bit code per pixel and frame that
 * brackets the exact Q11.20 term q of Eq 5-9 (c 2^sh <= q <= c 2^sh + wc), 32
 * frames per 32-byte record (33..64 frames: 64-byte records read by lane
 * pairs); stage 2 sums the codes of every voxel's cameras
 * and decides every voxel-frame whose bracket lies on one side of T_q; the
 * others (rare: |L - logit tau| within about ncam * 2^(sh-20)) are summed
 * exactly from the frames and the model with the exact path's per-pixel
 * arithmetic.  The bitmask is bit-identical to the exact path's.
 * The undecided voxel-frames of a pass are listed by k_voxel_c8 and summed by a
 * second kernel (k_fixup_c8, one warp per entry, cameras across the lanes) that
 * patches their bits; entries beyond the list's capacity are summed in place by
 * the voxel kernel (slow, still exact).
 * psfs_reconstruct_peer uses coarse passes only when this device has native
 * atomics to every device that holds a peer buffer (NVLink / NVSwitch; checked
 * by psfs_peer_open), since the fix-up patches bits in every rank's buffer.
 * mode: 0 = off (always the exact int32 path), 1 = on (default), 2 = test mode
 * (every voxel-frame resolved exactly through the fix-up).  max_frames: frames
 * per coarse pass, 1..64 (default 64, at most 2048 / ncam; a call's frames are split into balanced
 * passes).  min_frames: calls with fewer frames take the exact path, which is
 * faster for small batches (0 = default 16).  fix_capacity: list entries (8
 * bytes each), 0 = automatic (1/1024 of a 64-frame pass's voxel-frames, within
 * 2^20 .. 2^26).  Coarse passes apply when the params
 * admit them (psfs_coarse_plan), xlen % 32 == 0, the tile depth kz <= 8 and
 * carve is off; otherwise calls take the exact path. */
int psfs_set_coarse(psfs_handle *h, int32_t mode, int32_t max_frames, int32_t min_frames,
                    int64_t fix_capacity);

/* Host-only: the coarse-code plan for params and ncam cameras.  out (HOST, 7
 * int32): admitted (sigma_floor >= 0.25 and p_O in [1e-3, 1 - 1e-3]), sh (code
 * quantum 2^sh in Q11.20 units), bias (the code of t = 0), wc (bracket width:
 * q in [c 2^sh, c 2^sh + wc]), K0, K1 (a voxel-frame whose code sum U = sum
 * over the cameras of (c + bias) has U >= K1 is occupied, U < K0 unoccupied,
 * otherwise summed exactly), T_q (occupied <=> S > T_q); eps (nullable): the
 * FP32 error bound in t the bracket is widened by. */
int psfs_coarse_plan(const psfs_params *params, int32_t ncam, int32_t *out, double *eps);

/* applies (nullable): whether a bits-only call of max_frames frames on this
 * handle takes coarse passes; fixups (nullable): voxel-frames resolved exactly since the last reset
 * (synchronous read of a device counter); reset != 0 zeroes the counter. */
int psfs_coarse_status(psfs_handle *h, int32_t *applies, int64_t *fixups, int32_t reset);

/* Coarse stage 1 for one frame set over whole images: the code byte (c + bias)
 * of every pixel, cameras concatenated (DEVICE out, sum_c W_c*H_c bytes), for
 * checking the bracket against psfs_debug_terms.  Asynchronous on cuda_stream.
 * PSFS_ESTATE when the params admit no coarse codes. */
int psfs_debug_codes(psfs_handle *h, const uint8_t *const *frames, uint8_t *codes_out,
                     void *cuda_stream);

/* How psfs_reconstruct_host moves the frames' region-of-interest rectangles
 * to the device: mode 1 (default) = when every frame pointer of a group is
 * page-locked host memory mapped into the device address space (e.g.
 * cudaHostAlloc / torch pin_memory under unified addressing; checked with
 * cudaPointerGetAttributes), a copy kernel (k_h2d_rows) reads the rows over
 * PCIe directly (zero-copy); otherwise, and with mode 0, the DMA engines copy
 * each rectangle (cudaMemcpy2DAsync).  Results are identical.
 * Errors: PSFS_EINVAL. */
int psfs_set_host_upload(psfs_handle *h, int32_t mode);

/* Overlapped batches (default on): with more than one frame group in a
 * psfs_reconstruct_batch call, stage 1 of group g+1 runs on an internal stream
 * beside stage 2 of group g (two term buffers); voxel_blocks_per_sm > 0 caps
 * k_voxel's resident blocks per SM to leave room for stage-1 blocks (default 0:
 * no cap, the measured best on B200).  Results are bit-identical either way. */
int psfs_set_overlap(psfs_handle *h, int32_t enabled, int32_t voxel_blocks_per_sm);

/* Stage-2 tile shape: 32 x 8*ty voxel columns (ty = 1 or 4, default 1) by kz
 * z-slices (1..64, default 4).  Results are bit-identical for every shape. */
int psfs_set_voxel_tile(psfs_handle *h, int32_t ty, int32_t kz);

/* Cap the number of frames fused into one pass (1, 2, 4, 8 or 16; default 16).
 * A 16-frame pass stores 64-byte term records (two sectors of one 128-byte
 * line) that two lanes of k_voxel read together. */
int psfs_set_max_fuse(psfs_handle *h, int32_t fmax);

/* NEXT-4, voxel colour ("the color rendering is also an iterative
 * process of all voxels", "Voxel color calculation"):
 * for each listed voxel, the mean 8-bit RGB of one frame set over the cameras
 * whose pinned nearest pixel (R#10-R#13, as the occupancy path) is in view and
 * whose SLM there (Eq 1-2) exceeds slm_gate (0.5 by default, in (0,1);
 * DESIGN.md R#23-R#24); no occlusion test.  frames: HOST array of ncam
 * DEVICE pointers (one frame set).  indices: DEVICE int64 linear voxel indices
 * (e.g. psfs_surface's list); count: DEVICE, one int64 -- min(*count, capacity)
 * entries are coloured, so psfs_surface's outputs chain without a host sync.
 * rgb: DEVICE, capacity x 3 float (0 when unset); nviews: DEVICE, nullable,
 * capacity int32 qualifying views (0: colour unset, -1: index outside the grid).
 * Asynchronous on cuda_stream.  Errors: PSFS_EINVAL, PSFS_ESTATE, PSFS_ECOUNT,
 * PSFS_ECUDA. */
int psfs_color(psfs_handle *h, const uint8_t *const *frames, const int64_t *indices,
               const int64_t *count, int64_t capacity, double slm_gate, float *rgb,
               int32_t *nviews, void *cuda_stream);

/* ---- Fused z-slab bitmask exchange over peer memory (DESIGN.md
 * section 9).  Every rank of a z-slab partition (psfs_dist.world = N <= PSFS_MAX_PEERS,
 * one process per GPU of one node, or several processes sharing one GPU) holds a
 * library-owned buffer of nframes full-grid bitmasks; stage 2 stores each
 * ballot byte of its slab into ALL N buffers (NVLink / NVSwitch peer stores
 * through CUDA IPC mappings), so no separate all-gather runs, and a device-side
 * barrier (release / acquire flags at system scope) orders the exchange on the
 * caller's stream -- no host synchronisation.
 *
 * psfs_peer_alloc: allocate this rank's buffer for up to nframes frames;
 *   *bits_out (HOST out) = its DEVICE address (nframes consecutive arrays of
 *   ceil(nvox/32) words, valid after psfs_reconstruct_peer's barrier, owned by
 *   the handle until psfs_destroy); ipc_handle_out (HOST, PSFS_IPC_HANDLE_BYTES)
 *   = the handle to pass to every other rank (the caller moves it, e.g. with
 *   torch.distributed.all_gather_object).  Errors: PSFS_EINVAL, PSFS_ELIMIT
 *   (world > PSFS_MAX_PEERS), PSFS_ENOMEM, PSFS_ECUDA.
 * psfs_peer_open: handles = HOST, world * PSFS_IPC_HANDLE_BYTES bytes in rank
 *   order (this rank's own entry is ignored); maps every peer buffer.  Errors:
 *   PSFS_ESTATE (no psfs_peer_alloc), PSFS_EINVAL, PSFS_ECUDA.
 * psfs_reconstruct_peer: as psfs_reconstruct_batch (nframes <= the allocated
 *   count) with bits going to every rank's buffer: entry barrier (every rank has
 *   finished the work its stream ordered before this call, so no rank
 *   overwrites a buffer still being read), both stages with peer stores, exit
 *   barrier.  Every rank must make the same sequence of calls.  Asynchronous
 *   on cuda_stream.  A barrier that waits more than ~10 s for a peer gives up
 *   and records the failure, which psfs_peer_status reports.  Ragged rows
 *   (xlen % 8 != 0) OR bits into the peers' words atomically: without native
 *   peer atomics to every buffer's device (psfs_peer_open) the call returns
 *   PSFS_ESTATE before any work (use the caller's all-gather instead).
 * psfs_peer_status: synchronizes cuda_stream; PSFS_ETIMEOUT if a barrier timed
 *   out since the last call, else PSFS_OK. */
int psfs_peer_alloc(psfs_handle *h, int32_t nframes, uint32_t **bits_out, void *ipc_handle_out);
int psfs_peer_open(psfs_handle *h, const void *handles);
int psfs_reconstruct_peer(psfs_handle *h, int32_t nframes, const uint8_t *const *frames,
                          float *logodds, void *cuda_stream);
int psfs_peer_status(psfs_handle *h, void *cuda_stream);

/* NVLS multicast bitmask buffer for the fused exchange (SURVEY.md 8(e) stretch:
 * "k_voxel stores ballot words through an NVLS multicast address"): with it,
 * psfs_reconstruct_peer sends every bitmask word once, as a multimem store the
 * NVSwitch replicates into every rank's copy (per-rank NVLink egress 1x the
 * slab instead of (world - 1)x), and the coarse fix-up patches bits with
 * multimem reductions (no peer atomics needed).  The IPC peer buffers of
 * psfs_peer_alloc / psfs_peer_open stay in use for the device barriers.  Setup,
 * every rank in order, host barriers between the steps:
 *   psfs_mc_create(h, nframes, handle_out): sizes the buffer (nframes bitmasks);
 *     rank 0 creates the multicast object (world devices) and writes its fabric
 *     handle (PSFS_MC_HANDLE_BYTES, HOST) for the others; other ranks write zeros;
 *   psfs_mc_attach(h, handle): ranks != 0 import rank 0's handle; every rank
 *     adds its device;  -- barrier: every device added --
 *   psfs_mc_bind(h, &bits): allocates this device's replica, binds it, maps the
 *     multicast and the local views; *bits = the local view (DEVICE, nframes
 *     full-grid bitmasks, valid after psfs_reconstruct_peer's exit barrier).
 *   -- barrier: every replica bound --
 * psfs_mc_release drops it (psfs_destroy does too).  Errors: PSFS_ESTATE when
 * the driver, the device or the fabric has no multicast support (the caller
 * keeps the N-store peer exchange), PSFS_EINVAL, PSFS_ECUDA. */
int psfs_mc_create(psfs_handle *h, int32_t nframes, void *handle_out);
int psfs_mc_attach(psfs_handle *h, const void *handle);
int psfs_mc_bind(psfs_handle *h, uint32_t **bits_out);
int psfs_mc_release(psfs_handle *h);

/* Per-kernel device timing (bench instrumentation): when enabled, every
 * stage-1 and stage-2 launch is bracketed by CUDA events on the launching
 * stream.  psfs_kernel_times synchronizes those events and returns the summed
 * milliseconds and launch counts of [0] k_likelihood and [1] k_voxel since the
 * last reset (HOST outs, 2 entries each; either may be NULL). */
int psfs_set_profiling(psfs_handle *h, int32_t enabled);
int psfs_kernel_times(psfs_handle *h, double *ms, int64_t *launches, int32_t reset);

/* Number of kernel launches the last psfs_reconstruct* call enqueued. */
int psfs_last_launch_count(const psfs_handle *h);

/* 1 if the planner proved the fast reciprocal exact for this grid and rig
 * (DESIGN.md "Pinned projection"), else 0. */
int psfs_fast_rcp_enabled(const psfs_handle *h);

/* Microbenchmark on the current device: L1 load bandwidth (bytes/s) of fully
 * coalesced 128-bit loads from an L1-resident window, the peak the stage-2
 * gather is compared against. */
int psfs_probe_l1_bandwidth(double *bytes_per_s);

/* Microbenchmark on the current device: bytes/s delivered by a voxel kernel's
 * gather pattern over random 128-byte lines of a table of table_bytes
 * (L2-resident when below ~100 MB), non-allocating 256-bit loads, at
 * blocks_per_sm x 256 threads per SM (1..8): sectors_per_line = 2 is
 * k_voxel16's (lane pairs read the two 32-byte sectors of one line, 3 blocks
 * per SM), 1 is k_voxel_c8's (each lane one 32-byte sector of its own line, 2
 * blocks per SM) -- the measured peaks of their rooflines;
 * 4: lane quads read the four sectors of one line (a 128-byte record's pattern).
 * Errors: PSFS_EINVAL, PSFS_ENOMEM, PSFS_ECUDA. */
int psfs_probe_gather_bandwidth(int64_t table_bytes, int32_t sectors_per_line, int32_t blocks_per_sm,
                                double *bytes_per_s);

/* Test hook: on the current device, count the floats w in [lo, hi) (every bit
 * pattern) whose fast reciprocal differs from the IEEE RN(1/w).  lo > 0. */
int psfs_debug_rcp_check(float lo, float hi, int64_t *mismatches);

#ifdef __cplusplus
}
#endif
#endif /* PSFS_H */
