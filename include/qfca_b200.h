/*
 * qfca_b200.h -- C-ABI of the B200-native QFCA scoring path (sm_100a).
 *
 * The reference (arxiv 2510.15602, /root/reference/pkg/src/qfca) is pure
 * Python; it has no C FFI.  Its closest native surface is the pair of Numba
 * kernels that a binding would replace:
 *   _channel_score_kernel(idx, nbins, t, pad_code, refw, centers, score_out)
 *       scoring.py:177-232           -> qfca_score (+ qfca_select_reference)
 *   mismatch_batch(Pb, R, Q, out)      transport.py:110-125 -> qfca_mismatch_pixels
 * and the NumPy stages around them, each of which gets an entry point below
 * (file:line of the function it replaces in the comment).  libqfca_b200.so
 * exports exactly these symbols.
 *
 * Conventions (all entry points):
 *   - plain device pointers and sizes, no framework types; the caller owns
 *     and allocates every buffer (the library allocates nothing persistent);
 *   - work is enqueued on `stream` (a cudaStream_t, NULL = legacy default)
 *     and is asynchronous; no host synchronisation except where stated;
 *   - return value: QFCA_OK (0) or an error code (QFCA_ERR_*); argument
 *     errors are detected before anything is enqueued;
 *   - feature planes are float32, contiguous (images, channels, h, w); a
 *     "plane" is one (image, channel) h x w map; bins are uint8 (n_bins <=
 *     256), uint16 (<= 65536) or int32 (bins_bytes = 1, 2, 4);
 *   - pad codes follow scoring.py:155: 0 zero, 1 reflect, 2 wrap.
 */
#ifndef QFCA_B200_H
#define QFCA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QFCA_OK 0
#define QFCA_ERR_ARG 1
#define QFCA_ERR_CUDA 2
#define QFCA_ERR_UNSUPPORTED 3

#define QFCA_REF_MEDIAN_QUAN 0 /* quantize.py:174-183 (default) */
#define QFCA_REF_MEAN_QUAN 1   /* quantize.py:174-183 (per-rank mean) */
#define QFCA_REF_QUAN_MEDIAN 2 /* quantize.py:184-199 */
#define QFCA_REF_QUAN_MEAN 3   /* quantize.py:184-199 */

int qfca_abi_version(void);
/* number of kernels this library has launched since it was loaded */
int64_t qfca_launch_count(void);
const char* qfca_status_str(int status);

/* fit_quantizer (quantize.py:61-68) + FeatureMap finiteness (features.py:36-37):
 * per-plane min -> lo, max -> hi; *nonfinite |= 1 if any value is not finite. */
int qfca_fit_quantizer(const float* x, int64_t planes, int64_t plane_len, float* lo, float* hi,
                       int32_t* nonfinite, void* stream);

/* bin_indices (quantize.py:71-82), bit-exact fp64 rule; degenerate -> 0 */
int qfca_bin_indices(const float* x, int64_t planes, int64_t plane_len, const float* lo,
                     const float* hi, int32_t n_bins, void* bins, int32_t bins_bytes,
                     void* stream);

/* fit_quantizer + bin_indices in one call (quantize.py:61-82): lo/hi/nonfinite
 * as qfca_fit_quantizer, bins as qfca_bin_indices, bit-identical to the two
 * calls; one pass over x when a plane fits in shared memory (<= 16384 values,
 * plane_len % 4 == 0, 2 <= n_bins <= 65), else the two kernels. */
int qfca_quantize(const float* x, int64_t planes, int64_t plane_len, int32_t n_bins, float* lo,
                  float* hi, int32_t* nonfinite, void* bins, int32_t bins_bytes, void* stream);

/* _sample_grid stride (quantize.py:109-116); host-only helper */
int qfca_sample_stride(int32_t h, int32_t w, int32_t sample_budget);

/* select_reference (quantize.py:150-200), sort-free.  stats is (planes, n_bins)
 * int32:  mode 0 (median-quan): cumulative reference counts V_i, so the
 *         reference weights are R_i = V_i - V_{i-1} (exact integers);
 *         mode 2 (quan-median): per-bin lower median of the window counts;
 *         mode 3 (quan-mean): per-bin sum of the window counts over samples.
 * Degenerate planes: mode 0 -> V = T^2; modes 2/3 -> bin 0 only. */
int qfca_select_reference(const void* bins, int32_t bins_bytes, const float* lo, const float* hi,
                          int64_t planes, int32_t h, int32_t w, int32_t n_bins,
                          int32_t patch_size, int32_t pad, int32_t sample_budget, int32_t mode,
                          int32_t* stats, void* stream);

/* select_reference (quantize.py:150-200) of any mode as the reference's fp64
 * (planes, n_bins) weights, bit-identical: median-quan / quan-median / quan-mean
 * from the bins (K3 statistics, then NumPy's arithmetic for the quan-* rescale);
 * mean-quan from the float32 values (sample patches, per-patch sort, per-rank
 * fp64 mean in sample order, binned).  mode: QFCA_REF_*.  Degenerate planes
 * (hi <= lo) get [T^2, 0, ...]. */
int64_t qfca_reference_weights_workspace_bytes(int64_t planes, int32_t h, int32_t w,
                                               int32_t n_bins, int32_t patch_size,
                                               int32_t sample_budget, int32_t mode);
int qfca_reference_weights(const float* values, const void* bins, int32_t bins_bytes,
                           const float* lo, const float* hi, int64_t planes, int32_t h, int32_t w,
                           int32_t n_bins, int32_t patch_size, int32_t pad, int32_t sample_budget,
                           int32_t mode, void* workspace, int64_t workspace_bytes,
                           double* weights, void* stream);

/* patch_histograms (quantize.py:85-106): window counts (planes, n_bins, h, w),
 * counts_kind 0 = float32, 1 = uint16.  scratch: planes*n_bins*h*w uint16. */
int qfca_window_counts(const void* bins, int32_t bins_bytes, int64_t planes, int32_t h,
                       int32_t w, int32_t n_bins, int32_t patch_size, int32_t pad,
                       uint16_t* scratch, void* counts, int32_t counts_kind, void* stream);

/* mismatch_batch (transport.py:110-125) over every pixel of every plane:
 * counts (planes, n_bins, hw) uint16, ref_weights / centers (planes, n_bins)
 * fp64, err (planes, n_bins, hw) fp64.  skip[plane] != 0 -> zero errors. */
int qfca_mismatch_pixels(const uint16_t* counts, int64_t planes, int64_t hw, int32_t n_bins,
                         const double* ref_weights, const double* centers, const uint8_t* skip,
                         double* err, void* stream);

/* mismatch_batch (transport.py:110-125) verbatim: Pb (rows, n_bins) fp64
 * row-major, R / Q (n_bins) fp64, out (rows, n_bins) fp64 */
int qfca_mismatch_rows(const double* Pb, int64_t rows, int32_t n_bins, const double* R,
                       const double* Q, double* out, void* stream);

/* _smooth_error_planes + own-bin gather (scoring.py:88-112): separable filter
 * of the error planes with taps (host array, patch_size taps: ones for the
 * box, the normalised Gaussian for finite sigma_p), times post_scale, read at
 * each pixel's own bin.  scratch: planes*n_bins*h*w fp64; score: planes*h*w. */
int qfca_smooth_gather(const double* err, const void* bins, int32_t bins_bytes, int64_t planes,
                       int32_t h, int32_t w, int32_t n_bins, int32_t patch_size, int32_t pad,
                       const double* taps_host, double post_scale, double* scratch,
                       double* score, void* stream);

/* fixed-order channel sum (scoring.py:264-281) of per-channel scores */
int qfca_channel_sum(const double* score, int64_t images, int32_t channels, int64_t hw,
                     const uint8_t* skip, int32_t accumulate, double* acc, int32_t* used,
                     void* stream);

/* number of non-degenerate channels per image (scoring.py:281 `used`) */
int qfca_count_used(const float* lo, const float* hi, int64_t images, int32_t channels,
                    int32_t* used, void* stream);

/* which fused scoring kernel qfca_detect / qfca_score_ex (with a scratch) pick
 * for this shape (host-only): N = scoreN.cu (1 = score.cu), -1 none. */
int qfca_score_version(int32_t h, int32_t w, int32_t n_bins, int32_t patch_size,
                       int32_t channels, int64_t images, int32_t pad, int32_t sample_budget,
                       int32_t with_reference);

/* channel groups qfca_score will use (host-only) for groups_hint (<= 0: auto);
 * with_reference = 0 asks for the in-kernel reference selection (returns -1
 * where that is not available). */
int qfca_score_groups(int32_t h, int32_t w, int32_t n_bins, int32_t patch_size, int32_t channels,
                      int64_t images, int32_t groups_hint, int32_t pad, int32_t sample_budget,
                      int32_t with_reference);

/* select the fused scoring kernel: 0 = auto, the first that applies of
 * v6 score6.cu (128-wide planes / tiles, T <= 15, N <= 256; needs the
 * caller's scratch), v7 score7.cu (128-wide, T = 17..65, N <= 256; scratch),
 * v4 score4.cu (planes <= 64 wide), v3 score3.cu, v5 score5.cu (any odd T),
 * v2 score2.cu, v1 score.cu (any shape); 1..7 = force that version
 * (unsupported shapes then return status 3).  Process-global. */
int qfca_set_score_kernel(int32_t version);

/* THE HOT PATH: _channel_score_kernel + channel accumulation
 * (scoring.py:177-232, 258-281) fused, for uniform sigma_p, median-quan and
 * reflect / wrap padding.  ref_cum = qfca_select_reference mode-0 stats, or
 * NULL to select the reference inside the kernel (select_reference,
 * quantize.py:150-200, from the same window counts; sample_budget applies).
 * partial: (images, groups, h, w) float32, must be zeroed by the caller; each
 * group adds its channels' scores in fixed channel order. */
int qfca_score(const void* bins, int32_t bins_bytes, const float* lo, const float* hi,
               const int32_t* ref_cum, int64_t images, int32_t channels, int32_t h, int32_t w,
               int32_t n_bins, int32_t patch_size, int32_t pad, int32_t sample_budget,
               int32_t groups, float* partial, void* stream);

/* qfca_score with a caller-owned global scratch: the 128-column kernels (v6
 * csrc/score6.cu, v7 csrc/score7.cu) keep each plane's window counts in an
 * L2-resident scratch;
 * qfca_score_scratch_bytes gives its size for a configuration (0: the chosen
 * kernel needs none, -1: unsupported) and qfca_score_groups_ex the channel
 * groups of the kernel chosen with (with_scratch = 1) or without a scratch. */
int qfca_score_ex(const void* bins, int32_t bins_bytes, const float* lo, const float* hi,
                  const int32_t* ref_cum, int64_t images, int32_t channels, int32_t h, int32_t w,
                  int32_t n_bins, int32_t patch_size, int32_t pad, int32_t sample_budget,
                  int32_t groups, void* scratch, int64_t scratch_bytes, float* partial,
                  void* stream);
/* qfca_score_ex over tiles of wide planes read in place (no gathered copy):
 * "image" i of the launch is tile (i / ncs, i % ncs) of the channels x hbig x
 * wbig bins planes -- rows rst[i / ncs] .., columns cst[i % ncs] .. (device
 * int32 arrays; every column start and wbig a multiple of col_align bytes,
 * 4 / 8 / 16), th x tw (tw = 128) each; lo / hi / ref_cum per (tile, channel)
 * as qfca_score.  The 128-column kernel v6 only (status 3 otherwise: gather
 * the tiles and call qfca_score_ex).  sharding.py:_strip_partial, the
 * wide-plane route of detect (scoring.py:235-299 on 1024 x 1024 planes). */
int qfca_score_tiles(const void* bins, int32_t bins_bytes, const float* lo, const float* hi,
                     const int32_t* ref_cum, int32_t channels, int32_t hbig, int32_t wbig,
                     const int32_t* rst, int32_t nr, const int32_t* cst, int32_t ncs,
                     int32_t col_align, int32_t th, int32_t tw, int32_t n_bins,
                     int32_t patch_size, int32_t pad, int32_t sample_budget, int32_t groups,
                     void* scratch, int64_t scratch_bytes, float* partial, void* stream);
int64_t qfca_score_scratch_bytes(int32_t h, int32_t w, int32_t n_bins, int32_t patch_size,
                                 int32_t channels, int64_t images, int32_t groups_hint,
                                 int32_t pad, int32_t sample_budget, int32_t with_reference);
int qfca_score_groups_ex(int32_t h, int32_t w, int32_t n_bins, int32_t patch_size,
                         int32_t channels, int64_t images, int32_t groups_hint, int32_t pad,
                         int32_t sample_budget, int32_t with_reference, int32_t with_scratch);

/* agg = (sum over groups, fixed order, fp64) / used   (scoring.py:283-289) */
int qfca_reduce_partials(const float* partial, int64_t images, int32_t groups, int64_t hw,
                         const int32_t* used, double* agg, void* stream);
int qfca_divide_used(const double* acc, int64_t images, int64_t hw, const int32_t* used,
                     double* agg, void* stream);

/* one separable pass of gaussian_blur (features.py:56-77); axis 0 = rows */
int qfca_sep_conv(const double* in, int64_t images, int32_t h, int32_t w, int32_t axis,
                  const double* taps_host, int32_t ntaps, int32_t pad, double* out, void* stream);

/* image_score_of (scoring.py:141-146) */
int qfca_image_score(const double* scores, int64_t images, int32_t h, int32_t w, int32_t border,
                     double* image_score, void* stream);

/* upsample_scores (scoring.py:149-152, tensor_io.py:127-151) -> float32 */
int qfca_upsample(const double* in, int64_t images, int32_t h, int32_t w, int32_t out_h,
                  int32_t out_w, float* out, void* stream);

/* pca_fit pieces (features.py:157-180): per-plane fp64 mean, centred fp32 copy */
int qfca_plane_mean(const float* x, int64_t planes, int64_t plane_len, double* mean, void* stream);
int qfca_center(const float* x, int64_t planes, int64_t plane_len, const double* mean, float* out,
                void* stream);

/* pca_residual (features.py:183-193): r = (x-mu) - V^T V (x-mu), fp64 math,
 * float32 out.  mean (C) / comps (k, C) fp64, per image if per_image_model. */
int qfca_pca_residual(const float* x, int64_t images, int32_t channels, int64_t hw,
                      const double* mean, const double* comps, int32_t k,
                      int32_t per_image_model, float* out, void* stream);
/* pca_residual of the channel slice [c_lo, c_hi) only -> out (images, c_hi - c_lo,
 * hw): z = V (x - mu) still contracts all channels (a channel-sharded rank's
 * residual, sharding.detect_pca_sharded).  QFCA_ERR_UNSUPPORTED unless C % 8 == 0,
 * C >= 16, hw % 4 == 0 (the fp64 tensor-core kernel). */
int qfca_pca_residual_slice(const float* x, int64_t images, int32_t channels, int64_t hw,
                            const double* mean, const double* comps, int32_t k,
                            int32_t per_image_model, int32_t c_lo, int32_t c_hi, float* out,
                            void* stream);

/* Cholesky QR of a batch of tall fp64 blocks (batch, rows, cols) row-major,
 * in place: Y <- Y L^-T, L L^T = Y^T Y (re-orthonormalisation step of the
 * top-k subspace eigensolver that replaces np.linalg.eigh, features.py:173) */
int qfca_cholqr(double* blocks, int64_t batch, int32_t rows, int32_t cols, void* stream);

/* Cholesky-QR factor of a batch of p x p Gram matrices G = Y^T Y (p <= 32):
 * rinv = R^-1 with G = R^T R, so Y R^-1 has orthonormal columns (subspace
 * iteration of the top-k eigensolver replacing np.linalg.eigh,
 * features.py:173).  A numerically singular pivot yields a zero column. */
int qfca_chol_rinv(const double* gram, int64_t batch, int32_t p, double* rinv, void* stream);

/* Eigen-decomposition of a batch of symmetric p x p matrices (p <= 32) by
 * cyclic parallel Jacobi: evals (batch, p) descending, evecs (batch, p, p)
 * with eigenvector j in column j (Rayleigh-Ritz step of the same solver). */
int qfca_sym_eig(const double* h, int64_t batch, int32_t p, double* evals, double* evecs,
                 void* stream);

/* Block Lanczos (8-column blocks, full reorthogonalisation) on a batch of
 * symmetric C x C fp64 matrices (C % 64 == 0, C <= 512), the Krylov stage of the
 * top-k eigensolver replacing np.linalg.eigh of pca_fit (features.py:173):
 * q0 (C, 8) seeded start block R (the kernel starts from qr(cov R)); basis
 * (batch, 8*passes, C) receives the Krylov basis (vector-contiguous), h
 * (batch, n, n) row-major the upper block triangle of H = basis^T cov basis
 * (n = 8*passes <= C, passes <= 32); passes + 1 sweeps over cov in all.
 * With twin_basis (same shape as basis), exchange (batch * 4 * C * 8 doubles)
 * and flags (batch int32, zeroed) non-NULL, each matrix runs on a cluster of
 * two CTAs that split the passes over cov; NULL: one CTA per matrix. */
int qfca_lanczos(const double* cov, int64_t batch, int32_t C, int32_t passes, const double* q0,
                 double* basis, double* h, double* twin_basis, double* exchange,
                 int32_t* flags, void* stream);

/* Top-32 subspace of the Lanczos projection (batch, n, n), n <= 128, n % 8 == 0,
 * as qfca_lanczos writes it (upper block triangle): x <- qr(H (H x)) for `iters`
 * steps from the seeded start block x0 (n, 32); outputs x (batch, n, 32) and
 * the Rayleigh-Ritz matrix hm = x^T H x (batch, 32, 32), whose eigenpairs
 * (qfca_sym_eig) give the Ritz pairs (Ritz vectors basis^T x u). */
int qfca_ritz(const double* h, int64_t batch, int32_t n, const double* x0, int32_t iters,
              double* x, double* hm, void* stream);

/* Tiles of wide uint8 bin planes (channels, h, w), w % 4 == 0: out[t][c][y][x]
 * = bins[c][row_starts[t / n_cols] + y][col_starts[t % n_cols] + x] for tile_h x
 * tile_w tiles, column starts multiples of 4 (the 128-column fused kernel on
 * the 1024^2 feature planes of configs[4]; device arrays of starts). */
int qfca_gather_tiles(const void* bins, int32_t channels, int32_t h, int32_t w,
                      const int32_t* row_starts, int32_t n_rows, const int32_t* col_starts,
                      int32_t n_cols, int32_t tile_h, int32_t tile_w, void* out, void* stream);

/* ---- box-pooling API (pooling.py:20-172).  Pad modes: 0 zero, 1 reflect,
 * 2 wrap, 3 edge (np.pad 'edge': pad_plane's reflect on a length-1 axis,
 * pooling.py:31-35); given per axis.  dtype codes: 0 f32, 1 f64, 2 u8,
 * 3 i32, 4 i64, 5 i16, 6 u16, 7 bool. */
/* pad_plane (pooling.py:20-38): planes (planes, h, w) of elem_bytes-sized
 * elements -> out (planes, h + 2 margin, w + 2 margin), same element type. */
int qfca_pad_planes(const void* x, int64_t planes, int32_t h, int32_t w, int32_t margin,
                    int32_t mode_rows, int32_t mode_cols, int32_t elem_bytes, void* out,
                    void* stream);
/* build_sat (pooling.py:56-64): cumsum (planes, H + 1, W + 1) fp64, H = h +
 * 2 margin, of the padded plane -- np.cumsum down the rows, then across the
 * columns, both sequential (bit-identical to NumPy). */
int qfca_build_sat(const void* x, int32_t dtype, int64_t planes, int32_t h, int32_t w,
                   int32_t margin, int32_t mode_rows, int32_t mode_cols, double* cumsum,
                   void* stream);
/* _box_sum_map / box_average(_stack) (pooling.py:97-158) from a SAT: clamp = 1
 * for zero padding (SAT without margin, clamped rectangles), 0 for a SAT with
 * margin k / 2; out = ((c11 - c01) - c10) + c00, divided by divisor if > 0. */
int qfca_sat_box(const double* cumsum, int64_t planes, int32_t h, int32_t w, int32_t k,
                 int32_t clamp, double divisor, double* out, void* stream);
/* box_sum (pooling.py:71-94) for n rectangles (r0, r1, c0, c1) of one SAT of
 * row length sat_w. */
int qfca_sat_rects(const double* cumsum, int32_t sat_w, const int32_t* rects, int64_t n,
                   double* out, void* stream);
/* naive_box_average (pooling.py:161-172): the k^2 shifted planes summed in
 * (dy, dx) order in fp64, / k^2. */
int qfca_naive_box(const void* x, int32_t dtype, int64_t planes, int32_t h, int32_t w, int32_t k,
                   int32_t mode_rows, int32_t mode_cols, double* out, void* stream);

/* Covariance of pca_fit (features.py:167-171): cov = (x - mean)^T (x - mean) / n
 * for a batch of images, x (images, C, hw) fp32 channel-major, mean (images, C)
 * fp64 -> cov (images, C, C) fp64.  fp64-accurate (~1e-11 relative): the
 * centred values become 32-bit per-channel fixed point, split into int8
 * digits, and the digit products run exactly on the int8 tensor cores
 * (tcgen05.mma kind::i8).  Needs hw <= 16384; workspace from
 * qfca_covariance_workspace_bytes.  Returns 3 (unsupported) otherwise. */
int64_t qfca_covariance_workspace_bytes(int64_t images, int32_t C, int32_t hw);
int qfca_covariance(const float* x, int64_t images, int32_t C, int32_t hw, const double* mean,
                    void* workspace, int64_t workspace_bytes, double* cov, void* stream);
/* Same, also forming the plane means (features.py:170) in the same pass over x:
 * mean (images, C) fp64 is an output. */
int qfca_mean_covariance(const float* x, int64_t images, int32_t C, int32_t hw, double* mean,
                         void* workspace, int64_t workspace_bytes, double* cov, void* stream);

/* ---- evaluation metrics (metrics.py) ---- */

/* Pooled interiors of a batch of maps (metrics.py:37-41 EvalSample.interior,
 * 61-68 _pooled): scores (images, H, W) fp64 (scores_bytes 8) or fp32 (4),
 * mask (images, H, W) uint8 -> out (images, H-2b, W-2b) fp64 and, if labels is
 * not NULL, labels (same shape) uint8 0/1.  If out32 is not NULL it also gets
 * the values as float32, and *inexact (device int32, zeroed by the caller) is
 * set when some value is not a float32 value (then out32 must not be ranked).
 * If image_max is not NULL (images uint64, zeroed by the caller) it receives
 * each image's interior maximum (metrics.py:175-179) in an order-preserving
 * encoding: u = bits(v) | 2^63 for v >= 0, else u = ~bits(v). */
int qfca_pool_interior(const void* scores, int32_t scores_bytes, const uint8_t* mask,
                       int32_t images, int32_t H, int32_t W, int32_t border, double* out,
                       uint8_t* labels, float* out32, int32_t* inexact, uint64_t* image_max,
                       void* stream);

/* qfca_pool_interior over separately allocated maps (metrics.py:62-68, the
 * same _pooled order): score_images and mask_images are DEVICE arrays of
 * `images` device pointers, each to one contiguous H x W map (scores_bytes 8
 * or 4; masks one byte per pixel, nonzero = anomalous, e.g. torch.bool).
 * Saves stacking a class's maps into one buffer before pooling. */
int qfca_pool_interior_table(const void* const* score_images, int32_t scores_bytes,
                             const uint8_t* const* mask_images, int32_t images, int32_t H,
                             int32_t W, int32_t border, double* out, uint8_t* labels, float* out32,
                             int32_t* inexact, uint64_t* image_max, void* stream);

/* Rank statistics of pooled scores (metrics.py:44-58 _rank_auroc,
 * 157-172 f1_optimal): one stable sort, then stats[0] = positives,
 * stats[1] = 2 x the rank sum of the positives (average ranks for ties; exact),
 * stats[2] = the bits of the best F1 over all thresholds (fp64).  Keys are
 * fp64 (key_bytes 8) or float32 (4: same order and ties when every score is a
 * float32 value, half the radix passes).  sorted_out (n keys, may be NULL)
 * receives the ascending scores (for the PRO quantiles, metrics.py:83-88).
 * n < 2^31; workspace from qfca_rank_stats_workspace_bytes. */
int64_t qfca_rank_stats_workspace_bytes(int64_t n, int32_t key_bytes);
int qfca_rank_stats(const void* scores, int32_t key_bytes, const uint8_t* labels, int64_t n,
                    void* workspace, int64_t workspace_bytes, void* sorted_out, uint64_t* stats,
                    void* stream);

/* 8-connected components of a batch of masks (metrics.py:76-80, scipy
 * ndimage.label with a 3x3 structure), images x h x w uint8 -> comp (same
 * shape) int32: -1 outside the masks, else the component number in raster
 * order of first pixels, numbered across the batch (image 0 first);
 * *n_comp (device int32) = number of components.  labels (may be NULL) gets
 * the raster index of each pixel's component root.  images*h*w < 2^31. */
int64_t qfca_components_workspace_bytes(int64_t n);
int qfca_components(const uint8_t* mask, int32_t images, int32_t h, int32_t w, void* workspace,
                    int64_t workspace_bytes, int32_t* labels, int32_t* comp, int32_t* n_comp,
                    void* stream);

/* PRO histograms (metrics.py:91-120): thr_asc (m <= 2048 ascending distinct
 * thresholds); each pixel goes to slot #{thr <= score}.  comp_hist
 * ((comp_hi - comp_lo), m + 1) int32 counts the pixels of components
 * [comp_lo, comp_hi) (zeroed by the caller), normal_hist (m + 1) uint64 the
 * pixels with comp < 0 (may be NULL). */
int qfca_pro_histograms(const double* scores, const int32_t* comp, int64_t n,
                        const double* thr_asc, int32_t m, int32_t comp_lo, int32_t comp_hi,
                        int32_t* comp_hist, uint64_t* normal_hist, void* stream);
/* pro[j] += (pixels >= thr_asc[j]) / size over the ncomp histograms in order
 * (metrics.py:112-115); comp_hist is turned into suffix sums in place. */
int qfca_pro_accumulate(int32_t* comp_hist, int32_t ncomp, int32_t m, double* pro, void* stream);

/* ---- one-call detect (scoring.py:235-299) for the fused configuration ---- */
typedef struct qfca_config {
    int32_t n_bins;        /* PipelineConfig.n_bins (16) */
    int32_t patch_size;    /* PipelineConfig.patch_size (9) */
    int32_t pad;           /* 1 reflect (default) or 2 wrap */
    int32_t sample_budget; /* 4096 */
    int32_t border;        /* border exclusion (patch_size / 2 by default) */
    int32_t groups;        /* channel groups (<= 0: auto) */
    double sigma_s;        /* 1.0 */
} qfca_config;

int64_t qfca_detect_workspace_bytes(int64_t images, int32_t channels, int32_t h, int32_t w,
                                    const qfca_config* cfg);

/* features (images, channels, h, w) -> scores (images, h, w) fp64,
 * image_scores (images) fp64, used (images) int32, *nonfinite (device int32). */
int qfca_detect(const float* features, int64_t images, int32_t channels, int32_t h, int32_t w,
                const qfca_config* cfg, void* workspace, int64_t workspace_bytes, double* scores,
                double* image_scores, int32_t* used, int32_t* nonfinite, void* stream);

/* qfca_detect with optional timing hooks: stage_events[0] / [1] (cudaEvent_t
 * or NULL) are recorded on `stream` right before / after the fused scoring
 * kernel (qfca_score). */
int qfca_detect_ex(const float* features, int64_t images, int32_t channels, int32_t h, int32_t w,
                   const qfca_config* cfg, void* workspace, int64_t workspace_bytes,
                   double* scores, double* image_scores, int32_t* used, int32_t* nonfinite,
                   void* const* stage_events, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* QFCA_B200_H */
