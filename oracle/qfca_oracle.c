/*
 * qfca_oracle.c -- CPU ORACLE (test infrastructure, NOT product code).
 *
 * A plain-C restatement of the reference QFCA scoring path
 * (/root/reference/pkg/src/qfca, pure Python/NumPy/Numba).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker / CPU baseline.  The product
 * (paper_2510_15602_b200) never links or calls it.
 *
 * Every function follows the reference algorithm step for step (same fp64
 * arithmetic, same summed-area tables, same two-pointer walk) so that it is
 * pinned bit-for-bit against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py).  Citations are file:line in the reference.
 *
 * OpenMP is used only across channels (each channel is independent,
 * scoring.py:264-281); the channel sum is then done in fixed channel order in
 * fp64, exactly like the reference's `acc += chan_scores` (scoring.py:273).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PAD_ZERO 0
#define PAD_REFLECT 1
#define PAD_WRAP 2

/* transport.py:11 */
static const double EPS_FACTOR = 1e-9;

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* quantize.py:61-68 -- per-channel min/max, degenerate = hi <= lo */
void oracle_fit_quantizer(const float* v, int64_t C, int64_t HW, double* lo,
                          double* hi, uint8_t* degen) {
    for (int64_t c = 0; c < C; ++c) {
        const float* p = v + c * HW;
        float mn = p[0], mx = p[0];
        for (int64_t i = 1; i < HW; ++i) {
            if (p[i] < mn) mn = p[i];
            if (p[i] > mx) mx = p[i];
        }
        lo[c] = (double)mn;
        hi[c] = (double)mx;
        degen[c] = (hi[c] <= lo[c]) ? 1 : 0;
    }
}

/* quantize.py:71-82 -- floor((v - lo) * N / safe) in fp64, clip, degenerate -> 0 */
void oracle_bin_indices(const float* v, int64_t C, int64_t HW, const double* lo,
                        const double* hi, const uint8_t* degen, int n_bins,
                        int32_t* out) {
    for (int64_t c = 0; c < C; ++c) {
        double span = hi[c] - lo[c];
        double safe = span > 0 ? span : 1.0;
        for (int64_t i = 0; i < HW; ++i) {
            double q = ((double)v[c * HW + i] - lo[c]) * (double)n_bins / safe;
            double f = floor(q);
            int64_t k = (int64_t)f;
            if (f < 0) k = 0;
            if (f > (double)(n_bins - 1)) k = n_bins - 1;
            if (degen[c]) k = 0;
            out[c * HW + i] = (int32_t)k;
        }
    }
}

/* quantize.py:109-116 */
int oracle_sample_stride(int h, int w, int budget) {
    int s = 1;
    while ((int64_t)((h + s - 1) / s) * (int64_t)((w + s - 1) / s) > budget) ++s;
    return s;
}

/* pooling.py:20-38 (np.pad semantics) -- index into the source for a padded
 * coordinate.  np.pad 'reflect' = mirror without edge repeat, applied
 * repeatedly for large margins; pad_plane switches to 'edge' on BOTH axes if
 * either axis has size 1 (pooling.py:31-35).  Returns -1 for zero padding. */
static int np_pad_index(int c, int n, int pad, int edge_mode) {
    if (c >= 0 && c < n) return c;
    if (pad == PAD_ZERO) return -1;
    if (pad == PAD_WRAP) {
        int m = c % n;
        return m < 0 ? m + n : m;
    }
    if (edge_mode || n == 1) return c < 0 ? 0 : n - 1;
    while (c < 0 || c >= n) {
        if (c < 0) c = -c;
        if (c >= n) c = 2 * n - 2 - c;
    }
    return c;
}

/* scoring.py:158-174 (_map_coord) */
static int map_coord(int c, int n, int pad_code) {
    if (c >= 0 && c < n) return c;
    if (pad_code == PAD_ZERO) return -1;
    if (pad_code == PAD_WRAP) {
        int m = c % n;
        return m < 0 ? m + n : m;
    }
    if (n == 1) return 0;
    while (c < 0 || c >= n) {
        if (c < 0) c = -c;
        if (c >= n) c = 2 * n - 2 - c;
    }
    return c;
}

static int cmp_float(const void* a, const void* b) {
    float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}

/* quantize.py:150-200, mode "median-quan" (default) only:
 * sample_patches (119-132) -> per-row sort (178) -> per-rank lower median
 * (180, 135-140) -> _quantize_values_to_hist (143-147).
 * weights: (C, N) fp64. */
void oracle_select_reference_median(const float* v, int64_t C, int h, int w,
                                    const double* lo, const double* hi,
                                    const uint8_t* degen, int n_bins, int t,
                                    int budget, int pad, double* weights) {
    int r = t / 2;
    int t2 = t * t;
    int stride = oracle_sample_stride(h, w, budget);
    int ny = (h + stride - 1) / stride, nx = (w + stride - 1) / stride;
    int S = ny * nx;
    int edge_mode = (pad == PAD_REFLECT) && !(h > 1 && w > 1);
    int kmed = (S - 1) / 2;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < C; ++c) {
        double* wc = weights + c * n_bins;
        for (int i = 0; i < n_bins; ++i) wc[i] = 0.0;
        if (degen[c]) {
            wc[0] = (double)t2;
            continue;
        }
        const float* plane = v + c * (int64_t)h * w;
        float* patches = (float*)malloc(sizeof(float) * (size_t)S * t2);
        float* col = (float*)malloc(sizeof(float) * (size_t)S);
        int s = 0;
        for (int yi = 0; yi < ny; ++yi)
            for (int xi = 0; xi < nx; ++xi, ++s) {
                int y = yi * stride, x = xi * stride;
                float* row = patches + (size_t)s * t2;
                for (int dy = 0; dy < t; ++dy) {
                    int yy = np_pad_index(y + dy - r, h, pad, edge_mode);
                    for (int dx = 0; dx < t; ++dx) {
                        int xx = np_pad_index(x + dx - r, w, pad, edge_mode);
                        row[dy * t + dx] =
                            (yy < 0 || xx < 0) ? 0.0f : plane[(int64_t)yy * w + xx];
                    }
                }
                qsort(row, (size_t)t2, sizeof(float), cmp_float);
            }
        double span = hi[c] > lo[c] ? hi[c] - lo[c] : 1.0;
        for (int k = 0; k < t2; ++k) {
            for (int q = 0; q < S; ++q) col[q] = patches[(size_t)q * t2 + k];
            qsort(col, (size_t)S, sizeof(float), cmp_float);
            double val = (double)col[kmed];
            double f = floor((val - lo[c]) * (double)n_bins / span);
            if (f < 0) f = 0;
            if (f > n_bins - 1) f = n_bins - 1;
            wc[(int)f] += 1.0;
        }
        free(patches);
        free(col);
    }
}

/* transport.py:73-107 (_mismatch_row): Alg. 1 with the reference rescaled to
 * the patch mass and an eps tie guard. */
void oracle_mismatch_row(const double* P, const double* R, const double* Q,
                         int n, double eps, double* out) {
    double mp = 0.0, mr = 0.0;
    for (int b = 0; b < n; ++b) {
        mp += P[b];
        mr += R[b];
        out[b] = 0.0;
    }
    if (mr <= 0.0 || mp <= 0.0) return;
    double scale = mp / mr;
    double rem = P[0], rrem = R[0] * scale;
    int i = 0, j = 0;
    while (i < n && j < n) {
        double d = fabs(Q[i] - Q[j]);
        if (rem < rrem - eps) {
            out[i] += rem * d;
            rrem -= rem;
            ++i;
            if (i < n) rem = P[i];
        } else {
            out[i] += rrem * d;
            rem -= rrem;
            ++j;
            if (j < n) rrem = R[j] * scale;
        }
    }
    for (int b = 0; b < n; ++b) out[b] = P[b] > 0.0 ? out[b] / P[b] : 0.0;
}

/* transport.py:110-125 (mismatch_batch) */
void oracle_mismatch_batch(const double* Pb, int64_t M, int n, const double* R,
                           const double* Q, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < M; ++k) {
        double mp = 0.0;
        for (int b = 0; b < n; ++b) mp += Pb[k * n + b];
        oracle_mismatch_row(Pb + k * n, R, Q, n,
                            EPS_FACTOR * (mp > 1e-300 ? mp : 1e-300), out + k * n);
    }
}

/* scoring.py:177-232 (_channel_score_kernel): per-bin indicator SATs ->
 * counts, per-pixel Alg. 1, per-bin error SATs -> own-bin gather, x 1/T^2.
 * All fp64, identical loop order. */
void oracle_channel_score(const int32_t* idx, int h, int w, int nbins, int t,
                          int pad_code, const double* refw, const double* centers,
                          double* score_out) {
    int r = t / 2;
    int hp = h + 2 * r, wp = w + 2 * r;
    int64_t hw = (int64_t)h * w;
    double* counts = (double*)malloc(sizeof(double) * (size_t)hw * nbins);
    double* err = (double*)malloc(sizeof(double) * (size_t)hw * nbins);
    double* sat = (double*)calloc((size_t)(hp + 1) * (wp + 1), sizeof(double));
    int* ymap = (int*)malloc(sizeof(int) * hp);
    int* xmap = (int*)malloc(sizeof(int) * wp);
    int W1 = wp + 1;
    for (int y = 0; y < hp; ++y) ymap[y] = map_coord(y - r, h, pad_code);
    for (int x = 0; x < wp; ++x) xmap[x] = map_coord(x - r, w, pad_code);
    for (int i = 0; i < nbins; ++i) {
        for (int y = 0; y < hp; ++y) {
            int yy = ymap[y];
            double rowsum = 0.0;
            for (int x = 0; x < wp; ++x) {
                int xx = xmap[x];
                if (yy >= 0 && xx >= 0 && idx[(int64_t)yy * w + xx] == i) rowsum += 1.0;
                sat[(y + 1) * W1 + x + 1] = sat[y * W1 + x + 1] + rowsum;
            }
        }
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x)
                counts[((int64_t)y * w + x) * nbins + i] =
                    sat[(y + t) * W1 + x + t] - sat[y * W1 + x + t] -
                    sat[(y + t) * W1 + x] + sat[y * W1 + x];
    }
    for (int64_t p = 0; p < hw; ++p) {
        double mp = 0.0;
        for (int b = 0; b < nbins; ++b) mp += counts[p * nbins + b];
        oracle_mismatch_row(counts + p * nbins, refw, centers, nbins,
                            EPS_FACTOR * (mp > 1e-300 ? mp : 1e-300), err + p * nbins);
    }
    double inv = 1.0 / (double)(t * t);
    for (int i = 0; i < nbins; ++i) {
        for (int y = 0; y < hp; ++y) {
            int yy = ymap[y];
            double rowsum = 0.0;
            for (int x = 0; x < wp; ++x) {
                int xx = xmap[x];
                if (yy >= 0 && xx >= 0) rowsum += err[((int64_t)yy * w + xx) * nbins + i];
                sat[(y + 1) * W1 + x + 1] = sat[y * W1 + x + 1] + rowsum;
            }
        }
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x)
                if (idx[(int64_t)y * w + x] == i)
                    score_out[(int64_t)y * w + x] =
                        (sat[(y + t) * W1 + x + t] - sat[y * W1 + x + t] -
                         sat[(y + t) * W1 + x] + sat[y * W1 + x]) * inv;
    }
    free(counts);
    free(err);
    free(sat);
    free(ymap);
    free(xmap);
}

/* Window counts of one bin-index plane: (N, h, w) float64, via the same SAT
 * construction as the scoring kernel (scoring.py:191-211); equals
 * quantize.py:85-89 (box_average_stack of the one-hot planes x T^2). */
void oracle_channel_histograms(const int32_t* idx, int h, int w, int nbins,
                               int t, int pad_code, double* counts_nhw) {
    int r = t / 2;
    int hp = h + 2 * r, wp = w + 2 * r;
    int W1 = wp + 1;
    double* sat = (double*)calloc((size_t)(hp + 1) * (wp + 1), sizeof(double));
    int* ymap = (int*)malloc(sizeof(int) * hp);
    int* xmap = (int*)malloc(sizeof(int) * wp);
    for (int y = 0; y < hp; ++y) ymap[y] = map_coord(y - r, h, pad_code);
    for (int x = 0; x < wp; ++x) xmap[x] = map_coord(x - r, w, pad_code);
    for (int i = 0; i < nbins; ++i) {
        for (int y = 0; y < hp; ++y) {
            int yy = ymap[y];
            double rowsum = 0.0;
            for (int x = 0; x < wp; ++x) {
                int xx = xmap[x];
                if (yy >= 0 && xx >= 0 && idx[(int64_t)yy * w + xx] == i) rowsum += 1.0;
                sat[(y + 1) * W1 + x + 1] = sat[y * W1 + x + 1] + rowsum;
            }
        }
        if (pad_code == PAD_ZERO) {
            /* pooling.py:144-152: the zero-pad path clamps the window */
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x) {
                    int r0 = y - r < 0 ? 0 : y - r, r1 = y + r + 1 > h ? h : y + r + 1;
                    int c0 = x - r < 0 ? 0 : x - r, c1 = x + r + 1 > w ? w : x + r + 1;
                    counts_nhw[((int64_t)i * h + y) * w + x] =
                        sat[(r1 + r) * W1 + c1 + r] - sat[(r0 + r) * W1 + c1 + r] -
                        sat[(r1 + r) * W1 + c0 + r] + sat[(r0 + r) * W1 + c0 + r];
                }
        } else {
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x)
                    counts_nhw[((int64_t)i * h + y) * w + x] =
                        sat[(y + t) * W1 + x + t] - sat[y * W1 + x + t] -
                        sat[(y + t) * W1 + x] + sat[y * W1 + x];
        }
    }
    free(sat);
    free(ymap);
    free(xmap);
}

/* The per-channel loop of detect (scoring.py:258-281) for the uniform-sigma_p
 * path: channel scores for every non-degenerate channel, summed in channel
 * order in fp64.  Channels run in parallel into private buffers; the sum is
 * sequential so the result is independent of the thread count.
 * centers follow quantize.py:29-38.  Returns the number of used channels. */
int oracle_score_channels(const int32_t* bins, int64_t C, int h, int w,
                          int nbins, int t, int pad_code, const double* lo,
                          const double* hi, const uint8_t* degen,
                          const double* refw, double* acc) {
    int64_t hw = (int64_t)h * w;
    double* per = (double*)malloc(sizeof(double) * (size_t)C * hw);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < C; ++c) {
        if (degen[c]) continue;
        double* centers = (double*)malloc(sizeof(double) * nbins);
        double width = hi[c] > lo[c] ? (hi[c] - lo[c]) / nbins : 1.0;
        for (int i = 0; i < nbins; ++i) centers[i] = lo[c] + ((double)i + 0.5) * width;
        oracle_channel_score(bins + c * hw, h, w, nbins, t, pad_code,
                             refw + c * nbins, centers, per + c * hw);
        free(centers);
    }
    int used = 0;
    for (int64_t p = 0; p < hw; ++p) acc[p] = 0.0;
    for (int64_t c = 0; c < C; ++c) {
        if (degen[c]) continue;
        for (int64_t p = 0; p < hw; ++p) acc[p] += per[c * hw + p];
        ++used;
    }
    free(per);
    return used;
}
