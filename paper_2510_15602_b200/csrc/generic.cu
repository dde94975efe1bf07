// generic.cu -- K8: the general scoring path (any reference weights, any pad,
// finite sigma_p), materialising per-bin planes.
//
// It restates, plane by plane, the reference's non-fused route
// (scoring.py:59-112 and 274-280): window counts (quantize.py:85-89), the
// two-pointer Alg. 1 with the reference rescaled to each window's mass
// (transport.py:73-125) in fp64, and the box / Gaussian smoothing of the
// error planes followed by the own-bin gather (scoring.py:88-112).  It backs
// the public step APIs (patch_histograms, bin_error_maps, associate_errors)
// and the detect() configurations the fused kernel (score.cu) does not cover
// (zero padding, non-integer references, finite sigma_p).
#include "common.cuh"

namespace qfca {

// vertical window counts: col[p][i][y][x] = sum_dy [b(map(y+dy), x) == i]
template <typename BT>
__global__ void k_counts_vertical(const BT* __restrict__ bins, int64_t planes, int h, int w,
                                  int n_bins, int t, int pad, uint16_t* __restrict__ col) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = planes * n_bins * (int64_t)w;
    if (gid >= total) return;
    const int x = (int)(gid % w);
    const int i = (int)((gid / w) % n_bins);
    const int64_t p = gid / ((int64_t)w * n_bins);
    const BT* bp = bins + p * (int64_t)h * w;
    uint16_t* out = col + (p * n_bins + i) * (int64_t)h * w;
    const int r = t / 2;
    auto ind = [&](int yy) -> int {
        const int m = map_coord(yy, h, pad);
        return (m >= 0 && (int)bp[(int64_t)m * w + x] == i) ? 1 : 0;
    };
    int c = 0;
    for (int dy = -r; dy <= r; ++dy) c += ind(dy);
    out[x] = (uint16_t)c;
    for (int y = 1; y < h; ++y) {
        c += ind(y + r) - ind(y - r - 1);
        out[(int64_t)y * w + x] = (uint16_t)c;
    }
}

// horizontal window sums of the column counts -> counts (float or u16)
template <typename OT>
__global__ void k_counts_horizontal(const uint16_t* __restrict__ col, int64_t planes, int h,
                                    int w, int n_bins, int t, int pad, OT* __restrict__ out) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t hw = (int64_t)h * w;
    const int64_t total = planes * n_bins * hw;
    if (gid >= total) return;
    const int x = (int)(gid % w);
    const int64_t rowbase = gid - x;
    const int r = t / 2;
    int c = 0;
    for (int dx = -r; dx <= r; ++dx) {
        const int m = map_coord(x + dx, w, pad);
        if (m >= 0) c += col[rowbase + m];
    }
    out[gid] = (OT)c;
}

// Alg. 1 per pixel (transport.py:73-107) with R rescaled to the window mass,
// eps = 1e-9 * mass (transport.py:11, scoring.py:216-217).  E in fp64.
__global__ void k_mismatch_pixels(const uint16_t* __restrict__ counts, int64_t planes,
                                  int64_t hw, int n_bins, const double* __restrict__ refw,
                                  const double* __restrict__ centers,
                                  const uint8_t* __restrict__ skip, double* __restrict__ err) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= planes * hw) return;
    const int64_t p = gid / hw, px = gid % hw;
    const uint16_t* P = counts + p * n_bins * hw + px;
    double* out = err + p * n_bins * hw + px;
    const double* R = refw + p * n_bins;
    const double* Q = centers + p * n_bins;
    double mp = 0.0, mr = 0.0;
    for (int b = 0; b < n_bins; ++b) {
        mp += (double)P[b * hw];
        mr += R[b];
        out[b * hw] = 0.0;
    }
    if ((skip && skip[p]) || mr <= 0.0 || mp <= 0.0) return;
    const double eps = 1e-9 * (mp > 1e-300 ? mp : 1e-300);
    const double scale = mp / mr;
    double rem = (double)P[0], rrem = R[0] * scale, cur = 0.0;
    int i = 0, j = 0;
    while (i < n_bins && j < n_bins) {
        const double d = fabs(Q[i] - Q[j]);
        if (rem < rrem - eps) {
            cur = __dadd_rn(cur, __dmul_rn(rem, d));  // Numba does not contract
            rrem -= rem;
            out[i * hw] = cur;
            cur = 0.0;
            ++i;
            if (i < n_bins) rem = (double)P[i * hw];
        } else {
            cur = __dadd_rn(cur, __dmul_rn(rrem, d));
            rem -= rrem;
            ++j;
            if (j < n_bins) rrem = R[j] * scale;
        }
    }
    if (i < n_bins) out[i * hw] = cur;
    for (int b = 0; b < n_bins; ++b) {
        const double pb = (double)P[b * hw];
        out[b * hw] = pb > 0.0 ? out[b * hw] / pb : 0.0;
    }
}

// mismatch_batch (transport.py:110-125) on row-major fp64 rows: Pb (M, N),
// R / Q (N,), out (M, N).  One thread per row, identical arithmetic.
__global__ void k_mismatch_rows(const double* __restrict__ Pb, int64_t M, int n,
                                const double* __restrict__ R, const double* __restrict__ Q,
                                double* __restrict__ out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= M) return;
    const double* P = Pb + k * n;
    double* o = out + k * n;
    double mp = 0.0, mr = 0.0;
    for (int b = 0; b < n; ++b) mr += R[b];
    for (int b = 0; b < n; ++b) mp += P[b];
    const double eps = 1e-9 * (mp > 1e-300 ? mp : 1e-300);
    // _mismatch_row recomputes both masses (transport.py:76-81)
    mp = 0.0;
    mr = 0.0;
    for (int b = 0; b < n; ++b) {
        mp += P[b];
        mr += R[b];
        o[b] = 0.0;
    }
    if (mr <= 0.0 || mp <= 0.0) return;
    const double scale = mp / mr;
    double rem = P[0], rrem = R[0] * scale;
    int i = 0, j = 0;
    while (i < n && j < n) {
        const double d = fabs(Q[i] - Q[j]);
        if (rem < rrem - eps) {
            o[i] = __dadd_rn(o[i], __dmul_rn(rem, d));
            rrem -= rem;
            ++i;
            if (i < n) rem = P[i];
        } else {
            o[i] = __dadd_rn(o[i], __dmul_rn(rrem, d));
            rem -= rrem;
            ++j;
            if (j < n) rrem = R[j] * scale;
        }
    }
    for (int b = 0; b < n; ++b) o[b] = P[b] > 0.0 ? o[b] / P[b] : 0.0;
}

// vertical pass of the error-plane smoothing: tmp = sum_dy k[dy] E[map(y+dy)]
__global__ void k_smooth_vertical(const double* __restrict__ err, int64_t planes, int h, int w,
                                  int n_bins, int t, int pad, const Taps kern,
                                  double* __restrict__ tmp) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t hw = (int64_t)h * w;
    if (gid >= planes * n_bins * hw) return;
    const int64_t px = gid % hw, pl = gid / hw;
    const int y = (int)(px / w), x = (int)(px % w);
    const double* e = err + pl * hw;
    const int r = t / 2;
    double s = 0.0;
    for (int d = 0; d < t; ++d) {
        const int m = map_coord(y + d - r, h, pad);
        if (m >= 0) s = __dadd_rn(s, __dmul_rn(kern.k[d], e[(int64_t)m * w + x]));
    }
    tmp[gid] = s;
}

// horizontal pass + own-bin gather: score[p][y][x] = post * sum_dx k[dx] tmp[b][y][map(x+dx)]
template <typename BT>
__global__ void k_smooth_gather(const double* __restrict__ tmp, const BT* __restrict__ bins,
                                int64_t planes, int h, int w, int n_bins, int t, int pad,
                                const Taps kern, double post,
                                double* __restrict__ score) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t hw = (int64_t)h * w;
    if (gid >= planes * hw) return;
    const int64_t p = gid / hw, px = gid % hw;
    const int y = (int)(px / w), x = (int)(px % w);
    const int b = (int)bins[gid];
    const double* tp = tmp + (p * n_bins + b) * hw + (int64_t)y * w;
    const int r = t / 2;
    double s = 0.0;
    for (int d = 0; d < t; ++d) {
        const int m = map_coord(x + d - r, w, pad);
        if (m >= 0) s = __dadd_rn(s, __dmul_rn(kern.k[d], tp[m]));
    }
    score[gid] = s * post;
}

// fixed-order channel sum (scoring.py:264-281): acc[b][px] = sum_c score[b][c][px]
// over non-skipped channels; used[b] = number of those channels.
__global__ void k_channel_sum(const double* __restrict__ score, int64_t images, int channels,
                              int64_t hw, const uint8_t* __restrict__ skip, int accumulate,
                              double* __restrict__ acc, int* __restrict__ used) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= images * hw) return;
    const int64_t b = gid / hw, px = gid % hw;
    double s = accumulate ? acc[gid] : 0.0;
    int u = 0;
    for (int c = 0; c < channels; ++c) {
        if (skip && skip[b * channels + c]) continue;
        s += score[(b * channels + c) * hw + px];
        ++u;
    }
    acc[gid] = s;
    if (px == 0 && used) used[b] = (accumulate ? used[b] : 0) + u;
}

static inline unsigned nblk(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

int launch_window_counts(const void* bins, int bins_bytes, int64_t planes, int h, int w,
                         int n_bins, int t, int pad, uint16_t* col_scratch, void* out,
                         int out_kind, cudaStream_t st) {
    if (planes <= 0 || h <= 0 || w <= 0 || n_bins < 1 || t < 1 || (t & 1) == 0)
        return QFCA_ERR_ARG;
    if ((int64_t)t * t > 65535) return QFCA_ERR_UNSUPPORTED;
    const int64_t nv = planes * n_bins * (int64_t)w;
    if (bins_bytes == 1)
        k_counts_vertical<uint8_t><<<nblk(nv, 256), 256, 0, st>>>(
            (const uint8_t*)bins, planes, h, w, n_bins, t, pad, col_scratch);
    else if (bins_bytes == 2)
        k_counts_vertical<uint16_t><<<nblk(nv, 256), 256, 0, st>>>(
            (const uint16_t*)bins, planes, h, w, n_bins, t, pad, col_scratch);
    else if (bins_bytes == 4)
        k_counts_vertical<int32_t><<<nblk(nv, 256), 256, 0, st>>>(
            (const int32_t*)bins, planes, h, w, n_bins, t, pad, col_scratch);
    else
        return QFCA_ERR_ARG;
    const int64_t nh = planes * n_bins * (int64_t)h * w;
    if (out_kind == 0)
        k_counts_horizontal<float><<<nblk(nh, 256), 256, 0, st>>>(col_scratch, planes, h, w,
                                                                   n_bins, t, pad, (float*)out);
    else
        k_counts_horizontal<uint16_t><<<nblk(nh, 256), 256, 0, st>>>(
            col_scratch, planes, h, w, n_bins, t, pad, (uint16_t*)out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_mismatch_pixels(const uint16_t* counts, int64_t planes, int64_t hw, int n_bins,
                           const double* refw, const double* centers, const uint8_t* skip,
                           double* err, cudaStream_t st) {
    if (planes <= 0 || hw <= 0 || n_bins < 1) return QFCA_ERR_ARG;
    k_mismatch_pixels<<<nblk(planes * hw, 128), 128, 0, st>>>(counts, planes, hw, n_bins, refw,
                                                               centers, skip, err);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_mismatch_rows(const double* Pb, int64_t M, int n, const double* R, const double* Q,
                         double* out, cudaStream_t st) {
    if (M <= 0 || n < 1) return QFCA_ERR_ARG;
    k_mismatch_rows<<<nblk(M, 128), 128, 0, st>>>(Pb, M, n, R, Q, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_smooth_gather(const double* err, const void* bins, int bins_bytes, int64_t planes,
                         int h, int w, int n_bins, int t, int pad, const double* taps_host,
                         double post, double* tmp, double* score, cudaStream_t st) {
    if (planes <= 0 || h <= 0 || w <= 0 || n_bins < 1 || t < 1 || t > QFCA_MAX_TAPS)
        return QFCA_ERR_ARG;
    Taps kern;
    kern.n = t;
    for (int i = 0; i < t; ++i) kern.k[i] = taps_host[i];
    const int64_t hw = (int64_t)h * w;
    k_smooth_vertical<<<nblk(planes * n_bins * hw, 256), 256, 0, st>>>(err, planes, h, w, n_bins,
                                                                        t, pad, kern, tmp);
    if (bins_bytes == 1)
        k_smooth_gather<uint8_t><<<nblk(planes * hw, 256), 256, 0, st>>>(
            tmp, (const uint8_t*)bins, planes, h, w, n_bins, t, pad, kern, post, score);
    else if (bins_bytes == 2)
        k_smooth_gather<uint16_t><<<nblk(planes * hw, 256), 256, 0, st>>>(
            tmp, (const uint16_t*)bins, planes, h, w, n_bins, t, pad, kern, post, score);
    else if (bins_bytes == 4)
        k_smooth_gather<int32_t><<<nblk(planes * hw, 256), 256, 0, st>>>(
            tmp, (const int32_t*)bins, planes, h, w, n_bins, t, pad, kern, post, score);
    else
        return QFCA_ERR_ARG;
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_channel_sum(const double* score, int64_t images, int channels, int64_t hw,
                       const uint8_t* skip, int accumulate, double* acc, int* used,
                       cudaStream_t st) {
    if (images <= 0 || channels <= 0 || hw <= 0) return QFCA_ERR_ARG;
    k_channel_sum<<<nblk(images * hw, 256), 256, 0, st>>>(score, images, channels, hw, skip,
                                                           accumulate, acc, used);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
