// finalize.cu -- K5: channel mean, final Gaussian smoothing, border-excluded
// image score and bilinear upsampling.
//
// Restates scoring.py:311-319 (agg = acc / used, all-degenerate -> zeros),
// scoring.py:161-166 + features.py:49-77 (normalised Gaussian of radius
// ceil(3 sigma), rows (axis 0) then columns, np.pad modes), scoring.py:169-174
// (image_score_of) and scoring.py:177-180 + tensor_io.py:127-151 (bilinear,
// half-pixel centres, computed in fp64, rounded to float32).
#include "common.cuh"

namespace qfca {

// agg[b][px] = (sum_g partial[b][g][px]) / used[b]  (fixed group order)
__global__ void k_reduce_partials(const float* __restrict__ partial, int64_t images, int groups,
                                  int64_t hw, const int* __restrict__ used,
                                  double* __restrict__ agg) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= images * hw) return;
    const int64_t b = gid / hw, px = gid % hw;
    double s = 0.0;
    for (int g = 0; g < groups; ++g) s += (double)partial[(b * groups + g) * hw + px];
    const int u = used[b];
    agg[gid] = u > 0 ? s / (double)u : s;
}

// agg[b][px] = acc[b][px] / used[b]  (used == 0 -> acc, which is all zeros)
__global__ void k_divide_used(const double* __restrict__ acc, int64_t images, int64_t hw,
                              const int* __restrict__ used, double* __restrict__ agg) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= images * hw) return;
    const int u = used[gid / hw];
    agg[gid] = u > 0 ? acc[gid] / (double)u : acc[gid];
}

// separable convolution pass; axis 0 = along rows index y, axis 1 = along x
__global__ void k_sep_conv(const double* __restrict__ in, int64_t images, int h, int w,
                           int axis, const Taps taps, int pad, double* __restrict__ out) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t hw = (int64_t)h * w;
    if (gid >= images * hw) return;
    const int64_t b = gid / hw, px = gid % hw;
    const int y = (int)(px / w), x = (int)(px % w);
    const double* p = in + b * hw;
    const int r = taps.n / 2;
    double s = 0.0;
    for (int i = 0; i < taps.n; ++i) {
        const int m = axis == 0 ? map_coord(y + i - r, h, pad) : map_coord(x + i - r, w, pad);
        const double v = m < 0 ? 0.0 : (axis == 0 ? p[(int64_t)m * w + x] : p[(int64_t)y * w + m]);
        s = __dadd_rn(s, __dmul_rn(taps.k[i], v));  // no FMA: NumPy order
    }
    out[gid] = s;
}

// per-image max over pixels at least `border` away from the edges
__global__ void k_image_score(const double* __restrict__ scores, int h, int w, int border,
                              double* __restrict__ image_score) {
    const int64_t b = blockIdx.x;
    const double* p = scores + b * (int64_t)h * w;
    int bb = border;
    bb = min(bb, (h - 1) / 2);
    bb = min(bb, (w - 1) / 2);
    if (bb < 0) bb = 0;
    const int ih = h - 2 * bb, iw = w - 2 * bb;
    double m = -INFINITY;
    for (int64_t i = threadIdx.x; i < (int64_t)ih * iw; i += blockDim.x) {
        const int y = bb + (int)(i / iw), x = bb + (int)(i % iw);
        m = fmax(m, p[(int64_t)y * w + x]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ double sh[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[warp] = m;
    __syncthreads();
    if (warp == 0) {
        m = lane < (int)(blockDim.x >> 5) ? sh[lane] : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) image_score[b] = m;
    }
}

// bilinear resize with half-pixel centres (tensor_io.py:127-151), fp64 math,
// float32 result.  Source is fp64 (the score map).
__global__ void k_upsample(const double* __restrict__ in, int64_t images, int h, int w, int oh,
                           int ow, float* __restrict__ out) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ohw = (int64_t)oh * ow;
    if (gid >= images * ohw) return;
    const int64_t b = gid / ohw, px = gid % ohw;
    const int oy = (int)(px / ow), ox = (int)(px % ow);
    const double* p = in + b * (int64_t)h * w;
    if (h == oh && w == ow) {
        out[gid] = (float)p[(int64_t)oy * w + ox];
        return;
    }
    const double ys = ((double)oy + 0.5) * (double)h / (double)oh - 0.5;
    const double xs = ((double)ox + 0.5) * (double)w / (double)ow - 0.5;
    const double fyf = floor(ys), fxf = floor(xs);
    const int y0 = (int)fmin(fmax(fyf, 0.0), (double)(h - 1));
    const int x0 = (int)fmin(fmax(fxf, 0.0), (double)(w - 1));
    const int y1 = min(y0 + 1, h - 1), x1 = min(x0 + 1, w - 1);
    const double fy = fmin(fmax(ys - (double)y0, 0.0), 1.0);
    const double fx = fmin(fmax(xs - (double)x0, 0.0), 1.0);
    // explicit rounding (no FMA contraction) to match NumPy bit for bit
    const double top = __dadd_rn(__dmul_rn(p[(int64_t)y0 * w + x0], 1.0 - fx),
                                 __dmul_rn(p[(int64_t)y0 * w + x1], fx));
    const double bot = __dadd_rn(__dmul_rn(p[(int64_t)y1 * w + x0], 1.0 - fx),
                                 __dmul_rn(p[(int64_t)y1 * w + x1], fx));
    out[gid] = (float)__dadd_rn(__dmul_rn(top, 1.0 - fy), __dmul_rn(bot, fy));
}

static inline unsigned nblk(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

int launch_reduce_partials(const float* partial, int64_t images, int groups, int64_t hw,
                           const int* used, double* agg, cudaStream_t st) {
    if (images <= 0 || groups <= 0 || hw <= 0) return QFCA_ERR_ARG;
    k_reduce_partials<<<nblk(images * hw, 256), 256, 0, st>>>(partial, images, groups, hw, used,
                                                               agg);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_divide_used(const double* acc, int64_t images, int64_t hw, const int* used,
                       double* agg, cudaStream_t st) {
    if (images <= 0 || hw <= 0) return QFCA_ERR_ARG;
    k_divide_used<<<nblk(images * hw, 256), 256, 0, st>>>(acc, images, hw, used, agg);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_sep_conv(const double* in, int64_t images, int h, int w, int axis,
                    const double* taps_host, int ntaps, int pad, double* out, cudaStream_t st) {
    if (images <= 0 || h <= 0 || w <= 0 || ntaps < 1 || ntaps > QFCA_MAX_TAPS || !(ntaps & 1))
        return QFCA_ERR_ARG;
    Taps taps;
    taps.n = ntaps;
    for (int i = 0; i < ntaps; ++i) taps.k[i] = taps_host[i];
    k_sep_conv<<<nblk(images * (int64_t)h * w, 256), 256, 0, st>>>(in, images, h, w, axis, taps,
                                                                    pad, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_image_score(const double* scores, int64_t images, int h, int w, int border,
                       double* image_score, cudaStream_t st) {
    if (images <= 0 || h <= 0 || w <= 0) return QFCA_ERR_ARG;
    k_image_score<<<(unsigned)images, 256, 0, st>>>(scores, h, w, border, image_score);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_upsample(const double* in, int64_t images, int h, int w, int oh, int ow, float* out,
                    cudaStream_t st) {
    if (images <= 0 || h <= 0 || w <= 0 || oh <= 0 || ow <= 0) return QFCA_ERR_ARG;
    k_upsample<<<nblk(images * (int64_t)oh * ow, 256), 256, 0, st>>>(in, images, h, w, oh, ow,
                                                                      out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
