// finalize.cu -- K5: channel mean, final Gaussian smoothing, border-excluded
// image score and bilinear upsampling.
//
// Restates scoring.py:283-291 (agg = acc / used, all-degenerate -> zeros),
// scoring.py:133-138 + features.py:49-77 (normalised Gaussian of radius
// ceil(3 sigma), rows (axis 0) then columns, np.pad modes), scoring.py:141-146
// (image_score_of) and scoring.py:149-152 + tensor_io.py:127-151 (bilinear,
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
    const int iw = w - 2 * bb;
    double m = -INFINITY;
    if (iw >= (int)blockDim.x) {  // wide rows: coalesced row sweeps, no index division
        for (int y = bb; y < h - bb; ++y) {
            const double* row = p + (int64_t)y * w + bb;
#pragma unroll 4
            for (int x = threadIdx.x; x < iw; x += blockDim.x) m = fmax(m, row[x]);
        }
    } else {
        const int ih = h - 2 * bb;
        for (int64_t i = threadIdx.x; i < (int64_t)ih * iw; i += blockDim.x) {
            const int y = bb + (int)(i / iw), x = bb + (int)(i % iw);
            m = fmax(m, p[(int64_t)y * w + x]);
        }
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
// float32 result.  Source is fp64 (the score map).  One CTA per (image, band
// of UP_ROWS output rows, UP_CHUNK columns); thread = 4 consecutive columns
// (weights in registers), one float4 store per output row; each output costs
// four (cached) loads and the six rounded products / three sums of the
// reference formula.
constexpr int UP_THREADS = 256;
constexpr int UP_ROWS = 32;
constexpr int UP_CHUNK = 4 * UP_THREADS;  // output columns per CTA (4 per thread)

__device__ __forceinline__ void up_coord(int o, int n, int on, int& i0, int& i1, double& f) {
    const double s = ((double)o + 0.5) * (double)n / (double)on - 0.5;
    const double ff = floor(s);
    i0 = (int)fmin(fmax(ff, 0.0), (double)(n - 1));
    i1 = min(i0 + 1, n - 1);
    f = fmin(fmax(s - (double)i0, 0.0), 1.0);
}

__global__ void __launch_bounds__(UP_THREADS)
k_upsample(const double* __restrict__ in, int h, int w, int oh, int ow, int bands, int chunks,
           float* __restrict__ out) {
    __shared__ int sy0[UP_ROWS], sy1[UP_ROWS];
    __shared__ double sfy[UP_ROWS], sgy[UP_ROWS];
    const int b = blockIdx.x / (bands * chunks);
    const int band = (blockIdx.x / chunks) % bands, cx0 = (blockIdx.x % chunks) * UP_CHUNK;
    const int cw = min(UP_CHUNK, ow - cx0);
    const int oy0 = band * UP_ROWS, nrows = min(oh, oy0 + UP_ROWS) - oy0;
    const double* p = in + (int64_t)b * h * w;
    float* o = out + (int64_t)b * oh * ow + cx0;
    for (int i = threadIdx.x; i < nrows; i += UP_THREADS) {
        int y0, y1;
        double fy;
        up_coord(oy0 + i, h, oh, y0, y1, fy);
        sy0[i] = y0;
        sy1[i] = y1;
        sfy[i] = fy;
        sgy[i] = 1.0 - fy;
    }
    // this thread's 4 consecutive output columns: weights in registers (the
    // fp64 divisions once per CTA), then one float4 per output row
    const int c0 = 4 * threadIdx.x;
    int x0[4], x1[4];
    double fx[4], gx[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int ox = min(c0 + k, cw - 1);
        up_coord(cx0 + ox, w, ow, x0[k], x1[k], fx[k]);
        gx[k] = 1.0 - fx[k];
    }
    __syncthreads();
    if (c0 >= cw) return;
    const bool vec = c0 + 4 <= cw && ((ow | cx0) & 3) == 0;
    // the horizontal interpolations of the two source rows are shared by every
    // output row between the same pair (8 rows at 8x): recomputed only when the
    // pair changes (CTA-uniform), so an output row costs the vertical blend only
    int py0 = -1, py1 = -1;
    double top[4], bot[4];
    for (int r = 0; r < nrows; ++r) {
        const int y0 = sy0[r], y1 = sy1[r];
        if (y0 != py0 || y1 != py1) {
            const double* r0 = p + (int64_t)y0 * w;
            const double* r1 = p + (int64_t)y1 * w;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                // explicit rounding (no FMA contraction) to match NumPy bit for bit
                top[k] = __dadd_rn(__dmul_rn(__ldg(r0 + x0[k]), gx[k]),
                                   __dmul_rn(__ldg(r0 + x1[k]), fx[k]));
                bot[k] = __dadd_rn(__dmul_rn(__ldg(r1 + x0[k]), gx[k]),
                                   __dmul_rn(__ldg(r1 + x1[k]), fx[k]));
            }
            py0 = y0;
            py1 = y1;
        }
        const double fy = sfy[r], gy = sgy[r];
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = (float)__dadd_rn(__dmul_rn(top[k], gy), __dmul_rn(bot[k], fy));
        float* const orow = o + (int64_t)(oy0 + r) * ow + c0;
        if (vec) {
            *reinterpret_cast<float4*>(orow) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (c0 + k < cw) orow[k] = v[k];
        }
    }
}

__global__ void k_copy_f64_f32(const double* __restrict__ in, int64_t n, float* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (float)in[i];
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

// large maps: each of `parts` CTAs per image takes a band of interior rows;
// the band maxima are combined by a second kernel (max is order-free: exact)
__global__ void k_image_score_part(const double* __restrict__ scores, int h, int w, int border,
                                   int parts, double* __restrict__ part_max) {
    const int64_t b = blockIdx.x / parts;
    const int pi = blockIdx.x % parts;
    const double* p = scores + b * (int64_t)h * w;
    int bb = min(min(border, (h - 1) / 2), (w - 1) / 2);
    if (bb < 0) bb = 0;
    const int ih = h - 2 * bb, iw = w - 2 * bb;
    const int y0 = bb + (int)((int64_t)pi * ih / parts), y1 = bb + (int)((int64_t)(pi + 1) * ih / parts);
    double m = -INFINITY;
    for (int y = y0; y < y1; ++y) {
        const double* row = p + (int64_t)y * w + bb;
        for (int x = threadIdx.x; x < iw; x += blockDim.x) m = fmax(m, row[x]);
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
        if (lane == 0) part_max[blockIdx.x] = m;
    }
}

__global__ void k_image_score_combine(const double* __restrict__ part_max, int64_t images,
                                      int parts, double* __restrict__ image_score) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= images) return;
    double m = -INFINITY;
    for (int k = 0; k < parts; ++k) m = fmax(m, part_max[b * parts + k]);
    image_score[b] = m;
}

int launch_image_score(const double* scores, int64_t images, int h, int w, int border,
                       double* image_score, cudaStream_t st) {
    if (images <= 0 || h <= 0 || w <= 0) return QFCA_ERR_ARG;
    if ((int64_t)h * w > 65536 && images < 148) {
        // few large maps (an 8192^2 texture's 1024^2 map): split each over CTAs
        int bb = min(min(border, (h - 1) / 2), (w - 1) / 2);
        if (bb < 0) bb = 0;
        const int ih = h - 2 * bb;
        int parts = (int)((148 * 2 + images - 1) / images);
        parts = parts > ih ? ih : (parts < 1 ? 1 : parts);
        double* tmp = nullptr;
        keep_default_pool();
        if (cudaMallocAsync(&tmp, (size_t)images * parts * sizeof(double), st) != cudaSuccess)
            return QFCA_ERR_CUDA;
        k_image_score_part<<<(unsigned)(images * parts), 256, 0, st>>>(scores, h, w, border,
                                                                       parts, tmp);
        k_image_score_combine<<<(unsigned)((images + 127) / 128), 128, 0, st>>>(tmp, images,
                                                                                 parts, image_score);
        const bool ok = cudaGetLastError() == cudaSuccess;
        cudaFreeAsync(tmp, st);
        return ok ? QFCA_OK : QFCA_ERR_CUDA;
    }
    // one CTA per image
    const int threads = (int64_t)h * w > 65536 ? 1024 : 256;
    k_image_score<<<(unsigned)images, threads, 0, st>>>(scores, h, w, border, image_score);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_upsample(const double* in, int64_t images, int h, int w, int oh, int ow, float* out,
                    cudaStream_t st) {
    if (images <= 0 || h <= 0 || w <= 0 || oh <= 0 || ow <= 0) return QFCA_ERR_ARG;
    if (h == oh && w == ow) {
        k_copy_f64_f32<<<nblk(images * (int64_t)oh * ow, 256), 256, 0, st>>>(
            in, images * (int64_t)oh * ow, out);
    } else {
        const int bands = (oh + UP_ROWS - 1) / UP_ROWS;
        const int chunks = (ow + UP_CHUNK - 1) / UP_CHUNK;
        k_upsample<<<(unsigned)(images * bands * chunks), UP_THREADS, 0, st>>>(
            in, h, w, oh, ow, bands, chunks, out);
    }
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
