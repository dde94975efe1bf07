// pooling.cu -- the reference's box-pooling API on the GPU (pooling.py:20-172).
//
// The scoring path never materialises these (the fused kernel slides window
// counts in registers / shared memory); they back the public pooling API with
// the reference's exact arithmetic:
//   * k_pad_planes      pad_plane (pooling.py:20-38) / np.pad: pure data
//                       movement, any element size (1 / 2 / 4 / 8 bytes);
//   * k_sat_cols,
//     k_sat_rows        build_sat (pooling.py:56-64) and the SAT inside
//                       box_average_stack (pooling.py:144-147): the padded
//                       plane converted to fp64, cumsum down the rows, then
//                       across the columns -- each a sequential scan, one
//                       thread per column / row, so every partial sum is the
//                       one np.cumsum forms (bit-identical);
//   * k_sat_box         the four-corner window sums of _box_sum_map /
//                       box_average_stack (pooling.py:97-117, 148-158),
//                       ((c11 - c01) - c10) + c00, then / k^2 (IEEE);
//   * k_sat_rects       box_sum (pooling.py:71-94) for a list of rectangles;
//   * k_naive_box       naive_box_average (pooling.py:161-172): the k^2 shifted
//                       planes added in (dy, dx) order, then / k^2.
// Pad codes: 0 zero, 1 reflect, 2 wrap, 3 edge (np.pad 'edge', which
// pad_plane switches to when an axis has length 1, pooling.py:31-35).
#include "common.cuh"

namespace qfca {

constexpr int PAD_EDGE = 3;

// source index of padded coordinate c along an axis of length n (np.pad
// semantics of the given mode; reflect repeats for large margins, a length-1
// axis reflects to its single element)
__device__ __forceinline__ int np_pad_index(int c, int n, int mode) {
    if (c >= 0 && c < n) return c;
    if (mode == QFCA_PAD_ZERO) return -1;
    if (mode == PAD_EDGE) return c < 0 ? 0 : n - 1;
    return map_coord(c, n, mode);
}

template <typename T>
__device__ __forceinline__ double as_f64(const void* p, int64_t i) {
    return (double)reinterpret_cast<const T*>(p)[i];
}

// dtype codes: 0 f32, 1 f64, 2 u8, 3 i32, 4 i64, 5 i16, 6 u16, 7 bool(u8)
__device__ __forceinline__ double load_f64(const void* p, int dtype, int64_t i) {
    switch (dtype) {
        case 0: return as_f64<float>(p, i);
        case 1: return as_f64<double>(p, i);
        case 2: case 7: return as_f64<uint8_t>(p, i);
        case 3: return as_f64<int32_t>(p, i);
        case 4: return as_f64<long long>(p, i);
        case 5: return as_f64<int16_t>(p, i);
        default: return as_f64<uint16_t>(p, i);
    }
}

__global__ void k_pad_planes(const uint8_t* __restrict__ x, int64_t planes, int h, int w,
                             int margin, int mode_r, int mode_c, int es, uint8_t* __restrict__ out) {
    const int H = h + 2 * margin, W = w + 2 * margin;
    const int64_t n = planes * H * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / ((int64_t)H * W);
        const int rem = (int)(i - p * H * W);
        const int yy = rem / W, xx = rem - yy * W;
        const int sy = np_pad_index(yy - margin, h, mode_r);
        const int sx = np_pad_index(xx - margin, w, mode_c);
        uint8_t* d = out + i * es;
        if (sy < 0 || sx < 0) {
            for (int b = 0; b < es; ++b) d[b] = 0;
        } else {
            const uint8_t* s = x + ((p * h + sy) * (int64_t)w + sx) * es;
            for (int b = 0; b < es; ++b) d[b] = s[b];
        }
    }
}

// cs (planes, H + 1, W + 1): row 0 and column 0 zero; cs[i+1][j+1] =
// sum over rows <= i of padded[.][j] (the axis-0 cumsum), one thread per column
__global__ void k_sat_cols(const void* __restrict__ x, int dtype, int64_t planes, int h, int w,
                           int margin, int mode_r, int mode_c, double* __restrict__ cs) {
    const int H = h + 2 * margin, W = w + 2 * margin;
    const int64_t n = planes * (W + 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / (W + 1);
        const int j = (int)(i - p * (W + 1));
        double* col = cs + p * (int64_t)(H + 1) * (W + 1) + j;
        col[0] = 0.0;
        if (j == 0) {
            for (int r = 1; r <= H; ++r) col[(int64_t)r * (W + 1)] = 0.0;
            continue;
        }
        const int sx = np_pad_index(j - 1 - margin, w, mode_c);
        double acc = 0.0;
        for (int r = 0; r < H; ++r) {
            const int sy = np_pad_index(r - margin, h, mode_r);
            const double v = (sy < 0 || sx < 0) ? 0.0
                                                : load_f64(x, dtype, (p * h + sy) * (int64_t)w + sx);
            acc = __dadd_rn(acc, v);
            col[(int64_t)(r + 1) * (W + 1)] = acc;
        }
    }
}

// the axis-1 cumsum over each row of cs (columns 1..W), one thread per row
__global__ void k_sat_rows(int64_t planes, int H, int W, double* __restrict__ cs) {
    const int64_t n = planes * H;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / H;
        const int r = (int)(i - p * H) + 1;
        double* row = cs + (p * (int64_t)(H + 1) + r) * (W + 1);
        double acc = row[1];
        for (int j = 2; j <= W; ++j) {
            acc = __dadd_rn(acc, row[j]);
            row[j] = acc;
        }
    }
}

// window sums at every pixel from the SAT; clamp = 1: zero padding (rectangle
// clamped to the plane, SAT without margin), else the SAT carries margin k/2
__global__ void k_sat_box(const double* __restrict__ cs, int64_t planes, int h, int w, int k,
                          int clamp, double div, double* __restrict__ out) {
    const int r = k / 2;
    const int W1 = clamp ? w + 1 : w + 2 * r + 1;
    const int H1 = clamp ? h + 1 : h + 2 * r + 1;
    const int64_t n = planes * h * w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / ((int64_t)h * w);
        const int rem = (int)(i - p * h * w);
        const int y = rem / w, x = rem - y * w;
        int r0, r1, c0, c1;
        if (clamp) {
            r0 = max(y - r, 0); r1 = min(y + r + 1, h);
            c0 = max(x - r, 0); c1 = min(x + r + 1, w);
        } else {
            r0 = y; r1 = y + k; c0 = x; c1 = x + k;
        }
        const double* c = cs + p * (int64_t)H1 * W1;
        double s = __dsub_rn(c[(int64_t)r1 * W1 + c1], c[(int64_t)r0 * W1 + c1]);
        s = __dsub_rn(s, c[(int64_t)r1 * W1 + c0]);
        s = __dadd_rn(s, c[(int64_t)r0 * W1 + c0]);
        out[i] = div > 0.0 ? __ddiv_rn(s, div) : s;
    }
}

// rects (n, 4) int32 = (r0, r1, c0, c1) in SAT coordinates of one plane
__global__ void k_sat_rects(const double* __restrict__ cs, int W1, const int32_t* __restrict__ rects,
                            int64_t n, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int r0 = rects[4 * i], r1 = rects[4 * i + 1], c0 = rects[4 * i + 2],
                  c1 = rects[4 * i + 3];
        double s = __dsub_rn(cs[(int64_t)r1 * W1 + c1], cs[(int64_t)r0 * W1 + c1]);
        s = __dsub_rn(s, cs[(int64_t)r1 * W1 + c0]);
        out[i] = __dadd_rn(s, cs[(int64_t)r0 * W1 + c0]);
    }
}

__global__ void k_naive_box(const void* __restrict__ x, int dtype, int64_t planes, int h, int w,
                            int k, int mode_r, int mode_c, double* __restrict__ out) {
    const int r = k / 2;
    const int64_t n = planes * h * w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / ((int64_t)h * w);
        const int rem = (int)(i - p * h * w);
        const int y = rem / w, xx = rem - y * w;
        double acc = 0.0;
        for (int dy = 0; dy < k; ++dy) {
            const int sy = np_pad_index(y + dy - r, h, mode_r);
            for (int dx = 0; dx < k; ++dx) {
                const int sx = np_pad_index(xx + dx - r, w, mode_c);
                const double v = (sy < 0 || sx < 0)
                                     ? 0.0 : load_f64(x, dtype, (p * h + sy) * (int64_t)w + sx);
                acc = __dadd_rn(acc, v);
            }
        }
        out[i] = __ddiv_rn(acc, (double)k * (double)k);
    }
}

static unsigned grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 32) g = 148 * 32;
    return (unsigned)(g < 1 ? 1 : g);
}

static bool mode_ok(int m) { return m >= 0 && m <= PAD_EDGE; }

int launch_pad_planes(const void* x, int64_t planes, int h, int w, int margin, int mode_r,
                      int mode_c, int elem_bytes, void* out, cudaStream_t st) {
    if (!x || !out || planes < 0 || h < 1 || w < 1 || margin < 0 || !mode_ok(mode_r) ||
        !mode_ok(mode_c) || !(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 ||
                              elem_bytes == 8))
        return QFCA_ERR_ARG;
    const int64_t n = planes * (h + 2 * margin) * (int64_t)(w + 2 * margin);
    if (n == 0) return QFCA_OK;
    k_pad_planes<<<grid_for(n), 256, 0, st>>>((const uint8_t*)x, planes, h, w, margin, mode_r,
                                              mode_c, elem_bytes, (uint8_t*)out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_build_sat(const void* x, int dtype, int64_t planes, int h, int w, int margin,
                     int mode_r, int mode_c, double* cs, cudaStream_t st) {
    if (!x || !cs || planes < 0 || h < 1 || w < 1 || margin < 0 || dtype < 0 || dtype > 7 ||
        !mode_ok(mode_r) || !mode_ok(mode_c))
        return QFCA_ERR_ARG;
    if (planes == 0) return QFCA_OK;
    const int H = h + 2 * margin, W = w + 2 * margin;
    k_sat_cols<<<grid_for(planes * (W + 1)), 128, 0, st>>>(x, dtype, planes, h, w, margin, mode_r,
                                                           mode_c, cs);
    if (cudaGetLastError() != cudaSuccess) return QFCA_ERR_CUDA;
    k_sat_rows<<<grid_for(planes * H), 128, 0, st>>>(planes, H, W, cs);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_sat_box(const double* cs, int64_t planes, int h, int w, int k, int clamp, double div,
                   double* out, cudaStream_t st) {
    if (!cs || !out || planes < 0 || h < 1 || w < 1 || k < 1 || (k & 1) == 0) return QFCA_ERR_ARG;
    const int64_t n = planes * h * (int64_t)w;
    if (n == 0) return QFCA_OK;
    k_sat_box<<<grid_for(n), 256, 0, st>>>(cs, planes, h, w, k, clamp, div, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_sat_rects(const double* cs, int W1, const int32_t* rects, int64_t n, double* out,
                     cudaStream_t st) {
    if (!cs || !rects || !out || W1 < 1 || n < 0) return QFCA_ERR_ARG;
    if (n == 0) return QFCA_OK;
    k_sat_rects<<<grid_for(n), 256, 0, st>>>(cs, W1, rects, n, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_naive_box(const void* x, int dtype, int64_t planes, int h, int w, int k, int mode_r,
                     int mode_c, double* out, cudaStream_t st) {
    if (!x || !out || planes < 0 || h < 1 || w < 1 || k < 1 || (k & 1) == 0 || dtype < 0 ||
        dtype > 7 || !mode_ok(mode_r) || !mode_ok(mode_c))
        return QFCA_ERR_ARG;
    const int64_t n = planes * h * (int64_t)w;
    if (n == 0) return QFCA_OK;
    k_naive_box<<<grid_for(n), 256, 0, st>>>(x, dtype, planes, h, w, k, mode_r, mode_c, out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
