// quantize.cu -- K1 (per-plane min/max + finiteness) and K2 (bin indices).
//
// K1 restates quantize.py:61-68 (fit_quantizer) and the FeatureMap finiteness
// check (features.py:36-37); K2 restates quantize.py:71-82 (bin_indices) bit
// for bit: the fp64 expression is evaluated exactly as NumPy evaluates it.
// Both are streaming, HBM-bound passes: one CTA per plane for K1 (float4
// loads), a flat grid for K2 (float4 in, 4 bins out per thread).
#include "common.cuh"

namespace qfca {

constexpr int MINMAX_THREADS = 512;

__global__ void __launch_bounds__(MINMAX_THREADS)
k_minmax(const float* __restrict__ x, int64_t plane_len, float* __restrict__ lo,
         float* __restrict__ hi, int* __restrict__ nonfinite) {
    const int64_t plane = blockIdx.x;
    const float* p = x + plane * plane_len;
    float mn = INFINITY, mx = -INFINITY;
    bool bad = false;
    const bool vec = ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
    int64_t n4 = vec ? plane_len / 4 : 0;
    const float4* p4 = reinterpret_cast<const float4*>(p);
    for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) {
        float4 v = __ldg(p4 + i);
        mn = fminf(mn, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
        mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    }
    for (int64_t i = n4 * 4 + threadIdx.x; i < plane_len; i += blockDim.x) {
        float v = __ldg(p + i);
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
        bad |= !isfinite(v);
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    bad = __any_sync(0xffffffffu, bad);
    __shared__ float smn[32], smx[32];
    __shared__ int sbad;
    if (threadIdx.x == 0) sbad = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        smn[warp] = mn;
        smx[warp] = mx;
        if (bad) sbad = 1;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        mn = lane < nw ? smn[lane] : INFINITY;
        mx = lane < nw ? smx[lane] : -INFINITY;
        mn = warp_min(mn);
        mx = warp_max(mx);
        if (lane == 0) {
            lo[plane] = mn;
            hi[plane] = mx;
            if (sbad && nonfinite) atomicOr(nonfinite, 1);
        }
    }
}

template <typename BT>
__global__ void __launch_bounds__(256)
k_bin(const float* __restrict__ x, int64_t plane_len, int64_t blocks_per_plane,
      const float* __restrict__ lo, const float* __restrict__ hi, int n_bins,
      BT* __restrict__ out) {
    const int64_t plane = blockIdx.x / blocks_per_plane;
    const int64_t blk = blockIdx.x % blocks_per_plane;
    const double l = lo[plane], h = hi[plane];
    const bool degen = !(h > l);
    const double span = h - l;
    const double safe = span > 0 ? span : 1.0;
    const float* p = x + plane * plane_len;
    BT* o = out + plane * plane_len;
    const int64_t base = (blk * blockDim.x + threadIdx.x) * 4;
    if (base >= plane_len) return;
    if (base + 4 <= plane_len && ((reinterpret_cast<uintptr_t>(p + base) & 15) == 0)) {
        float4 v = __ldg(reinterpret_cast<const float4*>(p + base));
        int b0 = degen ? 0 : bin_of(v.x, l, safe, n_bins);
        int b1 = degen ? 0 : bin_of(v.y, l, safe, n_bins);
        int b2 = degen ? 0 : bin_of(v.z, l, safe, n_bins);
        int b3 = degen ? 0 : bin_of(v.w, l, safe, n_bins);
        o[base] = (BT)b0;
        o[base + 1] = (BT)b1;
        o[base + 2] = (BT)b2;
        o[base + 3] = (BT)b3;
    } else {
        for (int64_t i = base; i < base + 4 && i < plane_len; ++i)
            o[i] = (BT)(degen ? 0 : bin_of(__ldg(p + i), l, safe, n_bins));
    }
}

// per-plane mean in fp64 (pca_fit, features.py:170) -- one CTA per plane
__global__ void __launch_bounds__(256)
k_plane_mean(const float* __restrict__ x, int64_t plane_len, double* __restrict__ mean) {
    const int64_t plane = blockIdx.x;
    const float* p = x + plane * plane_len;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < plane_len; i += blockDim.x) s += (double)__ldg(p + i);
    s = warp_sum(s);
    __shared__ double sh[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[warp] = s;
    __syncthreads();
    if (warp == 0) {
        s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
        s = warp_sum(s);
        if (lane == 0) mean[plane] = s / (double)plane_len;
    }
}

int launch_minmax(const float* x, int64_t planes, int64_t plane_len, float* lo, float* hi,
                  int* nonfinite, cudaStream_t st) {
    if (planes <= 0 || plane_len <= 0) return QFCA_ERR_ARG;
    k_minmax<<<(unsigned)planes, MINMAX_THREADS, 0, st>>>(x, plane_len, lo, hi, nonfinite);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

// ---- threshold-table binning, bit-exact by construction:
// bin_of is monotone in v, so bin(v) = #{k >= 1 : v >= tau_k} with tau_k the
// smallest float32 whose fp64 bin is >= k.  One lane per threshold bisects the
// ordered float keys between lo and hi (exact bin_of at every probe); the
// element pass is then float compares only (no fp64 division per element).
constexpr int BT_MAXN = 64;  // thresholds held per plane in shared memory

__device__ __forceinline__ int fkey(float f) {
    const int k = __float_as_int(f);
    return k >= 0 ? k : k ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float fval(int key) {
    return __int_as_float(key >= 0 ? key : key ^ 0x7FFFFFFF);
}

// smallest float32 v with bin_of(v) >= k (lo < hi, 1 <= k <= n_bins - 1): start
// at the fp32 rounding of the exact boundary lo + k span / N (a few ulps off at
// most), walk a few ulps, fall back to bisection over the ordered keys
__device__ __forceinline__ float fq_threshold(int k, float lf, float hf, int n_bins) {
    const double l = lf, span = (double)hf - (double)lf;
    const int64_t klo = fkey(lf), khi = fkey(hf);
    int64_t key = fkey((float)(l + (double)k * span / (double)n_bins));
    key = key < klo + 1 ? klo + 1 : (key > khi ? khi : key);
    // invariant sought: bin(key) >= k > bin(key - 1)
    for (int it = 0; it < 6; ++it) {
        const bool ge = bin_of(fval((int)key), l, span, n_bins) >= k;
        if (ge) {
            if (key - 1 <= klo || bin_of(fval((int)(key - 1)), l, span, n_bins) < k)
                return fval((int)key);
            --key;
        } else {
            ++key;
        }
    }
    int64_t a = klo, b = khi;  // bin(a) = 0 < k <= n_bins - 1 = bin(b)
    while (b - a > 1) {
        const int64_t m = a + (b - a) / 2;
        if (bin_of(fval((int)m), l, span, n_bins) >= k) b = m; else a = m;
    }
    return fval((int)b);
}

__global__ void __launch_bounds__(128)
k_bin_thresholds(const float* __restrict__ lo, const float* __restrict__ hi, int64_t planes,
                 int n_bins, float* __restrict__ tau) {
    const int64_t plane = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (plane >= planes) return;
    const int lane = threadIdx.x & 31;
    const float lf = lo[plane], hf = hi[plane];
    for (int k = 1 + lane; k < n_bins; k += 32) {
        // degenerate channel: every bin is 0
        tau[plane * (n_bins - 1) + (k - 1)] = hf > lf ? fq_threshold(k, lf, hf, n_bins) : INFINITY;
    }
}

template <typename BT>
__global__ void __launch_bounds__(256)
k_bin_table(const float* __restrict__ x, int64_t plane_len, int splits,
            const float* __restrict__ lo, const float* __restrict__ hi,
            const float* __restrict__ tau, int n_bins, BT* __restrict__ out) {
    __shared__ float stp[BT_MAXN + 2];  // stp[k] = lower bound of bin k, +-inf sentinels
    // one CTA per plane (the setup is paid once), or per 1/splits of a large plane
    const int64_t plane = blockIdx.x / splits;
    const int part = blockIdx.x - (int)(plane * splits);
    const int nt = n_bins - 1;
    for (int k = threadIdx.x; k < nt; k += blockDim.x) stp[k + 1] = tau[plane * nt + k];
    if (threadIdx.x == 0) {
        stp[0] = -INFINITY;
        stp[n_bins] = INFINITY;
    }
    const float lf = lo[plane], hf = hi[plane];
    const float inv = hf > lf ? (float)((double)n_bins / ((double)hf - (double)lf)) : 0.f;
    const float top = (float)nt;
    __syncthreads();
    // this CTA's range of the plane (multiples of 4 elements)
    const int64_t q4 = (plane_len / 4 + splits - 1) / splits * 4;
    const int64_t b0_ = part * q4;
    const int64_t len = splits == 1 ? plane_len : max((int64_t)0, min(q4, plane_len - b0_));
    const float* p = x + plane * plane_len + b0_;
    BT* o = out + plane * plane_len + b0_;
    // fp32 estimate (within one bin of the exact fp64 rule), then one branch-free
    // correction each way against the thresholds (bin k starts at stp[k])
    auto bin = [&](float v) {
        int b = (int)fminf(fmaxf((v - lf) * inv, 0.f), top);  // NaN -> 0
        b = min(b + ((v >= stp[b + 1]) ? 1 : 0), nt);  // (+inf input: stays at nt)
        b -= (v < stp[b]) ? 1 : 0;
        return b;
    };
    const bool vec = (reinterpret_cast<uintptr_t>(p) & 15) == 0 &&
                     (sizeof(BT) == 2 || (reinterpret_cast<uintptr_t>(o) & 3) == 0);
    const int64_t n4 = vec ? len / 4 : 0;
    for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p) + i);
        const int b0 = bin(v.x), b1 = bin(v.y), b2 = bin(v.z), b3 = bin(v.w);
        if (sizeof(BT) == 1) {
            reinterpret_cast<uint32_t*>(o)[i] =
                (uint32_t)b0 | ((uint32_t)b1 << 8) | ((uint32_t)b2 << 16) | ((uint32_t)b3 << 24);
        } else {
            reinterpret_cast<uint2*>(o)[i] =
                make_uint2((uint32_t)b0 | ((uint32_t)b1 << 16), (uint32_t)b2 | ((uint32_t)b3 << 16));
        }
    }
    for (int64_t i = 4 * n4 + threadIdx.x; i < len; i += blockDim.x)
        o[i] = (BT)bin(__ldg(p + i));
}

// ---- fused K1 + K2 for planes that fit in shared memory (one CTA per plane):
// the plane is read from HBM once (min/max + finiteness from the staged copy,
// thresholds, bins) instead of twice.  Thresholds as k_bin_thresholds (the
// smallest float32 whose fp64 bin is >= k), one thread per threshold, started
// at the rounded exact boundary and corrected by a few ulps (instead of ~31
// serial bisection probes).  Bit-identical to K1 + K2.
constexpr int FQ_MAXLEN = 16384;  // 64 KB of fp32 staged per plane

template <typename BT, int FQ_THREADS>
__global__ void __launch_bounds__(FQ_THREADS)
k_quantize_plane(const float* __restrict__ x, int plane_len, int n_bins, float* __restrict__ lo,
                 float* __restrict__ hi, int* __restrict__ nonfinite, BT* __restrict__ out) {
    extern __shared__ __align__(16) float fq_x[];  // [plane_len]
    __shared__ float st[BT_MAXN + 2];
    __shared__ float smn[FQ_THREADS / 32], smx[FQ_THREADS / 32];
    __shared__ int sbad;
    const int64_t plane = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float4* p4 = reinterpret_cast<const float4*>(x + plane * plane_len);
    float mn = INFINITY, mx = -INFINITY;
    float nf = 0.f;  // v * 0 is NaN exactly for inf / NaN v: one FMA per value
    if (tid == 0) sbad = 0;
#pragma unroll 4
    for (int i = tid; i < plane_len / 4; i += FQ_THREADS) {
        const float4 v = __ldg(p4 + i);
        reinterpret_cast<float4*>(fq_x)[i] = v;
        mn = fminf(mn, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
        mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        nf = fmaf(v.x, 0.f, fmaf(v.y, 0.f, fmaf(v.z, 0.f, fmaf(v.w, 0.f, nf))));
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    const bool bad = __any_sync(0xffffffffu, nf != nf);
    __syncthreads();
    if (lane == 0) {
        smn[warp] = mn;
        smx[warp] = mx;
        if (bad) sbad = 1;
    }
    __syncthreads();
    mn = smn[0];
    mx = smx[0];
#pragma unroll
    for (int w = 1; w < FQ_THREADS / 32; ++w) {
        mn = fminf(mn, smn[w]);
        mx = fmaxf(mx, smx[w]);
    }
    if (tid == 0) {
        lo[plane] = mn;
        hi[plane] = mx;
        if (sbad && nonfinite) atomicOr(nonfinite, 1);
    }
    const int nt = n_bins - 1;
    // stp[k] = lower bound of bin k (stp[0] = -inf, stp[N] = +inf sentinels)
    float* const stp = st;
    for (int k = 1 + tid; k <= nt; k += FQ_THREADS)
        stp[k] = mx > mn ? fq_threshold(k, mn, mx, n_bins) : INFINITY;
    if (tid == 0) {
        stp[0] = -INFINITY;
        stp[n_bins] = INFINITY;
    }
    const float inv = mx > mn ? (float)((double)n_bins / ((double)mx - (double)mn)) : 0.f;
    const float top = (float)nt;
    __syncthreads();
    // the fp32 estimate is within one bin of the exact fp64 rule (its relative
    // error is a few ulps, N * 1e-7 bins): one branch-free correction each way
    auto bin = [&](float v) {
        int b = (int)fminf(fmaxf((v - mn) * inv, 0.f), top);  // NaN -> 0
        b = min(b + ((v >= stp[b + 1]) ? 1 : 0), nt);  // (+inf input: stays at nt)
        b -= (v < stp[b]) ? 1 : 0;
        return b;
    };
    BT* o = out + plane * plane_len;
    for (int i = tid; i < plane_len / 4; i += FQ_THREADS) {
        const float4 v = reinterpret_cast<const float4*>(fq_x)[i];
        const int b0 = bin(v.x), b1 = bin(v.y), b2 = bin(v.z), b3 = bin(v.w);
        if (sizeof(BT) == 1) {
            reinterpret_cast<uint32_t*>(o)[i] =
                (uint32_t)b0 | ((uint32_t)b1 << 8) | ((uint32_t)b2 << 16) | ((uint32_t)b3 << 24);
        } else {
            reinterpret_cast<uint2*>(o)[i] =
                make_uint2((uint32_t)b0 | ((uint32_t)b1 << 16), (uint32_t)b2 | ((uint32_t)b3 << 16));
        }
    }
}

// K1 + K2 in one pass when the planes fit; QFCA_ERR_UNSUPPORTED otherwise (the
// caller then runs launch_minmax + launch_bin)
int launch_quantize_fused(const float* x, int64_t planes, int64_t plane_len, int n_bins,
                          float* lo, float* hi, int* nonfinite, void* out, int out_bytes,
                          cudaStream_t st) {
    if (planes <= 0 || plane_len <= 0 || n_bins < 1) return QFCA_ERR_ARG;
    if (plane_len > FQ_MAXLEN || plane_len % 4 || n_bins < 2 || n_bins > BT_MAXN + 1 ||
        (out_bytes != 1 && out_bytes != 2) || planes > 0x7fffffffLL ||
        (reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(out) & 7))
        return QFCA_ERR_UNSUPPORTED;
    const size_t smem = (size_t)plane_len * sizeof(float);
    // large planes (few CTAs per SM by shared memory) get more threads in flight
    auto go = [&](auto kern, int threads, auto* o) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return QFCA_ERR_CUDA;
        kern<<<(unsigned)planes, threads, smem, st>>>(x, (int)plane_len, n_bins, lo, hi,
                                                      nonfinite, o);
        return QFCA_OK;
    };
    int rc;
    const bool big = false;  // (1024 threads measured slower on 128^2 planes: 1.44 vs 1.13 ms)
    // 64^2 planes: 128 threads (more, shorter CTAs per SM: 0.197 -> 0.149 ms per
    // 64 x 512 planes); 128^2: 256 (128 and 512 measured slower)
    const bool small = plane_len <= 4096;
    if (out_bytes == 1 && small)
        rc = go(k_quantize_plane<uint8_t, 128>, 128, (uint8_t*)out);
    else if (out_bytes == 1)
        rc = big ? go(k_quantize_plane<uint8_t, 1024>, 1024, (uint8_t*)out)
                 : go(k_quantize_plane<uint8_t, 256>, 256, (uint8_t*)out);
    else
        rc = big ? go(k_quantize_plane<uint16_t, 1024>, 1024, (uint16_t*)out)
                 : go(k_quantize_plane<uint16_t, 256>, 256, (uint16_t*)out);
    if (rc != QFCA_OK) return rc;
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_bin(const float* x, int64_t planes, int64_t plane_len, const float* lo,
               const float* hi, int n_bins, void* out, int out_bytes, cudaStream_t st) {
    if (planes <= 0 || plane_len <= 0 || n_bins < 1) return QFCA_ERR_ARG;
    const int64_t per = 256 * 4;
    const int64_t bpp = (plane_len + per - 1) / per;
    const int64_t grid = bpp * planes;
    if (grid > 0x7fffffffLL) return QFCA_ERR_ARG;
    if (n_bins >= 2 && n_bins <= BT_MAXN + 1 && (out_bytes == 1 || out_bytes == 2)) {
        // thresholds in a stream-ordered scratch allocation
        float* tau = nullptr;
        keep_default_pool();
        if (cudaMallocAsync(&tau, (size_t)planes * (n_bins - 1) * sizeof(float), st) !=
            cudaSuccess)
            return QFCA_ERR_CUDA;
        k_bin_thresholds<<<(unsigned)((planes + 3) / 4), 128, 0, st>>>(lo, hi, planes, n_bins, tau);
        // large planes (few of them) split so the grid fills the GPU; the vector
        // path needs every part to start on a 4-element boundary (plane_len % 4)
        const int splits = (plane_len % 4 == 0 && plane_len >= (1 << 17))
                               ? (int)min((int64_t)64, plane_len / (1 << 16)) : 1;
        const unsigned g2 = (unsigned)(planes * splits);
        if (out_bytes == 1)
            k_bin_table<uint8_t><<<g2, 256, 0, st>>>(x, plane_len, splits, lo, hi, tau, n_bins,
                                                     (uint8_t*)out);
        else
            k_bin_table<uint16_t><<<g2, 256, 0, st>>>(x, plane_len, splits, lo, hi, tau, n_bins,
                                                      (uint16_t*)out);
        const bool ok = cudaGetLastError() == cudaSuccess;
        cudaFreeAsync(tau, st);
        return ok ? QFCA_OK : QFCA_ERR_CUDA;
    }
    if (out_bytes == 1) {
        if (n_bins > 256) return QFCA_ERR_ARG;
        k_bin<uint8_t><<<(unsigned)grid, 256, 0, st>>>(x, plane_len, bpp, lo, hi, n_bins,
                                                        (uint8_t*)out);
    } else if (out_bytes == 2) {
        if (n_bins > 65536) return QFCA_ERR_ARG;
        k_bin<uint16_t><<<(unsigned)grid, 256, 0, st>>>(x, plane_len, bpp, lo, hi, n_bins,
                                                         (uint16_t*)out);
    } else if (out_bytes == 4) {
        k_bin<int32_t><<<(unsigned)grid, 256, 0, st>>>(x, plane_len, bpp, lo, hi, n_bins,
                                                        (int32_t*)out);
    } else {
        return QFCA_ERR_ARG;
    }
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_plane_mean(const float* x, int64_t planes, int64_t plane_len, double* mean,
                      cudaStream_t st) {
    if (planes <= 0 || plane_len <= 0) return QFCA_ERR_ARG;
    k_plane_mean<<<(unsigned)planes, 256, 0, st>>>(x, plane_len, mean);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
