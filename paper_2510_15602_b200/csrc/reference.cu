// reference.cu -- K3: sort-free global reference histogram (select_reference).
//
// Restates quantize.py:150-200.  The reference samples T x T patches on a
// stride grid (quantize.py:109-132), sorts every patch, takes the per-rank
// lower median over the samples and bins it (median-quan).  Binning is
// monotone, so the bin of the per-rank median equals the per-rank median of
// bins, and with A_i(s) = #{values of patch s in bins <= i}:
//
//     J_r <= i  <=>  #{s : A_i(s) > r} >= m + 1,   m = (S - 1) / 2
//
// so with V_i := the (S-1-m)-th smallest A_i(s) (0-based), the reference bin
// of rank r is J_r = min{i : V_i > r} and the reference counts are exactly
// R_i = V_i - V_{i-1}.  No float sort, no per-sample vectors: one order
// statistic per bin over small integers, found by binary search with packed
// SIMD compares.  quan-median / quan-mean (quantize.py:184-199) are per-bin
// lower median / sum of the window counts P_i(s) over the samples.
//
// Window counts at the sample points come from packed-lane column counts
// (vertical sliding between consecutive sample rows) and a modular 32-bit
// prefix scan along each row (window count = prefix difference; exact because
// every lane's true window count is < 2^lane_bits).
#include "common.cuh"

namespace qfca {

constexpr int REF_THREADS = 256;
constexpr int REF_NW = 5;  // 4 packed count words + 1 "below chunk" word

struct RefGeom {
    int h, w, t, r, wp, stride, ny, nx, S, G;
    int stage;  // 1: the plane's bins are staged in shared memory first
    int compact;  // 1 (stride >= t): only the sample windows' columns are counted,
                  // wp = nx * t of them, column q = padded (q / t) * stride + q % t
};

template <int LANE>
__device__ __forceinline__ void onehot_words(int b, int i0, uint32_t (&add)[REF_NW]) {
    constexpr int L = 32 / LANE;        // bins per word
    constexpr int NBC = 4 * L;          // bins per chunk
    const int rel = b - i0;
    const bool in = (unsigned)rel < (unsigned)NBC;
    const int word = rel / L;
    const uint32_t bit = 1u << ((rel - word * L) * LANE);
#pragma unroll
    for (int k = 0; k < 4; ++k) add[k] = (in && word == k) ? bit : 0u;
    add[4] = rel < 0 ? 1u : 0u;
}

// packed "how many lanes <= v" for the sample store (u8 lanes need values and
// v <= 127, u16 lanes <= 32767)
template <typename ST>
__device__ __forceinline__ int count_le(uint32_t word, int v);
template <>
__device__ __forceinline__ int count_le<uint8_t>(uint32_t word, int v) {
    return __popc(((0x80808080u | ((uint32_t)v * 0x01010101u)) - word) & 0x80808080u);
}
template <>
__device__ __forceinline__ int count_le<uint16_t>(uint32_t word, int v) {
    return __popc(((0x80008000u | ((uint32_t)v * 0x00010001u)) - word) & 0x80008000u);
}

template <typename BT, int LANE, typename ST>
__global__ void __launch_bounds__(REF_THREADS)
k_reference(const BT* __restrict__ bins, const float* __restrict__ lo,
            const float* __restrict__ hi, RefGeom g, int n_bins, int pad, int mode,
            int32_t* __restrict__ stats) {
    constexpr int L = 32 / LANE;
    constexpr int NBC = 4 * L;
    constexpr uint32_t LMASK = (LANE == 32) ? 0xffffffffu : ((1u << LANE) - 1u);
    extern __shared__ __align__(16) uint8_t smem[];
    const int plane = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = REF_THREADS / 32;
    const int t2 = g.t * g.t;
    int32_t* out = stats + (int64_t)plane * n_bins;

    const double l = lo[plane], hh = hi[plane];
    if (!(hh > l)) {  // degenerate channel (quantize.py:169-171)
        for (int i = tid; i < n_bins; i += REF_THREADS)
            out[i] = mode == 0 ? t2 : (i == 0 ? (mode == 3 ? t2 * g.S : t2) : 0);
        return;
    }
    const BT* bp = bins + (int64_t)plane * g.h * g.w;
    const bool edge = pad == QFCA_PAD_REFLECT && !(g.h > 1 && g.w > 1);
    // zero padding contributes literal 0.0 values (np.pad constant), binned
    const int bzero = bin_of(0.0f, l, hh - l, n_bins);

    // shared memory carve-up
    const int srow = (g.S + 3) & ~3;               // sample row length (padded)
    ST* SA = reinterpret_cast<ST*>(smem);          // [NBC][srow]
    size_t off = ((size_t)NBC * srow * sizeof(ST) + 15) & ~(size_t)15;
    uint32_t* state = reinterpret_cast<uint32_t*>(smem + off);   // [NW][wp]
    off += (size_t)REF_NW * g.wp * 4;
    uint32_t* CC = reinterpret_cast<uint32_t*>(smem + off);      // [G][NW][wp]
    off += (size_t)g.G * REF_NW * g.wp * 4;
    uint32_t* WS = reinterpret_cast<uint32_t*>(smem + off);      // [G][NW][nx]
    off += (size_t)g.G * REF_NW * g.nx * 4;
    if (g.stage) {  // one coalesced read of the plane; the window sweeps then hit smem
        BT* sbins = reinterpret_cast<BT*>(smem + ((off + 15) & ~(size_t)15));
        const int64_t n = (int64_t)g.h * g.w;
        if ((n * (int64_t)sizeof(BT)) % 16 == 0 && (reinterpret_cast<uintptr_t>(bp) & 15) == 0) {
            for (int64_t i = tid; i < n * (int64_t)sizeof(BT) / 16; i += REF_THREADS)
                reinterpret_cast<uint4*>(sbins)[i] = __ldg(reinterpret_cast<const uint4*>(bp) + i);
        } else {
            for (int64_t i = tid; i < n; i += REF_THREADS) sbins[i] = bp[i];
        }
        bp = sbins;
        __syncthreads();
    }

    for (int i0 = 0; i0 < n_bins; i0 += NBC) {
        const int nb = min(NBC, n_bins - i0);
        for (int j0 = 0; j0 < g.ny; j0 += g.G) {
            const int gn = min(g.G, g.ny - j0);
            // ---- vertical: packed column counts of each sample row's window
            for (int xp = tid; xp < g.wp; xp += REF_THREADS) {
                const int xpad = g.compact ? (xp / g.t) * g.stride + xp % g.t : xp;
                const int xx = pad_plane_index(xpad - g.r, g.w, pad, edge);
                uint32_t st[REF_NW];
#pragma unroll
                for (int k = 0; k < REF_NW; ++k) st[k] = j0 == 0 ? 0u : state[k * g.wp + xp];
                for (int gi = 0; gi < gn; ++gi) {
                    const int j = j0 + gi;
                    const int ys = j * g.stride;  // padded window rows [ys, ys + t)
                    auto row_bin = [&](int prow) -> int {
                        const int yy = pad_plane_index(prow - g.r, g.h, pad, edge);
                        return (yy < 0 || xx < 0) ? bzero : (int)bp[(int64_t)yy * g.w + xx];
                    };
                    if (j == 0 || g.stride >= g.t) {
#pragma unroll
                        for (int k = 0; k < REF_NW; ++k) st[k] = 0u;
                        // the window's rows in batches of 8 independent loads (one
                        // memory latency per batch instead of one per row)
                        for (int d0 = 0; d0 < g.t; d0 += 8) {
                            int bv[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q) bv[q] = d0 + q < g.t ? row_bin(ys + d0 + q) : -1;
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                if (bv[q] < 0) continue;
                                uint32_t a[REF_NW];
                                onehot_words<LANE>(bv[q], i0, a);
#pragma unroll
                                for (int k = 0; k < REF_NW; ++k) st[k] += a[k];
                            }
                        }
                    } else {
                        for (int d = 0; d < g.stride; ++d) {
                            uint32_t a[REF_NW], s_[REF_NW];
                            onehot_words<LANE>(row_bin(ys - g.stride + d), i0, s_);
                            onehot_words<LANE>(row_bin(ys - g.stride + g.t + d), i0, a);
#pragma unroll
                            for (int k = 0; k < REF_NW; ++k) st[k] += a[k] - s_[k];
                        }
                    }
#pragma unroll
                    for (int k = 0; k < REF_NW; ++k) CC[((size_t)gi * REF_NW + k) * g.wp + xp] = st[k];
                }
#pragma unroll
                for (int k = 0; k < REF_NW; ++k) state[k * g.wp + xp] = st[k];
            }
            __syncthreads();
            // ---- horizontal: modular inclusive prefix along each (row, word)
            for (int row = warp; row < gn * REF_NW; row += nwarps) {
                uint32_t* rp = CC + (size_t)row * g.wp;
                uint32_t carry = 0;
                for (int base = 0; base < g.wp; base += 32) {
                    const int xp = base + lane;
                    uint32_t v = xp < g.wp ? rp[xp] : 0u;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
                        if (lane >= o) v += u;
                    }
                    v += carry;
                    if (xp < g.wp) rp[xp] = v;
                    carry = __shfl_sync(0xffffffffu, v, 31);
                }
            }
            __syncthreads();
            // ---- window words at the sample columns
            for (int task = tid; task < gn * REF_NW * g.nx; task += REF_THREADS) {
                const int jx = task % g.nx;
                const int row = task / g.nx;  // gi * NW + k
                const uint32_t* rp = CC + (size_t)row * g.wp;
                const int xs = jx * (g.compact ? g.t : g.stride);  // window cols [xs, xs + t)
                WS[(size_t)row * g.nx + jx] = rp[xs + g.t - 1] - (xs > 0 ? rp[xs - 1] : 0u);
            }
            __syncthreads();
            // ---- per sample: cumulative (median-quan) or raw (quan-*) counts
            for (int task = tid; task < gn * g.nx; task += REF_THREADS) {
                const int jx = task % g.nx, gi = task / g.nx;
                const int s = (j0 + gi) * g.nx + jx;
                uint32_t acc = WS[((size_t)gi * REF_NW + 4) * g.nx + jx];  // below chunk
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t word = WS[((size_t)gi * REF_NW + k) * g.nx + jx];
#pragma unroll
                    for (int q = 0; q < L; ++q) {
                        const int bi = k * L + q;
                        const uint32_t cnt = (word >> (q * LANE)) & LMASK;
                        acc += cnt;
                        if (bi < nb) SA[(size_t)bi * srow + s] = (ST)(mode == 0 ? acc : cnt);
                    }
                }
            }
            __syncthreads();
        }
        // pad the sample rows so packed compares see values > any query
        for (int idx = tid; idx < nb * (srow - g.S); idx += REF_THREADS) {
            const int bi = idx / (srow - g.S), s = g.S + idx % (srow - g.S);
            SA[(size_t)bi * srow + s] = (ST)(sizeof(ST) == 1 ? 127 : 32767);
        }
        __syncthreads();
        // ---- selection: one warp per bin
        const int m = (g.S - 1) / 2;
        const int words = srow * (int)sizeof(ST) / 4;
        for (int bi = warp; bi < nb; bi += nwarps) {
            const uint32_t* row = reinterpret_cast<const uint32_t*>(SA + (size_t)bi * srow);
            int result;
            if (mode == 3) {  // quan-mean: integer sum of P_i(s)
                int s_ = 0;
                for (int idx = lane; idx < g.S; idx += 32) s_ += (int)SA[(size_t)bi * srow + idx];
                result = warp_sum_i(s_);
            } else {
                // smallest v with #{A <= v} >= c0
                const int c0 = mode == 0 ? g.S - m : m + 1;
                int a = 0, b = t2;
                while (a < b) {
                    const int mid = (a + b) >> 1;
                    int c = 0;
                    for (int wi = lane; wi < words; wi += 32) c += count_le<ST>(row[wi], mid);
                    c = warp_sum_i(c);
                    if (c >= c0) b = mid; else a = mid + 1;
                }
                result = a;
            }
            if (lane == 0) out[i0 + bi] = result;
        }
        __syncthreads();
    }
}

static size_t ref_smem_bytes(const RefGeom& g, int st_bytes, int nbc, int bt_bytes) {
    const int srow = (g.S + 3) & ~3;
    size_t off = ((size_t)nbc * srow * st_bytes + 15) & ~(size_t)15;
    off += (size_t)REF_NW * g.wp * 4;
    off += (size_t)g.G * REF_NW * g.wp * 4;
    off += (size_t)g.G * REF_NW * g.nx * 4;
    if (g.stage) off = ((off + 15) & ~(size_t)15) + (size_t)g.h * g.w * bt_bytes;
    return off;
}

int sample_stride(int h, int w, int budget) {
    int s = 1;
    while ((int64_t)((h + s - 1) / s) * (int64_t)((w + s - 1) / s) > budget) ++s;
    return s;
}

template <typename BT>
static int launch_reference_t(const BT* bins, const float* lo, const float* hi, int64_t planes,
                              int h, int w, int n_bins, int t, int pad, int budget, int mode,
                              int32_t* stats, cudaStream_t st) {
    RefGeom g;
    g.h = h; g.w = w; g.t = t; g.r = t / 2; g.wp = w + 2 * g.r;
    g.stride = sample_stride(h, w, budget);
    g.ny = (h + g.stride - 1) / g.stride;
    g.nx = (w + g.stride - 1) / g.stride;
    g.compact = g.stride >= t ? 1 : 0;
    if (g.compact) g.wp = g.nx * t;  // the sample windows' columns only
    g.S = g.ny * g.nx;
    const int t2 = t * t;
    if (t2 > 32767) return QFCA_ERR_UNSUPPORTED;
    const bool lane8 = t2 <= 255;
    const bool st8 = t2 <= 126;
    const int nbc = lane8 ? 16 : 8;
    const int st_bytes = st8 ? 1 : 2;
    const size_t limit = 200 * 1024;
    const int bt = (int)sizeof(BT);
    // stage small planes in shared memory (the sliding window sweeps re-read
    // every row 2 x (chunks) times; from global memory they are latency-bound)
    // while two CTAs still fit per SM, else read them from global memory
    g.stage = 0;
    g.G = 8;
    if ((int64_t)h * w * bt <= 48 * 1024) {
        g.stage = 1;
        while (g.G > 2 && ref_smem_bytes(g, st_bytes, nbc, bt) > 110 * 1024) g.G >>= 1;
        if (ref_smem_bytes(g, st_bytes, nbc, bt) > 110 * 1024) { g.stage = 0; g.G = 8; }
    }
    // unstaged planes read their rows from global memory: prefer two CTAs per SM
    // (more loads in flight) over more sample rows per pass
    if (!g.stage)
        while (g.G > 1 && ref_smem_bytes(g, st_bytes, nbc, bt) > 110 * 1024) g.G >>= 1;
    while (g.G > 1 && ref_smem_bytes(g, st_bytes, nbc, bt) > limit) g.G >>= 1;
    const size_t smem = ref_smem_bytes(g, st_bytes, nbc, bt);
    if (smem > limit) return QFCA_ERR_UNSUPPORTED;
    cudaError_t e;
#define QFCA_REF_LAUNCH(LANE, STT)                                                         \
    do {                                                                                   \
        auto kern = k_reference<BT, LANE, STT>;                                            \
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                 (int)smem);                                               \
        if (e != cudaSuccess) return QFCA_ERR_CUDA;                                        \
        kern<<<(unsigned)planes, REF_THREADS, smem, st>>>(bins, lo, hi, g, n_bins, pad,    \
                                                          mode, stats);                    \
    } while (0)
    if (lane8 && st8) QFCA_REF_LAUNCH(8, uint8_t);
    else if (lane8) QFCA_REF_LAUNCH(8, uint16_t);
    else QFCA_REF_LAUNCH(16, uint16_t);
#undef QFCA_REF_LAUNCH
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int launch_reference(const void* bins, int bins_bytes, const float* lo, const float* hi,
                     int64_t planes, int h, int w, int n_bins, int t, int pad, int budget,
                     int mode, int32_t* stats, cudaStream_t st) {
    if (planes <= 0 || h <= 0 || w <= 0 || n_bins < 1 || t < 1 || (t & 1) == 0 || budget < 1)
        return QFCA_ERR_ARG;
    if (mode != 0 && mode != 2 && mode != 3) return QFCA_ERR_UNSUPPORTED;
    if (bins_bytes == 1)
        return launch_reference_t((const uint8_t*)bins, lo, hi, planes, h, w, n_bins, t, pad,
                                  budget, mode, stats, st);
    if (bins_bytes == 2)
        return launch_reference_t((const uint16_t*)bins, lo, hi, planes, h, w, n_bins, t, pad,
                                  budget, mode, stats, st);
    return QFCA_ERR_ARG;
}

}  // namespace qfca
