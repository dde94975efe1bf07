// score.cu -- K4: fused per-(image, channel-group) scoring kernel.
//
// Replaces the reference hot loop: _channel_score_kernel (scoring.py:177-232,
// per-bin indicator SATs -> window counts -> per-pixel Alg. 1 -> per-bin error
// SATs -> own-bin gather) and the channel accumulation in detect
// (scoring.py:258-281), for the default family of configurations: uniform
// sigma_p, median-quan reference, reflect or wrap padding.
//
// Everything below is exact integer work except the error values:
//   * window counts are packed 8-bit (T <= 15) or 16-bit lanes; a column
//     tracker slides down the row stream, the row window is a modular 32-bit
//     prefix difference along the padded row (exact, lanes never exceed T^2);
//   * the reference enters as V_i (cumulative reference counts, reference.cu)
//     and the prefix table PJ[x] = sum_{k<x} J_k; Alg. 1 on integer masses of
//     equal total (scale = 1, transport.py:84) has the closed form
//         E_i = w * (G_i(A_i) - G_i(A_{i-1})) / P_i,
//         G_i(x) = x < V_{i-1} ? -(PJ[x] - i x) : (PJ[x] - i x) + D_i,
//         D_i = 2 (i V_{i-1} - PJ[V_{i-1}])
//     (G_i(x) = sum_{k<x} |i - J_k|; K_i is an exact int32);
//   * the vertical box sum of E runs in fp64 over fp32 E values, which is exact
//     (no drift over the row stream); the horizontal box is gathered for the
//     pixel's own bin only; the per-channel score is added to a per-group fp32
//     partial map in fixed channel order.
// Cost per (channel, pixel) is independent of T (box sums by sliding / prefix
// differences), linear in N.
#include "common.cuh"

namespace qfca {

constexpr int SC_THREADS = 512;
constexpr int SC_MAXT = 8;  // E-phase tasks per thread: w * NBP <= SC_MAXT * SC_THREADS

struct ScoreGeom {
    int h, w, t, r, wp, n_bins, pad;
    int C, groups, cpg;  // channels, channel groups per image, channels per group
    int NBP;             // bins per pass
    int NWq;             // packed words per (row, x): ceil(NBP / L) + 1 ("below" word)
    int RC;              // stream rows per chunk
    int t2;
};

struct ScoreSmem {
    int32_t* Vs;      // [N]   cumulative reference counts V_i
    int32_t* Dv;      // [N]   D_i
    int32_t* PJ;      // [T^2+1]
    uint32_t* cst;    // [NWq][w] column tracker state
    uint32_t* CH;     // [RC][NWq][w] column counts per stream row
    uint32_t* WH;     // [RC][NWq][w] window counts per stream row
    uint32_t* PS;     // [nwarps][wp] prefix scratch
    void* AC;         // [RC][NBP+1][w] cumulative counts (u8 or u16)
    float* ring;      // [T][NBP][w] E ring buffer (stream rows)
    float* Vb;        // [RC][NBP][w] vertical box sums for output rows
};

template <typename AT>
__host__ __device__ inline size_t score_smem_layout(const ScoreGeom& g, ScoreSmem* s,
                                                   uint8_t* base) {
    size_t off = 0;
    auto take = [&](size_t bytes) -> uint8_t* {
        uint8_t* p = base ? base + off : nullptr;
        off = (off + bytes + 15) & ~(size_t)15;
        return p;
    };
    const int nwarps = SC_THREADS / 32;
    uint8_t* p;
    p = take((size_t)g.n_bins * 4);                         if (s) s->Vs = (int32_t*)p;
    p = take((size_t)g.n_bins * 4);                         if (s) s->Dv = (int32_t*)p;
    p = take((size_t)(g.t2 + 1) * 4);                       if (s) s->PJ = (int32_t*)p;
    p = take((size_t)g.NWq * g.w * 4);                      if (s) s->cst = (uint32_t*)p;
    p = take((size_t)g.RC * g.NWq * g.w * 4);               if (s) s->CH = (uint32_t*)p;
    p = take((size_t)g.RC * g.NWq * g.w * 4);               if (s) s->WH = (uint32_t*)p;
    p = take((size_t)nwarps * g.wp * 4);                    if (s) s->PS = (uint32_t*)p;
    p = take((size_t)g.RC * (g.NBP + 1) * g.w * sizeof(AT)); if (s) s->AC = p;
    p = take((size_t)g.t * g.NBP * g.w * 4);                if (s) s->ring = (float*)p;
    p = take((size_t)g.RC * g.NBP * g.w * 4);               if (s) s->Vb = (float*)p;
    return off;
}

template <typename BT, int LANE, typename AT>
__global__ void __launch_bounds__(SC_THREADS, 1)
k_score(const BT* __restrict__ bins, const float* __restrict__ lo, const float* __restrict__ hi,
        const int32_t* __restrict__ Vref, ScoreGeom g, float* __restrict__ partial) {
    constexpr int L = 32 / LANE;
    constexpr uint32_t LMASK = (1u << LANE) - 1u;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    ScoreSmem S;
    score_smem_layout<AT>(g, &S, smem_raw);
    AT* AC = reinterpret_cast<AT*>(S.AC);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = SC_THREADS / 32;
    const int img = blockIdx.x / g.groups, grp = blockIdx.x % g.groups;
    const int c_begin = grp * g.cpg, c_end = min(g.C, c_begin + g.cpg);
    const int64_t hw = (int64_t)g.h * g.w;
    float* part = partial + ((int64_t)img * g.groups + grp) * hw;
    const int w = g.w, r = g.r, T = g.t;

    for (int c = c_begin; c < c_end; ++c) {
        const int64_t plane = (int64_t)img * g.C + c;
        const double lo_c = lo[plane], hi_c = hi[plane];
        if (!(hi_c > lo_c)) continue;  // degenerate: skipped (scoring.py:265-266)
        const float scale = (float)(((hi_c - lo_c) / (double)g.n_bins) / (double)g.t2);
        const BT* bp = bins + plane * hw;

        // ---- reference tables: V_i, J -> PJ prefix, D_i
        __syncthreads();
        for (int i = tid; i < g.n_bins; i += SC_THREADS) S.Vs[i] = Vref[plane * g.n_bins + i];
        __syncthreads();
        for (int k = tid; k < g.t2; k += SC_THREADS) {
            // J_k = min{i : V_i > k}
            int a = 0, b = g.n_bins - 1;
            while (a < b) {
                const int mid = (a + b) >> 1;
                if (S.Vs[mid] > k) b = mid; else a = mid + 1;
            }
            S.PJ[k + 1] = a;
        }
        if (tid == 0) S.PJ[0] = 0;
        __syncthreads();
        if (warp == 0) {  // inclusive scan of PJ[1..t2]
            int carry = 0;
            for (int base = 1; base <= g.t2; base += 32) {
                const int k = base + lane;
                int v = k <= g.t2 ? S.PJ[k] : 0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += u;
                }
                v += carry;
                if (k <= g.t2) S.PJ[k] = v;
                carry = __shfl_sync(0xffffffffu, v, 31);
            }
        }
        __syncthreads();
        for (int i = tid; i < g.n_bins; i += SC_THREADS) {
            const int vm = i > 0 ? S.Vs[i - 1] : 0;
            S.Dv[i] = 2 * (i * vm - S.PJ[vm]);
        }

        for (int p0 = 0; p0 < g.n_bins; p0 += g.NBP) {
            const int nbp = min(g.NBP, g.n_bins - p0);
            // reset the E ring (thread-owned slots: same (k, x) mapping as the E phase)
            __syncthreads();
            for (int idx = tid; idx < T * g.NBP * w; idx += SC_THREADS) S.ring[idx] = 0.f;
            double vsum[SC_MAXT];
#pragma unroll
            for (int m = 0; m < SC_MAXT; ++m) vsum[m] = 0.0;
            int yprev = 0;
            __syncthreads();

            for (int e0 = -r; e0 < g.h + r; e0 += g.RC) {
                const int nrow = min(g.RC, g.h + r - e0);
                // ---- H1: column trackers (task = (word, x)), state in smem
                {
                    int yp = yprev;
                    for (int rho = 0; rho < nrow; ++rho) {
                        const int e = e0 + rho;
                        const int yn = map_coord(e, g.h, g.pad);
                        for (int task = tid; task < g.NWq * w; task += SC_THREADS) {
                            const int word = task / w, x = task % w;
                            const bool below = word == g.NWq - 1;
                            const int wb0 = p0 + word * L;  // first bin of this word
                            auto oh = [&](int yrow) -> uint32_t {
                                const int bb = (int)bp[(int64_t)map_coord(yrow, g.h, g.pad) * w + x];
                                if (below) return bb < p0 ? 1u : 0u;
                                const int rel = bb - wb0;
                                return ((unsigned)rel < (unsigned)L && bb < p0 + nbp)
                                           ? (1u << (rel * LANE)) : 0u;
                            };
                            uint32_t st;
                            if (e == -r || (yn != yp + 1 && yn != yp - 1 && yn != yp)) {
                                st = 0u;
                                for (int dy = -r; dy <= r; ++dy) st += oh(yn + dy);
                            } else {
                                st = S.cst[task];
                                if (yn == yp + 1) st += oh(yn + r) - oh(yp - r);
                                else if (yn == yp - 1) st += oh(yn - r) - oh(yp + r);
                            }
                            S.cst[task] = st;
                            S.CH[(size_t)rho * g.NWq * w + task] = st;
                        }
                        yp = yn;
                    }
                    yprev = yp;
                }
                __syncthreads();
                // ---- H2: row windows by modular prefix over the padded row
                for (int row = warp; row < nrow * g.NWq; row += nwarps) {
                    const uint32_t* src = S.CH + (size_t)row * w;
                    uint32_t* ps = S.PS + (size_t)warp * g.wp;
                    uint32_t carry = 0;
                    for (int base = 0; base < g.wp; base += 32) {
                        const int xp = base + lane;
                        uint32_t v = xp < g.wp ? src[map_coord(xp - r, w, g.pad)] : 0u;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
                            if (lane >= o) v += u;
                        }
                        v += carry;
                        if (xp < g.wp) ps[xp] = v;
                        carry = __shfl_sync(0xffffffffu, v, 31);
                    }
                    __syncwarp();
                    uint32_t* dst = S.WH + (size_t)row * w;
                    for (int x = lane; x < w; x += 32)
                        dst[x] = ps[x + 2 * r] - (x > 0 ? ps[x - 1] : 0u);
                    __syncwarp();
                }
                __syncthreads();
                // ---- C: cumulative counts per (row, x): AC[rho][0] = below, [k+1] = A_{p0+k}
                for (int task = tid; task < nrow * w; task += SC_THREADS) {
                    const int rho = task / w, x = task % w;
                    const uint32_t* wh = S.WH + (size_t)rho * g.NWq * w + x;
                    uint32_t acc = wh[(size_t)(g.NWq - 1) * w];
                    AT* ac = AC + (size_t)rho * (g.NBP + 1) * w + x;
                    ac[0] = (AT)acc;
                    for (int word = 0; word < g.NWq - 1; ++word) {
                        const uint32_t v = wh[(size_t)word * w];
#pragma unroll
                        for (int q = 0; q < L; ++q) {
                            const int k = word * L + q;
                            if (k < nbp) {
                                acc += (v >> (q * LANE)) & LMASK;
                                ac[(size_t)(k + 1) * w] = (AT)acc;
                            }
                        }
                    }
                }
                __syncthreads();
                // ---- E: closed-form transport, E ring, vertical box sums (fp64, exact)
#pragma unroll
                for (int m = 0; m < SC_MAXT; ++m) {
                    const int task = tid + m * SC_THREADS;
                    if (task >= nbp * w) break;
                    const int k = task / w, x = task % w;
                    const int i = p0 + k;
                    const int vm = i > 0 ? S.Vs[i - 1] : 0;
                    const int di = S.Dv[i];
                    for (int rho = 0; rho < nrow; ++rho) {
                        const int e = e0 + rho;
                        const AT* ac = AC + (size_t)rho * (g.NBP + 1) * w + x;
                        const int a = (int)ac[(size_t)k * w];
                        const int b = (int)ac[(size_t)(k + 1) * w];
                        const int ua = S.PJ[a] - i * a, ub = S.PJ[b] - i * b;
                        const int ga = a < vm ? -ua : ua + di;
                        const int gb = b < vm ? -ub : ub + di;
                        const int pcount = b - a;
                        const float E = pcount > 0 ? (float)(gb - ga) / (float)pcount : 0.f;
                        const int slot = (e + r) % T;
                        float* rs = S.ring + ((size_t)slot * g.NBP + k) * w + x;
                        const float old = *rs;
                        *rs = E;
                        vsum[m] += (double)E - (double)old;
                        if (e - r >= 0) S.Vb[((size_t)rho * g.NBP + k) * w + x] = (float)vsum[m];
                    }
                }
                __syncthreads();
                // ---- A: horizontal box of the own-bin plane, add to the group partial
                for (int task = tid; task < nrow * w; task += SC_THREADS) {
                    const int rho = task / w, x = task % w;
                    const int y = e0 + rho - r;
                    if (y < 0) continue;
                    const int bb = (int)bp[(int64_t)y * w + x];
                    const int k = bb - p0;
                    if (k < 0 || k >= nbp) continue;
                    const float* vb = S.Vb + ((size_t)rho * g.NBP + k) * w;
                    float f = 0.f;
                    for (int dx = -r; dx <= r; ++dx) f += vb[map_coord(x + dx, w, g.pad)];
                    part[(int64_t)y * w + x] += f * scale;
                }
                __syncthreads();
            }
        }
    }
}

// used[b] = number of non-degenerate channels of image b
__global__ void k_count_used(const float* __restrict__ lo, const float* __restrict__ hi,
                             int64_t images, int C, int* __restrict__ used) {
    const int64_t b = blockIdx.x;
    int u = 0;
    for (int c = threadIdx.x; c < C; c += blockDim.x) u += (hi[b * C + c] > lo[b * C + c]) ? 1 : 0;
    u = warp_sum_i(u);
    __shared__ int sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = u;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
        used[b] = s;
    }
}

int score_plan(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
               ScoreGeom* out, size_t* smem_out, int* lane_out, int* at_out) {
    ScoreGeom g;
    g.h = h; g.w = w; g.t = t; g.r = t / 2; g.wp = w + 2 * g.r; g.n_bins = n_bins;
    g.t2 = t * t; g.C = C; g.pad = 0;
    const int lane = g.t2 <= 255 ? 8 : 16;
    const int L = 32 / lane;
    const int at = g.t2 <= 255 ? 1 : 2;
    const size_t limit = 220 * 1024;
    g.RC = 4;
    g.NBP = min(n_bins, (SC_MAXT * SC_THREADS) / w);
    if (g.NBP < 1) return QFCA_ERR_UNSUPPORTED;
    size_t bytes = 0;
    for (;;) {
        g.NWq = (g.NBP + L - 1) / L + 1;
        bytes = at == 1 ? score_smem_layout<uint8_t>(g, nullptr, nullptr)
                        : score_smem_layout<uint16_t>(g, nullptr, nullptr);
        if (bytes <= limit) break;
        if (g.NBP > 1) g.NBP = max(1, g.NBP / 2);
        else if (g.RC > 1) g.RC /= 2;
        else return QFCA_ERR_UNSUPPORTED;
    }
    int groups = groups_hint;
    if (groups <= 0) {
        // enough CTAs for ~8 waves on 148 SMs, channel groups of >= 4 channels
        const int64_t want = 8 * 148;
        int64_t gg = (want + images - 1) / images;
        if (gg < 1) gg = 1;
        if (gg > C) gg = C;
        groups = (int)gg;
        groups = min(groups, max(1, C / 4));
    }
    groups = max(1, min(groups, C));
    g.cpg = (C + groups - 1) / groups;
    g.groups = (C + g.cpg - 1) / g.cpg;
    *out = g;
    *smem_out = bytes;
    *lane_out = lane;
    *at_out = at;
    return QFCA_OK;
}

int launch_score(const void* bins, int bins_bytes, const float* lo, const float* hi,
                 const int32_t* V, int64_t images, int C, int h, int w, int n_bins, int t,
                 int pad, int groups, float* partial, cudaStream_t st) {
    if (images <= 0 || C <= 0 || h <= 0 || w <= 0 || n_bins < 1 || t < 1 || (t & 1) == 0)
        return QFCA_ERR_ARG;
    if (pad != QFCA_PAD_REFLECT && pad != QFCA_PAD_WRAP) return QFCA_ERR_UNSUPPORTED;
    if (t * t > 65535) return QFCA_ERR_UNSUPPORTED;
    ScoreGeom g;
    size_t smem;
    int lane, at;
    int rc = score_plan(h, w, n_bins, t, C, images, groups, &g, &smem, &lane, &at);
    if (rc != QFCA_OK) return rc;
    g.pad = pad;
    if (groups > 0 && g.groups != groups) return QFCA_ERR_ARG;
    const int64_t grid = images * g.groups;
    if (grid > 0x7fffffffLL) return QFCA_ERR_ARG;
    cudaError_t e;
#define QFCA_SCORE_LAUNCH(BTT, LANE, ATT)                                                  \
    do {                                                                                   \
        auto kern = k_score<BTT, LANE, ATT>;                                               \
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                 (int)smem);                                               \
        if (e != cudaSuccess) return QFCA_ERR_CUDA;                                        \
        kern<<<(unsigned)grid, SC_THREADS, smem, st>>>((const BTT*)bins, lo, hi, V, g,     \
                                                       partial);                           \
    } while (0)
    if (bins_bytes == 1) {
        if (lane == 8) QFCA_SCORE_LAUNCH(uint8_t, 8, uint8_t);
        else QFCA_SCORE_LAUNCH(uint8_t, 16, uint16_t);
    } else if (bins_bytes == 2) {
        if (lane == 8) QFCA_SCORE_LAUNCH(uint16_t, 8, uint8_t);
        else QFCA_SCORE_LAUNCH(uint16_t, 16, uint16_t);
    } else {
        return QFCA_ERR_ARG;
    }
#undef QFCA_SCORE_LAUNCH
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

int score_groups(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint) {
    ScoreGeom g;
    size_t smem;
    int lane, at;
    if (score_plan(h, w, n_bins, t, C, images, groups_hint, &g, &smem, &lane, &at) != QFCA_OK)
        return -1;
    return g.groups;
}

int launch_count_used(const float* lo, const float* hi, int64_t images, int C, int* used,
                      cudaStream_t st) {
    if (images <= 0 || C <= 0) return QFCA_ERR_ARG;
    k_count_used<<<(unsigned)images, 256, 0, st>>>(lo, hi, images, C, used);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
