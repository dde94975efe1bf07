// score2.cu -- K4 v2: the fused scoring kernel, specialised for the default
// family (uint8 bins, T <= 15 compile-time, a whole row of bins per CTA pass).
//
// Same mathematics as score.cu (see its header) -- exact integer window
// counts, closed-form Alg. 1, exact sliding box sums -- with a thread mapping
// chosen for instruction count and on-chip traffic:
//
//   thread (slot cs, bin group g, column x): 4 bins i = 4g..4g+3 of column x
//   of one channel; CPB channels ("slots") of one image share the CTA.
//
//   H1  vertical window counts as *thermometer* words: 8-bit lane j holds
//       #{rows of the column window with bin <= 4g+j}; one column tracker per
//       thread slides down the row stream (2 thermometer updates per row).
//   H2  horizontal window: a (row, slot, group, 8-column segment) task slides
//       the padded row of column words -> A_{4g+j}(y,x) directly (cumulative
//       counts, no cross-word prefix; A_{4g-1} is lane 3 of group g-1).
//   E   per thread, per row, 4 bins: E_i = (G_i(A_i) - G_i(A_{i-1})) / P_i in
//       fp32 from exact small integers; the vertical box sum keeps a T-row
//       ring of E in REGISTERS (row loop unrolled by T, static slots),
//       re-anchored every T rows (no drift).
//   A   own-bin horizontal box from the per-row V planes, all slots of the
//       CTA summed in fixed order, one RMW of the group partial per pixel.
//
// Shared rows are skewed (one pad word per 8) so the 8-column segment tasks
// of a warp hit distinct banks.
#include "common.cuh"

namespace qfca {

constexpr int S2_THREADS = 512;
constexpr int S2_SEG = 8;  // columns per H2 task

struct Score2Geom {
    int h, w, n_bins, pad, C, groups, cpg;
    int G;      // bin groups of 4 (ceil(N / 4))
    int CPB;    // channels per CTA pass
    int WP;     // padded row length (w + 2r), skewed storage length WPS
    int WPS;
    int S;      // stream rows h + 2r
};

__device__ __forceinline__ int skew(int p) { return p + (p >> 3); }

__device__ __forceinline__ uint32_t thermo(int b, int g4) {
    // lane j = [b <= g4 + j]
    const int d = b - g4;
    return d <= 0 ? 0x01010101u : (d < 4 ? (0x01010101u << (8 * d)) : 0u);
}

template <int T>
struct S2Smem {
    static constexpr int R = T / 2;
};

template <int T>
__host__ __device__ inline size_t score2_smem(const Score2Geom& g, size_t* offs) {
    size_t off = 0;
    int k = 0;
    auto take = [&](size_t bytes) {
        if (offs) offs[k] = off;
        ++k;
        off = (off + bytes + 15) & ~(size_t)15;
    };
    const int np = g.G * 4;
    take((size_t)g.CPB * g.h * g.w);                       // 0 bins planes (u8)
    take((size_t)g.CPB * (T * T + 1) * 4);                 // 1 PJ tables (float)
    take((size_t)g.CPB * np * 2 * 4);                      // 2 Vm / D per bin (float)
    take((size_t)g.S * 4 * 4);                             // 3 stream table (int4)
    take((size_t)T * g.CPB * g.G * g.WPS * 4);             // 4 CHp
    take((size_t)T * g.CPB * g.G * g.w * 4);               // 5 WH
    take((size_t)T * g.CPB * np * g.w * 4);                // 6 Vb
    take((size_t)g.WP * 4);                                // 7 padded-x -> x map
    take((size_t)g.CPB * 4);                               // 8 slot flags
    return off;
}

template <int T>
__global__ void __launch_bounds__(S2_THREADS, 1)
k_score2(const uint8_t* __restrict__ bins, const float* __restrict__ lo,
         const float* __restrict__ hi, const int32_t* __restrict__ Vref, Score2Geom g,
         float* __restrict__ partial) {
    constexpr int R = T / 2;
    constexpr int T2 = T * T;
    extern __shared__ __align__(16) uint8_t sm[];
    size_t offs[9];
    score2_smem<T>(g, offs);
    uint8_t* sb = sm + offs[0];
    float* sPJ = reinterpret_cast<float*>(sm + offs[1]);
    float* sVD = reinterpret_cast<float*>(sm + offs[2]);
    int4* stab = reinterpret_cast<int4*>(sm + offs[3]);
    uint32_t* CHp = reinterpret_cast<uint32_t*>(sm + offs[4]);
    uint32_t* WH = reinterpret_cast<uint32_t*>(sm + offs[5]);
    float* Vb = reinterpret_cast<float*>(sm + offs[6]);
    int* xmap = reinterpret_cast<int*>(sm + offs[7]);
    float* sscale = reinterpret_cast<float*>(sm + offs[8]);

    const int tid = threadIdx.x;
    const int w = g.w, h = g.h, G = g.G, NP = G * 4;
    const int per_slot = G * w;
    const int cs = tid / per_slot;
    const int gx = tid - cs * per_slot;
    const int grp4 = (gx / w) * 4;  // first bin of this thread's group
    const int x = gx % w;
    const bool active = cs < g.CPB;
    const int img = blockIdx.x / g.groups, cg = blockIdx.x % g.groups;
    const int c_begin = cg * g.cpg, c_end = min(g.C, c_begin + g.cpg);
    const int64_t hw = (int64_t)h * w;
    float* part = partial + ((int64_t)img * g.groups + cg) * hw;

    // ---- per-CTA geometry tables: stream rows and padded-x map
    for (int s = tid; s < g.S; s += S2_THREADS) {
        const int e = s - R;
        const int ye = map_coord(e, h, g.pad);
        int mode = 0, add = 0, rem = 0;
        if (s > 0) {
            const int yp = map_coord(e - 1, h, g.pad);
            if (ye == yp + 1) { mode = 1; add = map_coord(ye + R, h, g.pad); rem = map_coord(yp - R, h, g.pad); }
            else if (ye == yp - 1) { mode = 2; add = map_coord(ye - R, h, g.pad); rem = map_coord(yp + R, h, g.pad); }
            else if (ye == yp) { mode = 3; }
        }
        stab[s] = make_int4(ye, mode, add, rem);
    }
    for (int p = tid; p < g.WP; p += S2_THREADS) xmap[p] = map_coord(p - R, w, g.pad);
    __syncthreads();
    // halo positions this thread's column feeds (padded p with xmap[p] == x, p outside [R, R+w))
    uint32_t halo_mask = 0;
    if (active) {
        for (int j = 0; j < 2 * R; ++j) {
            const int p = j < R ? j : w + j;
            if (xmap[p] == x) halo_mask |= 1u << j;
        }
    }

    const int n_chunks = (g.S + T - 1) / T;
    for (int cb = c_begin; cb < c_end; cb += g.CPB) {
        // ---- load the slot channels: bins planes, reference tables
        __syncthreads();
        for (int k = 0; k < g.CPB; ++k) {
            const int c = cb + k;
            const int64_t plane = (int64_t)img * g.C + c;
            if (tid == 0) {
                // per-slot score scale w_c / T^2; 0 marks an empty or degenerate slot
                float sc = 0.f;
                if (c < c_end && hi[plane] > lo[plane])
                    sc = (float)(((double)hi[plane] - (double)lo[plane]) / (double)g.n_bins /
                                 (double)T2);
                sscale[k] = sc;
            }
            uint8_t* dst = sb + (size_t)k * hw;
            if (c < c_end) {
                const uint8_t* src = bins + plane * hw;
                if ((hw & 15) == 0) {
                    const uint4* s4 = reinterpret_cast<const uint4*>(src);
                    uint4* d4 = reinterpret_cast<uint4*>(dst);
                    for (int64_t i = tid; i < hw / 16; i += S2_THREADS) d4[i] = __ldg(s4 + i);
                } else {
                    for (int64_t i = tid; i < hw; i += S2_THREADS) dst[i] = src[i];
                }
                // PJ[x] = sum_{k<x} J_k, J_k = min{i : V_i > k}
                const int32_t* V = Vref + plane * g.n_bins;
                float* pj = sPJ + (size_t)k * (T2 + 1);
                for (int q = tid; q < T2; q += S2_THREADS) {
                    int a = 0, b = g.n_bins - 1;
                    while (a < b) {
                        const int mid = (a + b) >> 1;
                        if (__ldg(V + mid) > q) b = mid; else a = mid + 1;
                    }
                    pj[q + 1] = (float)a;
                }
            } else {
                for (int64_t i = tid; i < hw; i += S2_THREADS) dst[i] = 0;
                for (int q = tid; q < T2; q += S2_THREADS) sPJ[(size_t)k * (T2 + 1) + q + 1] = 0.f;
            }
        }
        __syncthreads();
        if (tid < 32 * g.CPB) {  // one warp per slot: inclusive scan of PJ[1..T2]
            const int k = tid >> 5, lane = tid & 31;
            float* pj = sPJ + (size_t)k * (T2 + 1);
            float carry = 0.f;
            if (lane == 0) pj[0] = 0.f;
            for (int base = 1; base <= T2; base += 32) {
                const int q = base + lane;
                float v = q <= T2 ? pj[q] : 0.f;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float u = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += u;
                }
                v += carry;
                if (q <= T2) pj[q] = v;
                carry = __shfl_sync(0xffffffffu, v, 31);
            }
        }
        __syncthreads();
        for (int idx = tid; idx < g.CPB * NP; idx += S2_THREADS) {
            const int k = idx / NP, i = idx % NP;
            const int c = cb + k;
            float vm = 0.f, d = 0.f;
            if (c < c_end && i < g.n_bins) {
                const int32_t* V = Vref + ((int64_t)img * g.C + c) * g.n_bins;
                const int vmi = i > 0 ? V[i - 1] : 0;
                vm = (float)vmi;
                d = 2.f * ((float)i * vm - sPJ[(size_t)k * (T2 + 1) + vmi]);
            }
            sVD[(size_t)(k * NP + i) * 2] = vm;
            sVD[(size_t)(k * NP + i) * 2 + 1] = d;
        }
        __syncthreads();

        const int cs_ = active ? cs : 0;
        const uint8_t* mb = sb + (size_t)cs_ * hw;
        const float* pj = sPJ + (size_t)cs_ * (T2 + 1);
        float Vm[4], Dv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            Vm[j] = sVD[(size_t)(cs_ * NP + grp4 + j) * 2];
            Dv[j] = sVD[(size_t)(cs_ * NP + grp4 + j) * 2 + 1];
        }
        uint32_t cst = 0;  // column tracker (thermometer word)
        float ring[T][4];
        float vs[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            vs[j] = 0.f;
#pragma unroll
            for (int q = 0; q < T; ++q) ring[q][j] = 0.f;
        }

        for (int ch = 0; ch < n_chunks; ++ch) {
            const int s0 = ch * T;
            const int nrow = min(T, g.S - s0);
            // ---- H1: vertical thermometer window counts for the chunk rows
            if (active) {
                uint32_t* chp = CHp + ((size_t)cs * G + grp4 / 4) * g.WPS;
#pragma unroll
                for (int rho = 0; rho < T; ++rho) {
                    if (rho < nrow) {
                        const int4 st = stab[s0 + rho];
                        if (st.y == 0) {
                            cst = 0;
#pragma unroll 1
                            for (int dy = -R; dy <= R; ++dy)
                                cst += thermo(mb[map_coord(st.x + dy, h, g.pad) * w + x], grp4);
                        } else if (st.y != 3) {
                            cst += thermo(mb[st.z * w + x], grp4) - thermo(mb[st.w * w + x], grp4);
                        }
                        uint32_t* row = chp + (size_t)rho * g.CPB * G * g.WPS;
                        row[skew(x + R)] = cst;
                        if (halo_mask) {
                            for (int j = 0; j < 2 * R; ++j)
                                if (halo_mask & (1u << j)) row[skew(j < R ? j : w + j)] = cst;
                        }
                    }
                }
            }
            __syncthreads();
            // ---- H2: horizontal windows of the column words (segments of 8)
            {
                const int nseg = (w + S2_SEG - 1) / S2_SEG;
                const int rows_tasks = nrow * g.CPB * G;
                for (int task = tid; task < rows_tasks * nseg; task += S2_THREADS) {
                    const int seg = task % nseg;
                    const int rg = task / nseg;  // (rho * CPB + cs) * G + grp
                    const uint32_t* src = CHp + (size_t)rg * g.WPS;
                    uint32_t* dst = WH + (size_t)rg * w;
                    const int x0 = seg * S2_SEG;
                    uint32_t sum = 0;
#pragma unroll
                    for (int p = 0; p < T; ++p) sum += src[skew(x0 + p)];
                    dst[x0] = sum;
#pragma unroll
                    for (int k = 1; k < S2_SEG; ++k) {
                        const int xx = x0 + k;
                        if (xx < w) {
                            sum += src[skew(xx + 2 * R)] - src[skew(xx - 1)];
                            dst[xx] = sum;
                        }
                    }
                }
            }
            __syncthreads();
            // ---- E: closed-form transport + register ring + vertical box
            if (active) {
                const int grp = grp4 / 4;
#pragma unroll
                for (int rho = 0; rho < T; ++rho) {
                    if (rho < nrow) {
                        const uint32_t* whr = WH + ((size_t)(rho * g.CPB + cs) * G) * w + x;
                        const uint32_t word = whr[(size_t)grp * w];
                        int a = grp > 0 ? (int)(whr[(size_t)(grp - 1) * w] >> 24) : 0;
                        float af = (float)a;
                        float pja = pj[a];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int b = (word >> (8 * j)) & 0xff;
                            const float bf = (float)b;
                            const float pjb = pj[b];
                            const float fi = (float)(grp4 + j);
                            const float ua = fmaf(-fi, af, pja);
                            const float ub = fmaf(-fi, bf, pjb);
                            const float ga = af < Vm[j] ? -ua : ua + Dv[j];
                            const float gb = bf < Vm[j] ? -ub : ub + Dv[j];
                            const float pc = bf - af;
                            const float E = pc > 0.f ? __fdividef(gb - ga, pc) : 0.f;
                            vs[j] += E - ring[rho][j];
                            ring[rho][j] = E;
                            af = bf;
                            pja = pjb;
                        }
                        if (rho == T - 1) {
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                float s = 0.f;
#pragma unroll
                                for (int q = 0; q < T; ++q) s += ring[q][j];
                                vs[j] = s;
                            }
                        }
                        const int y = s0 + rho - 2 * R;
                        if (y >= 0) {
                            float* vb = Vb + ((size_t)(rho * g.CPB + cs) * NP + grp4) * w + x;
#pragma unroll
                            for (int j = 0; j < 4; ++j) vb[(size_t)j * w] = vs[j];
                        }
                    }
                }
            }
            __syncthreads();
            // ---- A: own-bin horizontal box, slots summed in order, partial RMW
            for (int task = tid; task < nrow * w; task += S2_THREADS) {
                const int rho = task / w, xx = task % w;
                const int y = s0 + rho - 2 * R;
                if (y < 0) continue;
                float acc = 0.f;
                for (int k = 0; k < g.CPB; ++k) {
                    const float scale = sscale[k];
                    if (scale == 0.f) continue;
                    const int b = sb[(size_t)k * hw + (size_t)y * w + xx];
                    const float* vb = Vb + ((size_t)(rho * g.CPB + k) * NP + b) * w;
                    float f = 0.f;
                    if (xx >= R && xx + R < w) {
#pragma unroll
                        for (int d = -R; d <= R; ++d) f += vb[xx + d];
                    } else {
#pragma unroll
                        for (int d = 0; d < T; ++d) f += vb[xmap[xx + d]];
                    }
                    acc += f * scale;
                }
                part[(size_t)y * w + xx] += acc;
            }
        }
    }
}

static int score2_plan(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                       Score2Geom* out, size_t* smem_out) {
    if (t < 1 || t > 15 || (t & 1) == 0) return QFCA_ERR_UNSUPPORTED;
    if (n_bins > 256) return QFCA_ERR_UNSUPPORTED;
    Score2Geom g;
    g.h = h; g.w = w; g.n_bins = n_bins; g.pad = 0; g.C = C;
    g.G = (n_bins + 3) / 4;
    const int per = g.G * w;
    if (per > S2_THREADS || w < 8) return QFCA_ERR_UNSUPPORTED;
    g.CPB = S2_THREADS / per;
    if (g.CPB > 8) g.CPB = 8;
    const int r = t / 2;
    g.WP = w + 2 * r;
    g.WPS = g.WP + g.WP / 8 + 1;
    g.S = h + 2 * r;
    size_t bytes = 0;
    for (;;) {
        switch (t) {
#define QFCA_S2_CASE(TT) case TT: bytes = score2_smem<TT>(g, nullptr); break;
            QFCA_S2_CASE(1) QFCA_S2_CASE(3) QFCA_S2_CASE(5) QFCA_S2_CASE(7)
            QFCA_S2_CASE(9) QFCA_S2_CASE(11) QFCA_S2_CASE(13) QFCA_S2_CASE(15)
#undef QFCA_S2_CASE
        }
        if (bytes <= 225 * 1024) break;
        if (g.CPB > 1) { g.CPB--; continue; }
        return QFCA_ERR_UNSUPPORTED;
    }
    int groups = groups_hint;
    if (groups <= 0) {
        const int64_t want = 4 * 148;
        int64_t gg = (want + images - 1) / images;
        gg = gg < 1 ? 1 : gg;
        int64_t maxg = (C + g.CPB - 1) / g.CPB;  // at least CPB channels per group
        gg = gg > maxg ? maxg : gg;
        groups = (int)gg;
    }
    groups = groups < 1 ? 1 : (groups > C ? C : groups);
    g.cpg = (C + groups - 1) / groups;
    g.groups = (C + g.cpg - 1) / g.cpg;
    *out = g;
    *smem_out = bytes;
    return QFCA_OK;
}

int score2_groups(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint) {
    Score2Geom g;
    size_t smem;
    if (score2_plan(h, w, n_bins, t, C, images, groups_hint, &g, &smem) != QFCA_OK) return -1;
    return g.groups;
}

int launch_score2(const void* bins, int bins_bytes, const float* lo, const float* hi,
                  const int32_t* V, int64_t images, int C, int h, int w, int n_bins, int t,
                  int pad, int groups, float* partial, cudaStream_t st) {
    if (bins_bytes != 1) return QFCA_ERR_UNSUPPORTED;
    if (pad != QFCA_PAD_REFLECT && pad != QFCA_PAD_WRAP) return QFCA_ERR_UNSUPPORTED;
    Score2Geom g;
    size_t smem;
    int rc = score2_plan(h, w, n_bins, t, C, images, groups, &g, &smem);
    if (rc != QFCA_OK) return rc;
    if (groups > 0 && g.groups != groups) return QFCA_ERR_ARG;
    g.pad = pad;
    const int64_t grid = images * g.groups;
    cudaError_t e = cudaSuccess;
    switch (t) {
#define QFCA_S2_LAUNCH(TT)                                                                   \
    case TT:                                                                                 \
        e = cudaFuncSetAttribute(k_score2<TT>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                 (int)smem);                                                 \
        if (e != cudaSuccess) return QFCA_ERR_CUDA;                                          \
        k_score2<TT><<<(unsigned)grid, S2_THREADS, smem, st>>>((const uint8_t*)bins, lo, hi, \
                                                               V, g, partial);               \
        break;
        QFCA_S2_LAUNCH(1) QFCA_S2_LAUNCH(3) QFCA_S2_LAUNCH(5) QFCA_S2_LAUNCH(7)
        QFCA_S2_LAUNCH(9) QFCA_S2_LAUNCH(11) QFCA_S2_LAUNCH(13) QFCA_S2_LAUNCH(15)
#undef QFCA_S2_LAUNCH
        default: return QFCA_ERR_UNSUPPORTED;
    }
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
