// score3.cu -- K4 v3: warp-specialised, pipelined fused scoring kernel.
//
// Same mathematics and data layout as score2.cu (see its header); the
// difference is the execution schedule.  The CTA has 20 warps:
//
//   4 producer warps (P)   H1: one column tracker per thread slides the
//                          thermometer counts down the row stream and writes
//                          chunk c+1's column words to the double-buffered
//                          store CHp[(c+1)&1];
//   16 consumer warps (C)  H2 (row windows -> cumulative counts), E (closed-
//                          form transport, register E ring, vertical box) and
//                          A (own-bin horizontal box, partial-map update) for
//                          chunk c.
//
// Hand-off uses named barriers (bar.arrive / bar.sync): FULL[b] (producers ->
// consumers) and EMPTY[b] (consumers -> producers); the consumers synchronise
// among themselves on BAR_C; CTA-wide barriers only once per channel batch.
// The consumer phases are arranged as  E(c) | A(c) + H2(c+1)  so each chunk
// costs two consumer barriers.  The fused reference selection (pass 0) runs
// the same producer loop while the consumers window only the sample rows and
// gather the sample counts.  Fixed plane widths 32 / 64 / 128, N <= 16 bins
// (4 groups of 4), T <= 15.
#include <string.h>

#include "common.cuh"

namespace qfca {

constexpr int S3_CWARPS = 16;
constexpr int S3_PWARPS = 4;
constexpr int S3_CT = S3_CWARPS * 32;            // consumer threads
constexpr int S3_PT = S3_PWARPS * 32;            // producer threads
constexpr int S3_THREADS = S3_CT + S3_PT;        // 640
constexpr int S3_MAXSEG = 33;
// named barrier ids (0 is __syncthreads)
constexpr int BAR_C = 2, BAR_FULL0 = 3, BAR_EMPTY0 = 5;

struct Score3Geom {
    int h, n_bins, pad, C, groups, cpg;
    int WP;    // padded row length w + 2r
    int S;     // stream rows h + 2r
    int fref, stride, nsx, nsamp, sp;
    uint32_t moff;  // -4 * 0x4B000000 (mod 2^32): magic-float -> G-table byte offset
    int o_bins, o_pj, o_vd, o_gt, o_stab, o_chp, o_wh, o_vb, o_xmap, o_scale, o_th, o_sv, o_sa,
        o_srch, total;
};

__device__ __forceinline__ void bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
template <int OFF>
__device__ __forceinline__ float lds3_f32(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF));
    return v;
}
__device__ __forceinline__ float rcp_approx3(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// consumer H2 segment: odd (distinct banks across a warp), >= 5 columns,
// rows * segments <= consumer threads
__host__ __device__ constexpr int s3_seg(int t, int w) {
    return ((((w * t * (128 / w) + S3_CT - 1) / S3_CT) > 5
                 ? ((w * t * (128 / w) + S3_CT - 1) / S3_CT) : 5)) | 1;
}

template <int T, int W>
static void score3_layout(Score3Geom& g) {
    constexpr int CPB = 128 / W;
    int off = 0;
    auto take = [&](long long bytes) {
        const int o = off;
        off = (int)((off + bytes + 15) & ~15LL);
        return o;
    };
    g.o_bins = take((long long)CPB * g.h * W);
    g.o_pj = take((long long)CPB * (T * T + 1) * 4);
    g.o_vd = take((long long)CPB * 16 * 2 * 4);
    g.o_gt = take((long long)CPB * 16 * (T * T + 1) * 4);  // G_i(v) tables
    g.o_stab = take((long long)((g.S + T - 1) / T) * T * 16);
    g.o_chp = take((long long)2 * T * CPB * g.WP * 16);   // double-buffered column words
    g.o_wh = take((long long)T * CPB * W * 16);           // row windows (uint4 per pixel)
    const long long vb = (long long)T * CPB * 16 * W * 4;
    const long long sa = g.fref ? (long long)CPB * 16 * g.nsamp : 0;  // uint4 per sample
    g.o_vb = take(vb > sa ? vb : sa);
    g.o_sa = g.o_vb;
    g.o_xmap = take((long long)g.WP * 4);
    g.o_scale = take((long long)CPB * 4);
    g.o_th = take((long long)256 * 16);
    g.o_sv = take((long long)CPB * 16 * 4);
    g.o_srch = take(1024 + (S3_THREADS / 32) * 32);  // search brackets, packed mids, per-warp counts
    g.total = off;
}

template <int T, int W>
__global__ void __launch_bounds__(S3_THREADS, 1)
k_score3(const uint8_t* __restrict__ bins, const float* __restrict__ lo,
         const float* __restrict__ hi, const int32_t* __restrict__ Vref, const Score3Geom g,
         float* __restrict__ partial) {
    constexpr int R = T / 2;
    constexpr int T2 = T * T;
    constexpr int CPB = 128 / W;  // channel slots: CPB * W = 128 columns per CTA pass
    constexpr int SEG = s3_seg(T, W);
    constexpr int NSEG = (W + SEG - 1) / SEG;
    static_assert(T * CPB * NSEG <= S3_CT, "H2 tasks must fit the consumer warps");
    static_assert(SEG <= S3_MAXSEG, "segment too long");
    extern __shared__ __align__(16) uint8_t sm[];
    uint8_t* const sb = sm + g.o_bins;
    float* const sPJ = reinterpret_cast<float*>(sm + g.o_pj);
    float* const sVD = reinterpret_cast<float*>(sm + g.o_vd);
    float* const sGT = reinterpret_cast<float*>(sm + g.o_gt);
    int4* const stab = reinterpret_cast<int4*>(sm + g.o_stab);
    uint4* const CHp = reinterpret_cast<uint4*>(sm + g.o_chp);
    uint4* const WH = reinterpret_cast<uint4*>(sm + g.o_wh);
    float* const Vb = reinterpret_cast<float*>(sm + g.o_vb);
    int* const xmap = reinterpret_cast<int*>(sm + g.o_xmap);
    float* const sscale = reinterpret_cast<float*>(sm + g.o_scale);
    uint4* const TH = reinterpret_cast<uint4*>(sm + g.o_th);
    int* const sV = reinterpret_cast<int*>(sm + g.o_sv);
    uint4* const SA4 = reinterpret_cast<uint4*>(sm + g.o_sa);  // [CPB][nsamp] sample windows
    uint32_t* const scnt = reinterpret_cast<uint32_t*>(sm + g.o_srch + 1024); // [warps][8]
    uint8_t* const sqm8 = sm + g.o_srch + 256;                                 // [CPB][16]
    int* const sblo = reinterpret_cast<int*>(sm + g.o_srch + 320);            // [CPB * 16]
    int* const sbhi = reinterpret_cast<int*>(sm + g.o_srch + 576);            // [CPB * 16]

    const int tid = threadIdx.x;
    const bool is_p = tid >= S3_CT;
    const int h = g.h;
    const int hw = h * W;
    const int img = blockIdx.x / g.groups, cgi = blockIdx.x % g.groups;
    const int c_begin = cgi * g.cpg, c_end = min(g.C, c_begin + g.cpg);
    float* const part = partial + ((int64_t)img * g.groups + cgi) * hw;
    const int n_chunks = (g.S + T - 1) / T;
    const int CHSTRIDE = T * CPB * g.WP;  // uint4 per CHp buffer

    // ---- per-CTA tables (see score2.cu): stream rows, padded-x map, thermometer words
    for (int s = tid; s < n_chunks * T; s += S3_THREADS) {
        if (s >= g.S) {
            stab[s] = make_int4(0, 0, -1, -1);
            continue;
        }
        const int e = s - R;
        const int ye = map_coord(e, h, g.pad);
        int add = 0, rem = 0, recount = ye;
        if (s > 0) {
            const int yp = map_coord(e - 1, h, g.pad);
            if (ye == yp + 1) { recount = -1; add = map_coord(ye + R, h, g.pad); rem = map_coord(yp - R, h, g.pad); }
            else if (ye == yp - 1) { recount = -1; add = map_coord(ye - R, h, g.pad); rem = map_coord(yp + R, h, g.pad); }
            else if (ye == yp) { recount = -1; }
        }
        const int samp = (g.fref && e >= 0 && e < h && e % g.stride == 0)
                             ? (e / g.stride) * g.nsx : -1;
        stab[s] = make_int4(add * W, rem * W, recount, samp);
    }
    for (int p = tid; p < g.WP; p += S3_THREADS) xmap[p] = map_coord(p - R, W, g.pad);
    for (int b = tid; b < 256; b += S3_THREADS) {
        uint32_t v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // lane j of word q = [b <= 4q + j]
            const int d = b - 4 * q;
            v[q] = d <= 0 ? 0x01010101u : (d < 4 ? (0x01010101u << (8 * d)) : 0u);
        }
        TH[b] = make_uint4(v[0], v[1], v[2], v[3]);
    }
    __syncthreads();

    // ---- producer role: thread (slot pcs, column px)
    const int pt = tid - S3_CT;
    const int px = pt % W, pcs = is_p ? pt / W : 0;
    int halo0 = -1, halo1 = -1;
    if (is_p) {
        for (int j = 0; j < 2 * R; ++j) {
            const int p = j < R ? j : W + j;
            if (xmap[p] == px) {
                if (halo0 < 0) halo0 = p;
                else if (halo1 < 0) halo1 = p;
            }
        }
    }
    const bool many_halo = W <= R;
    const uint8_t* const pbx = sb + pcs * hw + px;

    // ---- consumer role: thread (slot cs, group grp, column x)
    const int cs = tid / (4 * W);
    const int grp = (tid / W) & 3;
    const int grp4 = grp * 4;
    const int x = tid % W;
    const int xsamp = (g.fref && x % g.stride == 0) ? x / g.stride : -1;
    const int csx = is_p ? 0 : cs;
    const float* const pj = sPJ + csx * (T2 + 1);
    constexpr int A_ROWS = S3_CT / W;  // A-phase rows per pass
    const int a_x = tid % W, a_r0 = tid / W;

    // H1 (producers) for chunk c into CHp[c & 1]
    uint4 cst = make_uint4(0, 0, 0, 0);
    auto h1_chunk = [&](int c) {
        uint4* base = CHp + (c & 1) * CHSTRIDE + pcs * g.WP;
#pragma unroll
        for (int rho = 0; rho < T; ++rho) {
            const int4 st = stab[c * T + rho];
            if (st.z < 0) {
                const uint4 a = TH[pbx[st.x]], r = TH[pbx[st.y]];
                cst.x += a.x - r.x;
                cst.y += a.y - r.y;
                cst.z += a.z - r.z;
                cst.w += a.w - r.w;
            } else {
                cst = make_uint4(0, 0, 0, 0);
#pragma unroll 1
                for (int dy = -R; dy <= R; ++dy) {
                    const uint4 a = TH[pbx[map_coord(st.z + dy, h, g.pad) * W]];
                    cst.x += a.x;
                    cst.y += a.y;
                    cst.z += a.z;
                    cst.w += a.w;
                }
            }
            uint4* row = base + rho * CPB * g.WP;
            row[px + R] = cst;
            if (halo0 >= 0) row[halo0] = cst;
            if (halo1 >= 0) row[halo1] = cst;
            if (many_halo) {
                for (int j = 0; j < 2 * R; ++j) {
                    const int p = j < R ? j : W + j;
                    if (xmap[p] == px) row[p] = cst;
                }
            }
        }
    };
    auto produce = [&]() {
        for (int c = 0; c < n_chunks; ++c) {
            const int b = c & 1;
            if (c >= 2) bar_sync(BAR_EMPTY0 + b, S3_THREADS);  // consumers done with CHp[b]
            h1_chunk(c);
            bar_arrive(BAR_FULL0 + b, S3_THREADS);
        }
    };
    // H2 (consumers): CHp[c & 1] -> WH (row windows of chunk c)
    auto h2_chunk = [&](int c, bool only_samples) {
        const int task = tid;
        if (task >= T * CPB * NSEG) return;
        const int rc = task / NSEG;  // rho * CPB + cs
        const int x0 = (task - rc * NSEG) * SEG;
        if (only_samples && stab[c * T + rc / CPB].w < 0) return;
        const uint4* src = CHp + (c & 1) * CHSTRIDE + rc * g.WP + x0;
        uint4* dst = WH + rc * W + x0;
        uint4 sum = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int p = 0; p < T; ++p) {
            const uint4 v = src[p];
            sum.x += v.x;
            sum.y += v.y;
            sum.z += v.z;
            sum.w += v.w;
        }
        dst[0] = sum;
        if (x0 + SEG <= W) {
#pragma unroll
            for (int k = 1; k < SEG; ++k) {
                const uint4 a = src[k + 2 * R], r = src[k - 1];
                sum.x += a.x - r.x;
                sum.y += a.y - r.y;
                sum.z += a.z - r.z;
                sum.w += a.w - r.w;
                dst[k] = sum;
            }
        } else {
            for (int k = 1; k < W - x0; ++k) {
                const uint4 a = src[k + 2 * R], r = src[k - 1];
                sum.x += a.x - r.x;
                sum.y += a.y - r.y;
                sum.z += a.z - r.z;
                sum.w += a.w - r.w;
                dst[k] = sum;
            }
        }
    };
    // consumer: wait for chunk c's column words, window them, release CHp[c & 1]
    auto consume_h2 = [&](int c, bool only_samples) {
        bar_sync(BAR_FULL0 + (c & 1), S3_THREADS);
        h2_chunk(c, only_samples);
        if (c + 2 < n_chunks) bar_arrive(BAR_EMPTY0 + (c & 1), S3_THREADS);
    };

    for (int cb = c_begin; cb < c_end; cb += CPB) {
        // ---- load the slot channels (all warps)
        __syncthreads();
        for (int k = 0; k < CPB; ++k) {
            const int c = cb + k;
            const int64_t plane = (int64_t)img * g.C + c;
            if (tid == 0) {
                float sc = 0.f;
                if (c < c_end && hi[plane] > lo[plane])
                    sc = (float)(((double)hi[plane] - (double)lo[plane]) / (double)g.n_bins /
                                 (double)T2);
                sscale[k] = sc;
            }
            uint8_t* dst = sb + k * hw;
            if (c < c_end) {
                const uint8_t* src = bins + plane * hw;
                const uint4* s4 = reinterpret_cast<const uint4*>(src);
                uint4* d4 = reinterpret_cast<uint4*>(dst);
                for (int i = tid; i < hw / 16; i += S3_THREADS) d4[i] = __ldg(s4 + i);
                if (!g.fref)
                    for (int i = tid; i < 16; i += S3_THREADS)
                        sV[k * 16 + i] = i < g.n_bins ? __ldg(Vref + plane * g.n_bins + i) : T2;
            } else {
                for (int i = tid; i < hw; i += S3_THREADS) dst[i] = 0;
                for (int i = tid; i < 16; i += S3_THREADS) sV[k * 16 + i] = T2;
            }
        }
        __syncthreads();

        if (g.fref) {
            // ---- pass 0: reference selection from the sample-row windows
            if (is_p) {
                produce();
            } else {
                for (int c = 0; c < n_chunks; ++c) {
                    consume_h2(c, true);
                    bar_sync(BAR_C, S3_CT);  // WH complete
                    if (xsamp >= 0 && grp == 0) {  // sample windows, pixel-major (uint4)
#pragma unroll
                        for (int rho = 0; rho < T; ++rho) {
                            const int si = stab[c * T + rho].w;
                            if (si < 0) continue;
                            SA4[cs * g.nsamp + si + xsamp] = WH[(rho * CPB + cs) * W + x];
                        }
                    }
                    bar_sync(BAR_C, S3_CT);  // WH may be overwritten
                }
            }
            __syncthreads();
            {  // all 16 bins at once: lock-step binary search with packed 8-bit
               // compares (see score4.cu): smallest v with #{A <= v} >= S - m
                constexpr int TPS = S3_THREADS / CPB;  // search threads per slot
                static_assert(TPS % 32 == 0, "search warps must not straddle slots");
                constexpr int ROUNDS = T2 < 2 ? 1 : (T2 < 4 ? 2 : (T2 < 8 ? 3 : (T2 < 16 ? 4 :
                                       (T2 < 32 ? 5 : (T2 < 64 ? 6 : 7)))));
                const int c0 = g.nsamp - (g.nsamp - 1) / 2;
                if (tid < CPB * 16) {
                    const int k = tid >> 4, i = tid & 15;
                    const int top = (i < g.n_bins - 1 && sscale[k] != 0.f) ? 0 : T2;
                    sblo[tid] = top;
                    sbhi[tid] = T2;
                    sqm8[tid] = (uint8_t)((top + T2) >> 1);
                }
                __syncthreads();
                const int k = tid / TPS, lt = tid - k * TPS, lane = tid & 31;
                constexpr int WPS = TPS / 32;  // search warps per slot
                const uint4* sa = SA4 + (size_t)k * g.nsamp;
                const uint32_t* sqm = reinterpret_cast<const uint32_t*>(sqm8);
#pragma unroll 1
                for (int r = 0; r < ROUNDS; ++r) {
                    uint32_t Q[4], acc[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int q = 0; q < 4; ++q) Q[q] = 0x80808080u | sqm[k * 4 + q];
                    for (int smp = lt; smp < g.nsamp; smp += TPS) {
                        const uint4 v = sa[smp];
                        acc[0] += __umulhi((Q[0] - v.x) & 0x80808080u, 1u << 25);
                        acc[1] += __umulhi((Q[1] - v.y) & 0x80808080u, 1u << 25);
                        acc[2] += __umulhi((Q[2] - v.z) & 0x80808080u, 1u << 25);
                        acc[3] += __umulhi((Q[3] - v.w) & 0x80808080u, 1u << 25);
                    }
                    // per-warp sums of the 16-bit count fields (no shared atomics)
                    uint32_t* cp = scnt + (tid >> 5) * 8;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t ev = __reduce_add_sync(0xffffffffu, acc[q] & 0x00FF00FFu);
                        const uint32_t od =
                            __reduce_add_sync(0xffffffffu, (acc[q] >> 8) & 0x00FF00FFu);
                        if (lane == 0) {
                            cp[2 * q] = ev;
                            cp[2 * q + 1] = od;
                        }
                    }
                    __syncthreads();
                    if (tid < CPB * 16) {
                        const int kk = tid >> 4, i = tid & 15, j = i & 3, q = i >> 2;
                        uint32_t word = 0;  // fields stay < 65536: nsamp < 65536
#pragma unroll
                        for (int w = 0; w < WPS; ++w) word += scnt[(kk * WPS + w) * 8 + 2 * q + (j & 1)];
                        const int count = (int)((j >> 1) ? word >> 16 : word & 0xFFFFu);
                        int a = sblo[tid], bnd = sbhi[tid];
                        const int mid = (a + bnd) >> 1;
                        if (count >= c0) bnd = mid; else a = mid + 1;
                        sblo[tid] = a;
                        sbhi[tid] = bnd;
                        sqm8[tid] = (uint8_t)((a + bnd) >> 1);
                    }
                    __syncthreads();
                }
                if (tid < CPB * 16) sV[tid] = sblo[tid];
            }
            __syncthreads();
        }
        // ---- reference tables: PJ = prefix of J, (V_{i-1}, D_i) per bin
        for (int k = 0; k < CPB; ++k) {
            float* pjk = sPJ + k * (T2 + 1);
            const int* V = sV + k * 16;
            for (int q = tid; q < T2; q += S3_THREADS) {
                int a = 0, bnd = g.n_bins - 1;
                while (a < bnd) {
                    const int mid = (a + bnd) >> 1;
                    if (V[mid] > q) bnd = mid; else a = mid + 1;
                }
                pjk[q + 1] = (float)a;
            }
        }
        __syncthreads();
        if (tid < 32 * CPB) {
            const int k = tid >> 5, lane = tid & 31;
            float* pjk = sPJ + k * (T2 + 1);
            float carry = 0.f;
            if (lane == 0) pjk[0] = 0.f;
            for (int base = 1; base <= T2; base += 32) {
                const int q = base + lane;
                float v = q <= T2 ? pjk[q] : 0.f;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float u = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += u;
                }
                v += carry;
                if (q <= T2) pjk[q] = v;
                carry = __shfl_sync(0xffffffffu, v, 31);
            }
        }
        __syncthreads();
        for (int idx = tid; idx < CPB * 16; idx += S3_THREADS) {
            const int k = idx / 16, i = idx % 16;
            float vm = 0.f, d = 0.f;
            if (i < g.n_bins) {
                const int vmi = i > 0 ? sV[k * 16 + i - 1] : 0;
                vm = (float)vmi;
                d = 2.f * ((float)i * vm - sPJ[k * (T2 + 1) + vmi]);
            }
            sVD[(k * 16 + i) * 2] = vm;
            sVD[(k * 16 + i) * 2 + 1] = d;
        }
        // G_i(v) for every bin and count (same fp32 operations as the inline form)
        for (int idx = tid; idx < CPB * 16 * (T2 + 1); idx += S3_THREADS) {
            const int ki = idx / (T2 + 1), v = idx - ki * (T2 + 1);
            const int k = ki >> 4, i = ki & 15;
            const float* pjk = sPJ + k * (T2 + 1);
            float vm = 0.f, d = 0.f;
            if (i < g.n_bins) {
                const int vmi = i > 0 ? sV[k * 16 + i - 1] : 0;
                vm = (float)vmi;
                d = 2.f * ((float)i * vm - pjk[vmi]);
            }
            const float fv = (float)v;
            const float nu = fmaf((float)i, fv, -pjk[v]);
            sGT[idx] = fv < vm ? nu : d - nu;
        }
        __syncthreads();

        // ---- pass 1: scoring
        if (is_p) {
            produce();
        } else {
            constexpr int GP = T2 + 1;
            const bool g1 = (grp & 1) != 0, g2 = (grp & 2) != 0;
            // G-table address of count b = gaddr + 4 * magic(b) (see score4.cu)
            const uint32_t gaddr =
                (uint32_t)__cvta_generic_to_shared(sGT + (cs * 16 + grp4) * GP) + g.moff;
            float ring[T][4];
            float vs[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                vs[j] = 0.f;
#pragma unroll
                for (int q = 0; q < T; ++q) ring[q][j] = 0.f;
            }
            consume_h2(0, false);
            bar_sync(BAR_C, S3_CT);  // WH(0) complete
            constexpr int MAXA = (T + A_ROWS - 1) / A_ROWS;  // box rows per thread
            for (int c = 0; c < n_chunks; ++c) {
                const int s0 = c * T;
                // partial-map values of this chunk's box rows, fetched before the
                // transport so their latency hides behind it
                float pold[MAXA];
#pragma unroll
                for (int q = 0; q < MAXA; ++q) {
                    const int rho = a_r0 + q * A_ROWS;
                    const int y = s0 + rho - 2 * R;
                    pold[q] = (rho < T && y >= 0 && y < h) ? part[y * W + a_x] : 0.f;
                }
                // ---- E(c): closed-form transport, register ring, vertical box
#pragma unroll
                for (int rho = 0; rho < T; ++rho) {
                    const uint4 v = WH[(rho * CPB + cs) * W + x];
                    // (word, prev) = words grp, grp - 1 (0 for grp 0): branch-free selects
                    const uint32_t wlo = g1 ? v.y : v.x, whi = g1 ? v.w : v.z;
                    const uint32_t plo = g1 ? v.x : 0u, phi = g1 ? v.z : v.y;
                    const uint32_t word = g2 ? whi : wlo, prev = g2 ? phi : plo;
                    const bool mass = (word >> 24) != (prev >> 24);
                    float E[4] = {0.f, 0.f, 0.f, 0.f};  // no mass in the group: E = 0
                    if (__any_sync(0xffffffffu, mass)) {
                        uint32_t ma = __byte_perm(prev, 0x4B000000u, 0x7653);
                        uint32_t aa = gaddr + 4u * ma;
#define S3_E(J)                                                                 \
    {                                                                           \
        const uint32_t mb = __byte_perm(word, 0x4B000000u, 0x7650 + J);         \
        const uint32_t ab = gaddr + 4u * mb;                                    \
        const float gb = lds3_f32<J * GP * 4>(ab);                              \
        const float ga = lds3_f32<J * GP * 4>(aa);                              \
        const float pc = __uint_as_float(mb) - __uint_as_float(ma);             \
        E[J] = (gb - ga) * rcp_approx3(fmaxf(pc, 1.f));                         \
        ma = mb;                                                                \
        aa = ab;                                                                \
    }
                        S3_E(0) S3_E(1) S3_E(2) S3_E(3)
#undef S3_E
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        vs[j] += E[j] - ring[rho][j];
                        ring[rho][j] = E[j];
                    }
                    if (rho == T - 1) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            float s = ring[0][j];
#pragma unroll
                            for (int q = 1; q < T; ++q) s += ring[q][j];
                            vs[j] = s;
                        }
                    }
                    if (s0 + rho >= 2 * R) {
                        float* vb = Vb + ((rho * CPB + cs) * 16 + grp4) * W + x;
#pragma unroll
                        for (int j = 0; j < 4; ++j) vb[j * W] = vs[j];
                    }
                }
                bar_sync(BAR_C, S3_CT);  // Vb complete, WH free
                // ---- A(c): own-bin horizontal box, slots in fixed order, partial RMW
#pragma unroll
                for (int q = 0; q < MAXA; ++q) {
                    const int rho = a_r0 + q * A_ROWS;
                    const int y = s0 + rho - 2 * R;
                    if (rho >= T || y < 0 || y >= h) continue;
                    float acc = 0.f;
#pragma unroll
                    for (int k = 0; k < CPB; ++k) {
                        const float scale = sscale[k];
                        if (scale == 0.f) continue;
                        const int bb = sb[k * hw + y * W + a_x];
                        const float* vb = Vb + ((rho * CPB + k) * 16 + bb) * W;
                        float f = 0.f;
                        if (a_x >= R && a_x + R < W) {
#pragma unroll
                            for (int d = -R; d <= R; ++d) f += vb[a_x + d];
                        } else {
#pragma unroll
                            for (int d = 0; d < T; ++d) f += vb[xmap[a_x + d]];
                        }
                        acc = fmaf(f, scale, acc);
                    }
                    part[y * W + a_x] = pold[q] + acc;
                }
                // ---- H2(c+1) in the same phase (WH is free, Vb is only read)
                if (c + 1 < n_chunks) consume_h2(c + 1, false);
                bar_sync(BAR_C, S3_CT);  // Vb free, WH(c+1) complete
            }
        }
    }
}

int sample_stride(int h, int w, int budget);

template <int T, int W>
static int s3_total(Score3Geom& g) {
    score3_layout<T, W>(g);
    return g.total;
}

static int score3_plan(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                       int pad, int budget, bool fused_ref, Score3Geom* out, size_t* smem_out) {
    if (t < 1 || t > 15 || (t & 1) == 0 || n_bins > 16) return QFCA_ERR_UNSUPPORTED;
    if (w != 32 && w != 64 && w != 128) return QFCA_ERR_UNSUPPORTED;
    if ((int64_t)h * w > (1 << 24) || ((int64_t)h * w) % 16) return QFCA_ERR_UNSUPPORTED;
    if (pad != QFCA_PAD_REFLECT && pad != QFCA_PAD_WRAP) return QFCA_ERR_UNSUPPORTED;
    Score3Geom g;
    memset(&g, 0, sizeof(g));
    g.h = h; g.n_bins = n_bins; g.pad = pad; g.C = C;
    g.moff = 0u - 4u * 0x4B000000u;
    g.WP = w + 2 * (t / 2);
    g.S = h + 2 * (t / 2);
    g.fref = fused_ref && t * t <= 126 && budget >= 1 && (pad == QFCA_PAD_WRAP || h > 1) ? 1 : 0;
    if (g.fref) {
        g.stride = sample_stride(h, w, budget);
        g.nsx = (w + g.stride - 1) / g.stride;
        g.nsamp = ((h + g.stride - 1) / g.stride) * g.nsx;
        g.sp = (g.nsamp + 3) & ~3;
    }
    size_t bytes = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        switch (t * 1000 + w) {
#define S3C(TT, WW) case TT * 1000 + WW: bytes = s3_total<TT, WW>(g); break;
            S3C(1, 32) S3C(1, 64) S3C(1, 128) S3C(3, 32) S3C(3, 64) S3C(3, 128)
            S3C(5, 32) S3C(5, 64) S3C(5, 128) S3C(7, 32) S3C(7, 64) S3C(7, 128)
            S3C(9, 32) S3C(9, 64) S3C(9, 128) S3C(11, 32) S3C(11, 64) S3C(11, 128)
            S3C(13, 32) S3C(13, 64) S3C(13, 128) S3C(15, 32) S3C(15, 64) S3C(15, 128)
#undef S3C
            default: return QFCA_ERR_UNSUPPORTED;
        }
        if (bytes <= 225 * 1024) break;
        if (!g.fref) return QFCA_ERR_UNSUPPORTED;
        g.fref = 0;
    }
    if (bytes > 225 * 1024) return QFCA_ERR_UNSUPPORTED;
    const int cpb = 128 / w;
    int groups = groups_hint;
    if (groups <= 0) groups = balanced_groups(images, C, cpb, 1);
    groups = groups < 1 ? 1 : (groups > C ? C : groups);
    // whole batches per group
    g.cpg = ((C + groups - 1) / groups + cpb - 1) / cpb * cpb;
    g.groups = (C + g.cpg - 1) / g.cpg;
    *out = g;
    *smem_out = bytes;
    return QFCA_OK;
}

int score3_query(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                 int pad, int budget, int want_fref, int* fref) {
    Score3Geom g;
    size_t smem;
    if (score3_plan(h, w, n_bins, t, C, images, groups_hint, pad, budget, want_fref != 0, &g,
                    &smem) != QFCA_OK)
        return -1;
    if (fref) *fref = g.fref;
    return g.groups;
}

int launch_score3(const void* bins, int bins_bytes, const float* lo, const float* hi,
                  const int32_t* V, int64_t images, int C, int h, int w, int n_bins, int t,
                  int pad, int budget, int groups, float* partial, cudaStream_t st) {
    if (bins_bytes != 1) return QFCA_ERR_UNSUPPORTED;
    Score3Geom g;
    size_t smem;
    int rc = score3_plan(h, w, n_bins, t, C, images, groups, pad, budget, V == nullptr, &g,
                         &smem);
    if (rc != QFCA_OK) return rc;
    if (groups > 0 && g.groups != groups) return QFCA_ERR_ARG;
    if (V == nullptr && !g.fref) return QFCA_ERR_UNSUPPORTED;
    void (*kern)(const uint8_t*, const float*, const float*, const int32_t*, const Score3Geom,
                 float*) = nullptr;
    switch (t * 1000 + w) {
#define S3K(TT, WW) case TT * 1000 + WW: kern = k_score3<TT, WW>; break;
        S3K(1, 32) S3K(1, 64) S3K(1, 128) S3K(3, 32) S3K(3, 64) S3K(3, 128)
        S3K(5, 32) S3K(5, 64) S3K(5, 128) S3K(7, 32) S3K(7, 64) S3K(7, 128)
        S3K(9, 32) S3K(9, 64) S3K(9, 128) S3K(11, 32) S3K(11, 64) S3K(11, 128)
        S3K(13, 32) S3K(13, 64) S3K(13, 128) S3K(15, 32) S3K(15, 64) S3K(15, 128)
#undef S3K
        default: return QFCA_ERR_UNSUPPORTED;
    }
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return QFCA_ERR_CUDA;
    const int64_t grid = images * g.groups;
    kern<<<(unsigned)grid, S3_THREADS, smem, st>>>((const uint8_t*)bins, lo, hi, V, g, partial);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
