// score6.cu -- K4 v6: the fused scoring kernel for 128-wide planes (the
// 128 x 128 feature planes of 1024^2 textures, configs[2]; the 256 x 128
// tiles of wide planes, configs[4]).
//
// Same mathematics and the same fp32 arithmetic sequence as score3.cu (see
// score2.cu's header for the closed forms), so v6 reproduces v3 bit for bit;
// a different schedule, built from the ncu profile of v3 (shared-memory
// wavefronts ~5 per (channel, pixel) and ~35% barrier stalls of its
// producer / consumer warps):
//
//   phase 1  window counts of the whole plane, all 16 warps: vertical
//            windows (H1, four threads per column, each sliding over a quarter
//            of the rows) into a staging band of 32 rows, then the row windows
//            (H2, 8-column segments, one task per thread) -> the cumulative
//            thermometer counts of every pixel go to a per-SM scratch in
//            global memory (L2-resident, word-major rows: [row][word][x]) and
//            the sample-grid pixels' counts to SA4 in shared memory.  Counts
//            are computed once per channel (v3 computed them twice).
//   phase 2  the median-quan reference of all bins by lock-step binary search
//            over SA4 (score4.cu's packed compares);
//   phase 3  the transport tables G_i(v);
//   phase 4  stream rows in sub-chunks of CH = 4 rows (period lcm(T, CH), so the E
//            ring stays in registers with static indices): thread (x, group
//            g) loads its two count words straight from the scratch (loads of
//            the next sub-chunk in flight during this one), computes E for
//            each of its 4 bins only when some lane of the warp has mass in
//            that bin (per-bin, not per-group, warp vote), keeps the vertical
//            box in the register ring, and stores the vertical sums of bin i
//            only when some lane's window has bin i (the own-bin gather can
//            only read those); the own-bin horizontal box of the previous
//            sub-chunk runs in the same phase from the other Vb buffer, so
//            there is ONE barrier per sub-chunk and every warp does the same
//            work.
// Degenerate channels are skipped outright.  The scratch is indexed by %smid:
// the kernel's shared memory (> 114 KB) keeps one CTA per SM.
#include <string.h>

#include "common.cuh"

namespace qfca {

constexpr int S6_THREADS = 512;
constexpr int S6_W = 128;
constexpr int S6_BAND = 8;                 // H1 steps per band (x 4 quarters = 32 rows)
constexpr int S6_SLOTS = 4 * S6_BAND;      // staging rows
constexpr int S6_SEG = 8;                  // H2 columns per task
constexpr int S6_SMEM_MAX = 227 * 1024;
constexpr int S6_MAXNB = 256;              // bins (17 passes)
// Vb row pitch: the 128 columns plus mirrored copies of the R <= 7 edge
// columns on both sides (padded to a multiple of 32 floats, so lanes reading
// different bins' rows at consecutive columns stay in distinct banks)
constexpr int S6_VP = S6_W + 32;
constexpr int S6_VO = 16;                  // column 0's position in a Vb row

struct Score6Geom {
    int h, n_bins, pad, C, groups, cpg;
    int S;      // stream rows h + 2R
    int qrows;  // H1 rows per quarter, ceil(h / 4)
    int fref, stride, sshift, nsx, nsamp;  // sshift = log2(stride) or -1
    int dbsb;   // bins double-buffered (next channel prefetched)
    int passes;  // bin passes (16 lanes each, 15 new bins after the first)
    uint32_t moff;
    int o_sb, o_sa, o_stg, o_gt, o_xmap, o_rmap, o_stab, o_pj, o_misc, total;
    // tile source (wide planes, sharding.py strips): "image" i of the launch is
    // tile (i / ncs, i % ncs) of the C big planes (hbig x wbig) -- rows rst[.],
    // columns cst[.] -- read in place (no gathered copy); csz = copy bytes
    const int* rst;
    const int* cst;
    int tsrc, ncs, hbig, wbig, csz;
};

__device__ __forceinline__ void cp_async_n(void* smem, const void* gmem, int n) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    if (n == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
    else if (n == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}

__device__ __forceinline__ float rcp_approx6(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <int OFF>
__device__ __forceinline__ float lds6_f32(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF));
    return v;
}
// thermometer words of bin b for a pass whose lanes count bins <= tb .. tb + 15
// (lane j of word q = [b <= tb + 4q + j]) by ALU: 0x01010101 shifted left by
// 8 (b - tb - 4q) bytes, clamped (shf.l.clamp gives 0 past 32 bits) -- no
// shared-memory table lookup on the phase-1 critical path
__device__ __forceinline__ uint4 thermo6(int b, int tb) {
    const int s = 8 * (b - tb);
    return make_uint4(__funnelshift_lc(0u, 0x01010101u, max(s, 0)),
                      __funnelshift_lc(0u, 0x01010101u, max(s - 32, 0)),
                      __funnelshift_lc(0u, 0x01010101u, max(s - 64, 0)),
                      __funnelshift_lc(0u, 0x01010101u, max(s - 96, 0)));
}
__device__ __forceinline__ uint32_t smid6() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// staging element of padded column p: one pad element after every 8 columns,
// so the 8-column H2 segments of a quarter-warp start in distinct bank groups
__host__ __device__ constexpr int s6_elem(int p) { return p + (p >> 3); }

// stream rows per sub-chunk (one barrier each) and rows per unrolled period:
// the period is a multiple of T, so the E ring keeps static register slots
// (4 rows: one own-bin box row per bin group and a quarter fewer barriers than
// 3; T = 15 keeps 3, its 60-row period with 4 measured slower)
template <int T>
__host__ __device__ constexpr int s6_ch() { return T == 15 ? 3 : 4; }
__host__ __device__ constexpr int s6_gcd(int a, int b) { return b == 0 ? a : s6_gcd(b, a % b); }
template <int T>
__host__ __device__ constexpr int s6_period() { return T / s6_gcd(T, s6_ch<T>()) * s6_ch<T>(); }

template <int T>
static void score6_layout(Score6Geom& g) {
    constexpr int R = T / 2;
    constexpr int CH = s6_ch<T>();
    constexpr int GP = T * T + 1;
    const int wpp = s6_elem(S6_W + 2 * R) + 1;
    int off = 0;
    auto take = [&](long long bytes) {
        const int o = off;
        off = (int)((off + bytes + 15) & ~15LL);
        return o;
    };
    g.o_sb = take((long long)(g.dbsb ? 2 : 1) * g.h * S6_W);
    // SA4 (phases 1-2) and Vb (phase 4, 2 x CH rows x 16 bins x S6_VP) share one region
    const long long sa = (long long)g.nsamp * 16;
    const long long vb = 2LL * CH * 16 * S6_VP * 4;
    g.o_sa = take(sa > vb ? sa : vb);
    g.o_stg = take((long long)S6_SLOTS * wpp * 16);
    g.o_gt = take(16LL * GP * 4);  // the current pass's 16 bins
    g.o_pj = take((long long)GP * 4);
    g.o_xmap = take((long long)(S6_W + 2 * R) * 4);
    constexpr int P = s6_period<T>();
    const int n_chunks = (g.S + P - 1) / P;
    g.o_rmap = take((long long)(n_chunks * P + 2 * CH) * 4);
    g.o_stab = take((long long)g.h * 8);
    g.o_misc = take(2048);  // scale, V[256], search brackets / mids / per-warp counts
    g.total = off;
}

template <int T, bool MP>  // MP: more than 16 bins (several bin passes)
__global__ void __launch_bounds__(S6_THREADS, 1)
k_score6(const uint8_t* __restrict__ bins, const float* __restrict__ lo,
         const float* __restrict__ hi, const int32_t* __restrict__ Vref, const Score6Geom g,
         uint32_t* __restrict__ scratch, float* __restrict__ partial) {
    constexpr int W = S6_W;
    constexpr int R = T / 2;
    constexpr int T2 = T * T;
    constexpr int GP = T2 + 1;
    constexpr int CH = s6_ch<T>();
    constexpr int P = s6_period<T>();        // stream rows per unrolled period
    constexpr int NSUB = P / CH;             // sub-chunks per period
    constexpr int WPP = s6_elem(W + 2 * R) + 1;
    constexpr uint32_t FULL = 0xffffffffu;
    extern __shared__ __align__(16) uint8_t sm[];
    uint8_t* const sbase = sm + g.o_sb;
    uint4* const SA4 = reinterpret_cast<uint4*>(sm + g.o_sa);
    float* const Vb = reinterpret_cast<float*>(sm + g.o_sa);
    uint4* const STG = reinterpret_cast<uint4*>(sm + g.o_stg);
    float* const GT = reinterpret_cast<float*>(sm + g.o_gt);
    float* const sPJ = reinterpret_cast<float*>(sm + g.o_pj);
    int* const xmap = reinterpret_cast<int*>(sm + g.o_xmap);
    int* const rmap = reinterpret_cast<int*>(sm + g.o_rmap);
    int2* const stab = reinterpret_cast<int2*>(sm + g.o_stab);
    float* const sscale = reinterpret_cast<float*>(sm + g.o_misc);      // [1]
    int* const sV = reinterpret_cast<int*>(sm + g.o_misc + 16);         // [S6_MAXNB]
    int* const blo = reinterpret_cast<int*>(sm + g.o_misc + 1088);      // [16]
    int* const bhi = reinterpret_cast<int*>(sm + g.o_misc + 1152);      // [16]
    uint8_t* const qm8 = sm + g.o_misc + 1216;                           // [16]
    uint32_t* const cnt = reinterpret_cast<uint32_t*>(sm + g.o_misc + 1280);  // [16 warps][8]

    const int tid = threadIdx.x;
    const int h = g.h;
    const int hw = h * W;
    const int img = blockIdx.x / g.groups, cgi = blockIdx.x % g.groups;
    const int c_begin = cgi * g.cpg, c_end = min(g.C, c_begin + g.cpg);
    float* const part = partial + ((int64_t)img * g.groups + cgi) * hw;
    uint32_t* const scr = scratch + (size_t)smid6() * (size_t)(h + 1) * 4 * W;
    const int n_chunks = (g.S + P - 1) / P;

    // ---- per-CTA tables
    for (int p = tid; p < W + 2 * R; p += S6_THREADS) xmap[p] = map_coord(p - R, W, g.pad);
    // stream rows past the plane read row h of the scratch: all-zero counts, so
    // E = 0 there without a branch
    for (int s = tid; s < n_chunks * P + 2 * CH; s += S6_THREADS)
        rmap[s] = s < g.S ? map_coord(s - R, h, g.pad) : h;
    for (int e = tid; e < h; e += S6_THREADS)
        stab[e] = make_int2(map_coord(e + R, h, g.pad) * W, map_coord(e - 1 - R, h, g.pad) * W);
    for (int i = tid; i < 4 * W; i += S6_THREADS) scr[(size_t)h * 4 * W + i] = 0u;
    // the bins of channel c of this image / tile -> dst (asynchronous)
    auto load_bins = [&](uint8_t* dst, int c) {
        if (!g.tsrc) {
            const uint8_t* const src = bins + ((int64_t)img * g.C + c) * hw;
            for (int i = tid; i < hw / 16; i += S6_THREADS) cp_async16(dst + 16 * i, src + 16 * i);
        } else {
            const int r = img / g.ncs, s_ = img - r * g.ncs;
            const uint8_t* const src =
                bins + ((int64_t)c * g.hbig + g.rst[r]) * g.wbig + g.cst[s_];
            const int per_row = W / g.csz;
            for (int i = tid; i < h * per_row; i += S6_THREADS) {
                const int y = i / per_row, k = i - y * per_row;
                cp_async_n(dst + y * W + k * g.csz, src + (int64_t)y * g.wbig + k * g.csz, g.csz);
            }
        }
    };
    if (c_begin < c_end) load_bins(sbase, c_begin);  // bins of the first channel

    __syncthreads();  // xmap (read below by every thread) complete
    // phase-1 roles: H1 thread (column col, quarter q); H2 task (slot, segment)
    const int col = tid & (W - 1), q1 = tid >> 7;
    const int hy0 = q1 * g.qrows, hy1 = min(h, hy0 + g.qrows);
    int halo0 = -1, halo1 = -1;  // padded columns (other than col + R) that map to col
    for (int j = 0; j < 2 * R; ++j) {
        const int p = j < R ? j : W + j;
        if (xmap[p] == col) {
            if (halo0 < 0) halo0 = p;
            else if (halo1 < 0) halo1 = p;
        }
    }
    const int t_slot = tid >> 4, t_seg = tid & 15;
    const int t_q = t_slot >> 3, t_k = t_slot & 7;
    // phase-4 roles: thread (column x, bin group grp)
    const int x = tid & (W - 1), grp = tid >> 7;
    // a pass's 16 thermometer lanes count bins <= tb .. tb + 15 (thermo6)
    int thb = 0;
    auto build_th = [&](int tb) {
        thb = tb;
        if (MP) __syncthreads();  // the previous pass's readers of the scratch are done
    };

    int buf = 0;
    for (int c = c_begin; c < c_end; ++c) {
        const int64_t plane = (int64_t)img * g.C + c;
        const uint8_t* const sb = sbase + (g.dbsb ? buf * hw : 0);
        if (tid == 0) {
            float sc = 0.f;
            if (hi[plane] > lo[plane])
                sc = (float)(((double)hi[plane] - (double)lo[plane]) / (double)g.n_bins /
                             (double)T2);
            sscale[0] = sc;
        }
        if (!g.fref)
            for (int i = tid; i < S6_MAXNB; i += S6_THREADS)
                sV[i] = i < g.n_bins ? __ldg(Vref + plane * g.n_bins + i) : T2;
        cp_async_wait_all();
        __syncthreads();
        const float scale = sscale[0];
        if (scale == 0.f) {  // degenerate channel: skipped (scoring.py:265-266)
            __syncthreads();  // every thread has read sscale before tid 0 rewrites it
            if (!g.dbsb) {
                if (c + 1 < c_end) load_bins(sbase, c + 1);
            } else {
                buf ^= 1;
                if (c + 1 < c_end) load_bins(sbase + buf * hw, c + 1);
            }
            continue;
        }
        // prefetch the next channel's bins into the other buffer
        if (g.dbsb && c + 1 < c_end) load_bins(sbase + (buf ^ 1) * hw, c + 1);

        // ======== phase 1: window counts -> scratch (word-major rows) + SA4 samples
        auto phase1 = [&](bool samples) {
            uint4 cst = make_uint4(0, 0, 0, 0);
            const uint8_t* const pb = sb + col;
            if (hy0 < hy1) {  // window sum of row hy0 - 1: the slide starts there
#pragma unroll
                for (int dy = -R; dy <= R; ++dy) {
                    const uint4 a = thermo6(pb[map_coord(hy0 - 1 + dy, h, g.pad) * W], thb);
                    cst.x += a.x;
                    cst.y += a.y;
                    cst.z += a.z;
                    cst.w += a.w;
                }
            }
            for (int kb = 0; kb < g.qrows; kb += S6_BAND) {
                // H1: S6_BAND rows of this quarter -> staging slots q1 * 8 + kk
                // (cst enters as the window sum of row hy0 + kb - 1)
                // the bin bytes of BPG rows first, then their windows and staging
                // stores -- a store before a load keeps the compiler from issuing the
                // load early (it cannot prove the two disjoint): the whole band at
                // T <= 11 (-1.6 % at T = 9), half bands at T >= 13 (registers)
                constexpr int BPG = T <= 11 ? S6_BAND : S6_BAND / 2;
#pragma unroll
                for (int k0 = 0; k0 < S6_BAND; k0 += BPG) {
                    int ba[BPG], br[BPG];
#pragma unroll
                    for (int e = 0; e < BPG; ++e) {
                        const int y = hy0 + kb + k0 + e;
                        ba[e] = br[e] = 0;
                        if (y < hy1) {
                            const int2 st = stab[y];
                            ba[e] = pb[st.x];
                            br[e] = pb[st.y];
                        }
                    }
#pragma unroll
                    for (int e = 0; e < BPG; ++e) {
                        const int kk = k0 + e;
                        const int y = hy0 + kb + kk;
                        if (y < hy1) {
                            const uint4 a = thermo6(ba[e], thb), r = thermo6(br[e], thb);
                            cst.x += a.x - r.x;
                            cst.y += a.y - r.y;
                            cst.z += a.z - r.z;
                            cst.w += a.w - r.w;
                            uint4* row = STG + (q1 * S6_BAND + kk) * WPP;
                            row[s6_elem(col + R)] = cst;
                            if (halo0 >= 0) row[s6_elem(halo0)] = cst;
                            if (halo1 >= 0) row[s6_elem(halo1)] = cst;
                        }
                    }
                }
                __syncthreads();
                // H2: task (slot, 8-column segment) -> 8 cumulative counts
                {
                    const int y = t_q * g.qrows + kb + t_k;
                    if (kb + t_k < g.qrows && y < min(h, (t_q + 1) * g.qrows)) {
                        const int x0 = t_seg * S6_SEG;
                        const uint4* src = STG + t_slot * WPP + 9 * t_seg;  // elem(x0)
                        uint4 out[S6_SEG];
                        uint4 sum = make_uint4(0, 0, 0, 0);
#pragma unroll
                        for (int p = 0; p < T; ++p) {
                            const uint4 v = src[s6_elem(p)];
                            sum.x += v.x;
                            sum.y += v.y;
                            sum.z += v.z;
                            sum.w += v.w;
                        }
                        out[0] = sum;
#pragma unroll
                        for (int k = 1; k < S6_SEG; ++k) {
                            const uint4 a = src[s6_elem(k + 2 * R)], rr = src[s6_elem(k - 1)];
                            sum.x += a.x - rr.x;
                            sum.y += a.y - rr.y;
                            sum.z += a.z - rr.z;
                            sum.w += a.w - rr.w;
                            out[k] = sum;
                        }
                        if (samples) {
                            if (g.sshift >= 0) {  // power-of-two stride
                                const int sm1 = (1 << g.sshift) - 1;
                                if ((y & sm1) == 0) {
                                    uint4* sa = SA4 + (y >> g.sshift) * g.nsx;
#pragma unroll
                                    for (int k = 0; k < S6_SEG; ++k)
                                        if (((x0 + k) & sm1) == 0) sa[(x0 + k) >> g.sshift] = out[k];
                                }
                            } else if (y % g.stride == 0) {
                                uint4* sa = SA4 + (y / g.stride) * g.nsx;
#pragma unroll
                                for (int k = 0; k < S6_SEG; ++k)
                                    if ((x0 + k) % g.stride == 0) sa[(x0 + k) / g.stride] = out[k];
                            }
                        }
                        uint32_t* dst = scr + (size_t)y * 4 * W + x0;
                        reinterpret_cast<uint4*>(dst)[0] = make_uint4(out[0].x, out[1].x, out[2].x, out[3].x);
                        reinterpret_cast<uint4*>(dst)[1] = make_uint4(out[4].x, out[5].x, out[6].x, out[7].x);
                        reinterpret_cast<uint4*>(dst + W)[0] = make_uint4(out[0].y, out[1].y, out[2].y, out[3].y);
                        reinterpret_cast<uint4*>(dst + W)[1] = make_uint4(out[4].y, out[5].y, out[6].y, out[7].y);
                        reinterpret_cast<uint4*>(dst + 2 * W)[0] = make_uint4(out[0].z, out[1].z, out[2].z, out[3].z);
                        reinterpret_cast<uint4*>(dst + 2 * W)[1] = make_uint4(out[4].z, out[5].z, out[6].z, out[7].z);
                        reinterpret_cast<uint4*>(dst + 3 * W)[0] = make_uint4(out[0].w, out[1].w, out[2].w, out[3].w);
                        reinterpret_cast<uint4*>(dst + 3 * W)[1] = make_uint4(out[4].w, out[5].w, out[6].w, out[7].w);
                    }
                }
                __syncthreads();
            }
        };

        // ======== phase 2: reference (smallest v with #{samples: A_i <= v} >= S - m)
        // of the pass's bins tb + klo .. tb + 15 (lane 0 of a later pass is the
        // previous pass's last threshold)
        auto search = [&](int tb, int klo) {
            constexpr int ROUNDS = T2 < 2 ? 1 : (T2 < 4 ? 2 : (T2 < 8 ? 3 : (T2 < 16 ? 4 :
                                   (T2 < 32 ? 5 : (T2 < 64 ? 6 : (T2 < 128 ? 7 : 8))))));
            // counts <= 127: four 8-bit compares per word; up to 255 (T = 13, 15):
            // the word's lanes widened to two words of 16-bit lanes
            constexpr bool WIDE = T2 > 126;
            constexpr int WPS = S6_THREADS / 32;
            const int c0 = g.nsamp - (g.nsamp - 1) / 2;
            if (tid < 16) {
                const int top = (tid >= klo && tb + tid < g.n_bins - 1) ? 0 : T2;
                blo[tid] = top;
                bhi[tid] = T2;
                qm8[tid] = (uint8_t)((top + T2) >> 1);
            }
            __syncthreads();
            const uint32_t* const qm = reinterpret_cast<const uint32_t*>(qm8);
#pragma unroll 1
            for (int r = 0; r < ROUNDS; ++r) {
                uint32_t Q[4], acc[4] = {0u, 0u, 0u, 0u};
                uint32_t QE[4], QO[4], ace[4] = {0u, 0u, 0u, 0u}, aco[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    Q[qq] = 0x80808080u | qm[qq];
                    QE[qq] = 0x80008000u | (qm[qq] & 0x00FF00FFu);
                    QO[qq] = 0x80008000u | ((qm[qq] >> 8) & 0x00FF00FFu);
                }
                for (int s = tid; s < g.nsamp; s += S6_THREADS) {
                    const uint4 v = SA4[s];
                    const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        if (WIDE) {  // 16-bit lanes (even / odd bytes), counts <= 255
                            ace[qq] += ((QE[qq] - (vw[qq] & 0x00FF00FFu)) & 0x80008000u) >> 15;
                            aco[qq] += ((QO[qq] - ((vw[qq] >> 8) & 0x00FF00FFu)) & 0x80008000u) >> 15;
                        } else {
                            acc[qq] += __umulhi((Q[qq] - vw[qq]) & 0x80808080u, 1u << 25);
                        }
                    }
                }
                uint32_t* cp = cnt + (tid >> 5) * 8;
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                    const uint32_t ev = __reduce_add_sync(FULL, WIDE ? ace[qq] : acc[qq] & 0x00FF00FFu);
                    const uint32_t od =
                        __reduce_add_sync(FULL, WIDE ? aco[qq] : (acc[qq] >> 8) & 0x00FF00FFu);
                    if ((tid & 31) == 0) {
                        cp[2 * qq] = ev;
                        cp[2 * qq + 1] = od;
                    }
                }
                __syncthreads();
                if (tid < 16) {
                    const int i = tid, j = i & 3, qq = i >> 2;
                    uint32_t word = 0;  // 16-bit fields: nsamp < 65536
#pragma unroll
                    for (int w = 0; w < WPS; ++w) word += cnt[w * 8 + 2 * qq + (j & 1)];
                    const int count = (int)((j >> 1) ? word >> 16 : word & 0xFFFFu);
                    int a = blo[i], bnd = bhi[i];
                    const int mid = (a + bnd) >> 1;
                    if (count >= c0) bnd = mid; else a = mid + 1;
                    blo[i] = a;
                    bhi[i] = bnd;
                    qm8[i] = (uint8_t)((a + bnd) >> 1);
                }
                __syncthreads();
            }
            if (tid >= klo && tid < 16) sV[tb + tid] = blo[tid];
            __syncthreads();
        };

        const int npass = MP ? g.passes : 1;
        if (g.fref)
            for (int p = 0; p < npass; ++p) {
                build_th(15 * p);
                phase1(true);
                search(15 * p, p > 0 ? 1 : 0);
            }

        // ======== phase 3: PJ = prefix of J, G_i(v) for every bin and count
        for (int qq = tid; qq < T2; qq += S6_THREADS) {
            int a = 0, bnd = g.n_bins - 1;
            while (a < bnd) {
                const int mid = (a + bnd) >> 1;
                if (sV[mid] > qq) bnd = mid; else a = mid + 1;
            }
            sPJ[qq + 1] = (float)a;
        }
        __syncthreads();
        if (tid < 32) {
            const int lane = tid;
            float carry = 0.f;
            if (lane == 0) sPJ[0] = 0.f;
            for (int base = 1; base <= T2; base += 32) {
                const int qq = base + lane;
                float v = qq <= T2 ? sPJ[qq] : 0.f;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float u = __shfl_up_sync(FULL, v, o);
                    if (lane >= o) v += u;
                }
                v += carry;
                if (qq <= T2) sPJ[qq] = v;
                carry = __shfl_sync(FULL, v, 31);
            }
        }
        __syncthreads();
        // G_i(v) of the pass's 16 bins tb .. tb + 15 (rebuilt per bin pass)
        auto build_gt = [&](int tb) {
            for (int idx = tid; idx < 16 * GP; idx += S6_THREADS) {
                const int j = idx / GP, v = idx - j * GP, i = tb + j;
                float vm = 0.f, d = 0.f;
                if (i < g.n_bins) {
                    const int vmi = i > 0 ? sV[i - 1] : 0;
                    vm = (float)vmi;
                    d = 2.f * ((float)i * vm - sPJ[vmi]);
                }
                const float fv = (float)v;
                const float nu = fmaf((float)i, fv, -sPJ[v]);
                GT[idx] = fv < vm ? nu : d - nu;
            }
            __syncthreads();  // GT ready; SA4 free (Vb aliases it)
        };

        // ======== phase 4: E (register ring) + own-bin box, one barrier per sub-chunk.
        // T = 5..11: each thread's count words of sub-chunk u + 2 are loaded from the
        // L2-resident scratch into registers while sub-chunk u runs (-1 % at T = 9);
        // T >= 13 (the E ring needs the registers) and T = 3 (measured +3 % with
        // the register path): the count rows of sub-chunk
        // u + 2 are copied (cp.async) from the scratch into a 3-slot ring in the
        // (now free) staging region; each slot is [row][word][x].  A pass scores the pixels whose bin
        // is in [bin_lo, bin_hi]; its lanes are bins tb .. tb + 15.
        auto phase4 = [&](int tb, int bin_lo, int bin_hi) {
            const uint32_t gaddr =
                (uint32_t)__cvta_generic_to_shared(GT + grp * 4 * GP) + g.moff;
            constexpr bool RP = T >= 5 && T <= 11;  // register prefetch (else the cp.async ring)
            const bool g1 = grp > 0;
            const uint32_t* const scol = scr + grp * W + x;
            auto load_words = [&](int sub, uint32_t (&wd)[CH], uint32_t (&pv)[CH]) {
#pragma unroll
                for (int rr = 0; rr < CH; ++rr) {
                    const uint32_t* const p_ = scol + (size_t)rmap[sub * CH + rr] * 4 * W;
                    wd[rr] = __ldcg(p_);  // (written by phase 1 of this CTA: L2, not L1)
                    pv[rr] = g1 ? __ldcg(p_ - W) : 0u;
                }
            };
            uint32_t wA[CH], pA[CH], wB[CH], pB[CH];
            uint32_t* const cring = reinterpret_cast<uint32_t*>(STG);
            constexpr int SLOT = CH * 4 * W;  // uint32 per slot
            const int n_sub = n_chunks * NSUB;
            // copy tasks (row of the sub-chunk, 16-byte piece): 128 pieces per 2 KB row
            constexpr int NCP = (CH * 128 + S6_THREADS - 1) / S6_THREADS;
#define S6_COPY(SUB)                                                            \
    {                                                                           \
        const int sub_ = (SUB);                                                 \
        if (!RP && sub_ < n_sub) {                                              \
            uint32_t* const dst_ = cring + (sub_ % 3) * SLOT;                   \
            _Pragma("unroll") for (int k_ = 0; k_ < NCP; ++k_) {                \
                const int task_ = (S6_THREADS - 1 - tid) + S6_THREADS * k_;     \
                if (task_ < CH * 128) {                                         \
                    const int rr_ = task_ >> 7, pc_ = 4 * (task_ & 127);        \
                    const int row_ = rmap[sub_ * CH + rr_];                     \
                    cp_async16(dst_ + rr_ * 4 * W + pc_, scr + (size_t)row_ * 4 * W + pc_); \
                }                                                               \
            }                                                                   \
        }                                                                       \
        asm volatile("cp.async.commit_group;" ::: "memory");                    \
    }
            if (RP) {
                load_words(0, wA, pA);
                load_words(1, wB, pB);
            } else {
                S6_COPY(0)
                S6_COPY(1)
                asm volatile("cp.async.wait_group 1;" ::: "memory");
                __syncthreads();  // slot 0 visible
            }
            float ring[T][4];
            bool mring[T];  // group mass of the last T stream rows (static slots)
            float vs[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                vs[j] = 0.f;
#pragma unroll
                for (int qq = 0; qq < T; ++qq) ring[qq][j] = 0.f;
            }
#pragma unroll
            for (int qq = 0; qq < T; ++qq) mring[qq] = false;
            // own-bin box rows of a sub-chunk: row a * 4 + ((grp + 3) & 3), so bin
            // group 0 (mass in nearly every window, the longest E) boxes last
            const int arow0 = (grp + 3) & 3;
            // the padded position (if any) that mirrors column x: the box then
            // reads Vb rows straight, without index reflection
            constexpr int NOM = 1 << 20;  // no mirror position
            int xm = NOM;
            if (g.pad == QFCA_PAD_REFLECT) {
                if (x >= 1 && x <= R) xm = -x;
                else if (x >= W - 1 - R && x <= W - 2) xm = 2 * (W - 1) - x;
            } else {
                if (x < R) xm = W + x;
                else if (x >= W - R) xm = x - W;
            }
            constexpr int NA = (CH + 3) / 4;
            float pold[NA];  // partial-map values of the rows boxed next
#pragma unroll
            for (int a = 0; a < NA; ++a) pold[a] = 0.f;
            auto own_bin_box = [&](int u, const float* pv, bool last) {
                const float* const vbr = Vb + (size_t)((u & 1) * CH) * 16 * S6_VP + S6_VO;
#pragma unroll
                for (int a = 0; a < NA; ++a) {
                    const int rr = arow0 + 4 * a;
                    const int y = u * CH + rr - 2 * R;
                    if (rr >= CH || y < 0 || y >= h) continue;
                    const int bb = sb[y * W + x];
                    if (MP && (bb < bin_lo || bb > bin_hi)) continue;  // another pass's pixel
                    const float* vb = vbr + (rr * 16 + bb - (MP ? tb : 0)) * S6_VP;
                    float f = 0.f;
#pragma unroll
                    for (int d = -R; d <= R; ++d) f += vb[x + d];
                    const float old = last ? part[y * W + x] : pv[a];
                    part[y * W + x] = old + fmaf(f, scale, 0.f);
                }
            };
            for (int ck = 0; ck < n_chunks; ++ck) {
#pragma unroll
                for (int sc = 0; sc < NSUB; ++sc) {
                    const int u = ck * NSUB + sc;  // sub-chunk index
                    if (!RP) S6_COPY(u + 2)
                    const uint32_t* const cs = cring + (u % 3) * SLOT + grp * W + x;
                    float* const vbw = Vb + (size_t)((u & 1) * CH) * 16 * S6_VP + S6_VO;
                    // ---- E for CH stream rows (rows past the plane read zero counts):
                    // all rows' count words first, one warp vote per sub-chunk, then
                    // the CH x 4 transports as independent instruction streams
                    uint32_t word[CH], prev[CH];
                    bool mass[CH];
                    bool any = false;
#pragma unroll
                    for (int rr = 0; rr < CH; ++rr) {
                        if (RP) {
                            word[rr] = wA[rr];
                            prev[rr] = pA[rr];
                            wA[rr] = wB[rr];
                            pA[rr] = pB[rr];
                        } else {
                            word[rr] = cs[rr * 4 * W];
                            prev[rr] = g1 ? cs[rr * 4 * W - W] : 0u;
                        }
                    }
                    if (RP) load_words(u + 2, wB, pB);  // (past the plane: the zero row h)
#pragma unroll
                    for (int rr = 0; rr < CH; ++rr) {
                        mass[rr] = (word[rr] >> 24) != (prev[rr] >> 24);  // mass in the group
                        any |= mass[rr];
                    }
                    float E[CH][4];
#pragma unroll
                    for (int rr = 0; rr < CH; ++rr)
#pragma unroll
                        for (int j = 0; j < 4; ++j) E[rr][j] = 0.f;
                    if (__any_sync(FULL, any)) {
#pragma unroll
                        for (int rr = 0; rr < CH; ++rr) {
                            uint32_t ma = __byte_perm(prev[rr], 0x4B000000u, 0x7653);
                            uint32_t aa = gaddr + 4u * ma;
#define S6_E(J)                                                                 \
    {                                                                           \
        const uint32_t mb = __byte_perm(word[rr], 0x4B000000u, 0x7650 + J);     \
        const uint32_t ab = gaddr + 4u * mb;                                    \
        const float gb = lds6_f32<J * GP * 4>(ab);                              \
        const float ga = lds6_f32<J * GP * 4>(aa);                              \
        const float pc = __uint_as_float(mb) - __uint_as_float(ma);             \
        E[rr][J] = (gb - ga) * rcp_approx6(fmaxf(pc, 1.f));                     \
        ma = mb;                                                                \
        aa = ab;                                                                \
    }
                            S6_E(0) S6_E(1) S6_E(2) S6_E(3)
#undef S6_E
                        }
                    }
#pragma unroll
                    for (int rr = 0; rr < CH; ++rr) {
                        const int rho = (sc * CH + rr) % T;  // static ring slot
                        const int s = u * CH + rr;
                        mring[rho] = mass[rr];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            vs[j] += E[rr][j] - ring[rho][j];
                            ring[rho][j] = E[rr][j];
                        }
                        if (rho == T - 1) {
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                float sum = ring[0][j];
#pragma unroll
                                for (int qq = 1; qq < T; ++qq) sum += ring[qq][j];
                                vs[j] = sum;
                            }
                        }
                        const int y = s - 2 * R;
                        // vertical sums of output row y; the own-bin box reads bin i
                        // at (y, x) only if the window centred there holds bin i,
                        // i.e. only if this group has mass there (stream row s - R)
                        if (y >= 0 && y < h && __any_sync(FULL, mring[(rho + T - R) % T])) {
                            float* vb = vbw + (rr * 16 + grp * 4) * S6_VP;
#pragma unroll
                            for (int j = 0; j < 4; ++j) vb[j * S6_VP + x] = vs[j];
                            if (xm != NOM)
#pragma unroll
                                for (int j = 0; j < 4; ++j) vb[j * S6_VP + xm] = vs[j];
                        }
                    }
                    // ---- own-bin horizontal box of sub-chunk u - 1 (other Vb buffer)
                    if (u >= 1) own_bin_box(u - 1, pold, false);
                    // partial-map values for the box of sub-chunk u (next iteration)
#pragma unroll
                    for (int a = 0; a < NA; ++a) {
                        const int rr = arow0 + 4 * a;
                        const int y = u * CH + rr - 2 * R;
                        pold[a] = (rr < CH && y >= 0 && y < h) ? part[y * W + x] : 0.f;
                    }
                    if (!RP) asm volatile("cp.async.wait_group 1;" ::: "memory");  // slot u + 1 landed
                    __syncthreads();
                }
            }
            own_bin_box(n_sub - 1, pold, false);  // the last sub-chunk
        };
#undef S6_COPY
        for (int p = npass - 1; p >= 0; --p) {
            if (!(g.fref && p == npass - 1)) {  // else the last search pass left them
                build_th(15 * p);
                phase1(false);
            }
            if (MP && p != npass - 1) __syncthreads();  // the previous pass's GT readers done
            build_gt(15 * p);
            phase4(15 * p, p == 0 ? 0 : 15 * p + 1, min(15 * p + 15, g.n_bins - 1));
        }
        __syncthreads();
        if (g.dbsb) {
            buf ^= 1;
        } else if (c + 1 < c_end) {
            load_bins(sbase, c + 1);
        }
    }
    cp_async_wait_all();
}

int sample_stride(int h, int w, int budget);

__global__ void k_nsmid(int* out) {
    uint32_t n;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(n));
    *out = (int)n;
}

// %nsmid (an upper bound of %smid) of the current device, read once
static int nsmid_cached() {
    static int n = 0;
    if (n <= 0) {
        int* d = nullptr;
        int v = 0;
        if (cudaMalloc(&d, sizeof(int)) == cudaSuccess) {
            k_nsmid<<<1, 1>>>(d);
            if (cudaMemcpy(&v, d, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) v = 0;
            cudaFree(d);
        }
        int dev = 0, sms = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 148;
        n = v > sms ? v : sms + 32;
    }
    return n;
}

template <int T>
static int s6_total(Score6Geom& g) {
    score6_layout<T>(g);
    return g.total;
}

static int score6_plan(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                       int pad, int budget, bool has_ref, Score6Geom* out, size_t* smem_out) {
    if (w != S6_W || t < 1 || t > 15 || (t & 1) == 0 || n_bins < 1 || n_bins > S6_MAXNB)
        return QFCA_ERR_UNSUPPORTED;
    if (h < 1 || h > 256 || (h * w) % 16) return QFCA_ERR_UNSUPPORTED;
    if (pad != QFCA_PAD_REFLECT && pad != QFCA_PAD_WRAP) return QFCA_ERR_UNSUPPORTED;
    if (!(pad == QFCA_PAD_WRAP || h > 1)) return QFCA_ERR_UNSUPPORTED;
    Score6Geom g;
    memset(&g, 0, sizeof(g));
    g.h = h; g.n_bins = n_bins; g.pad = pad; g.C = C;
    g.S = h + 2 * (t / 2);
    g.qrows = (h + 3) / 4;
    g.moff = 0u - 4u * 0x4B000000u;
    // pass p covers lanes 15p .. 15p + 15: bins 0..15, then 15 new bins per pass
    g.passes = n_bins <= 16 ? 1 : 1 + (n_bins - 16 + 14) / 15;
    if (!has_ref) {
        if (t * t > 255 || budget < 1) return QFCA_ERR_UNSUPPORTED;
        g.fref = 1;
        g.stride = sample_stride(h, w, budget);
        g.sshift = -1;
        for (int k = 0; k < 8; ++k)
            if (g.stride == (1 << k)) g.sshift = k;
        g.nsx = (w + g.stride - 1) / g.stride;
        g.nsamp = ((h + g.stride - 1) / g.stride) * g.nsx;
        if (g.nsamp > 4096 || g.nsamp >= 65536) return QFCA_ERR_UNSUPPORTED;
    }
    size_t bytes = 0;
    for (int db = 1; db >= 0; --db) {
        g.dbsb = db;
        switch (t) {
#define S6C(TT) case TT: bytes = s6_total<TT>(g); break;
            S6C(1) S6C(3) S6C(5) S6C(7) S6C(9) S6C(11) S6C(13) S6C(15)
#undef S6C
            default: return QFCA_ERR_UNSUPPORTED;
        }
        if (bytes <= (size_t)S6_SMEM_MAX) break;
    }
    if (bytes > (size_t)S6_SMEM_MAX || bytes <= 114 * 1024) return QFCA_ERR_UNSUPPORTED;
    int groups = groups_hint;
    if (groups <= 0) groups = balanced_groups(images, C, 1, 1);
    groups = groups < 1 ? 1 : (groups > C ? C : groups);
    g.cpg = (C + groups - 1) / groups;
    g.groups = (C + g.cpg - 1) / g.cpg;
    *out = g;
    *smem_out = bytes;
    return QFCA_OK;
}

int score6_query(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                 int pad, int budget, int want_fref, int* fref) {
    Score6Geom g;
    size_t smem;
    if (score6_plan(h, w, n_bins, t, C, images, groups_hint, pad, budget, want_fref == 0, &g,
                    &smem) != QFCA_OK)
        return -1;
    if (fref) *fref = g.fref;
    return g.groups;
}

int64_t score6_scratch_bytes(int h) {
    return (int64_t)nsmid_cached() * (h + 1) * 4 * S6_W * 4;
}

int launch_score6_src(const void* bins, int bins_bytes, const float* lo, const float* hi,
                      const int32_t* V, int64_t images, int C, int h, int w, int n_bins, int t,
                      int pad, int budget, int groups, void* scratch, int64_t scratch_bytes,
                      float* partial, cudaStream_t st, const int* rst, const int* cst, int ncs,
                      int hbig, int wbig, int csz);

int launch_score6(const void* bins, int bins_bytes, const float* lo, const float* hi,
                  const int32_t* V, int64_t images, int C, int h, int w, int n_bins, int t,
                  int pad, int budget, int groups, void* scratch, int64_t scratch_bytes,
                  float* partial, cudaStream_t st) {
    return launch_score6_src(bins, bins_bytes, lo, hi, V, images, C, h, w, n_bins, t, pad, budget,
                             groups, scratch, scratch_bytes, partial, st, nullptr, nullptr, 0, 0,
                             0, 0);
}

int launch_score6_src(const void* bins, int bins_bytes, const float* lo, const float* hi,
                      const int32_t* V, int64_t images, int C, int h, int w, int n_bins, int t,
                      int pad, int budget, int groups, void* scratch, int64_t scratch_bytes,
                      float* partial, cudaStream_t st, const int* rst, const int* cst, int ncs,
                      int hbig, int wbig, int csz) {
    if (bins_bytes != 1) return QFCA_ERR_UNSUPPORTED;
    if (!scratch || scratch_bytes < score6_scratch_bytes(h)) return QFCA_ERR_ARG;
    Score6Geom g;
    size_t smem;
    int rc = score6_plan(h, w, n_bins, t, C, images, groups, pad, budget, V != nullptr, &g, &smem);
    if (rc != QFCA_OK) return rc;
    if (groups > 0 && g.groups != groups) return QFCA_ERR_ARG;
    g.rst = rst;
    g.cst = cst;
    g.tsrc = rst != nullptr;
    g.ncs = ncs;
    g.hbig = hbig;
    g.wbig = wbig;
    g.csz = csz;
    if (g.tsrc && (ncs < 1 || (csz != 4 && csz != 8 && csz != 16) || wbig % csz ||
                   (reinterpret_cast<uintptr_t>(bins) % csz)))
        return QFCA_ERR_ARG;
    void (*kern)(const uint8_t*, const float*, const float*, const int32_t*, const Score6Geom,
                 uint32_t*, float*) = nullptr;
    const bool mp = g.passes > 1;
    switch (t) {
#define S6K(TT) case TT: kern = mp ? k_score6<TT, true> : k_score6<TT, false>; break;
        S6K(1) S6K(3) S6K(5) S6K(7) S6K(9) S6K(11) S6K(13) S6K(15)
#undef S6K
        default: return QFCA_ERR_UNSUPPORTED;
    }
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return QFCA_ERR_CUDA;
    const int64_t grid = images * g.groups;
    kern<<<(unsigned)grid, S6_THREADS, smem, st>>>((const uint8_t*)bins, lo, hi, V, g,
                                                   (uint32_t*)scratch, partial);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
