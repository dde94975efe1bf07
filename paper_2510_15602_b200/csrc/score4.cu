// score4.cu -- K4 v4: plane-resident fused scoring kernel.
//
// Same mathematics as score2.cu / score3.cu (closed-form transport, E ring,
// own-bin box; see score2.cu's header), different data flow.  When every
// pixel is a reference sample (sample stride 1, quantize.py:109-116) the
// window counts of the whole channel batch fit in shared memory, so each
// channel batch runs as
//
//   pass 0  all warps: vertical windows (H1, four threads per column, each
//           sliding over a quarter of the rows) into SA4 in place, then the
//           row windows (H2) over 2T staged rows at a time -> the cumulative
//           counts of every pixel, pixel-major (one uint4 = 16 8-bit
//           thermometer lanes per pixel) in SA4;
//   search  all 16 warps: the median-quan reference V_i of all 16 bins at once
//           -- a lock-step binary search whose counting pass compares the 16
//           lanes of each SA4 word against 16 packed thresholds
//           (0x80 | mid) - count has bit 7 set iff count <= mid (no borrow
//           because counts <= 127);
//   tables  G_i(v) for every bin i and count v (the piecewise transport
//           potential of score2.cu, same fp32 operations) -> GT;
//   pass 1  E_i = (G_i(A_i) - G_i(A_{i-1})) / max(P_i, 1) from two table
//           reads per bin, vertical box in the register ring -> Vb; then the
//           own-bin horizontal box + partial-map update.
//
// Pass 1 reads SA4 instead of recomputing the windows, the sample scatter of
// score3.cu disappears, and the transport needs no per-bin branch.  The fp32
// transport expressions are score3.cu's; with one channel slot per CTA the
// per-slot sums are added to the partial map one at a time, so the maps agree
// with score3.cu to fp32 rounding.
// With a host-supplied reference (Vref) the search is skipped and any sample
// stride is accepted.
#include <string.h>

#include "common.cuh"

namespace qfca {

// A CTA covers NCOL = CPB * W columns (CPB channel slots of width W) with
// 4 * NCOL threads -- one per (slot, bin group, column) in pass 1; every phase
// uses all of them.
// NCOL = 64 (256 threads, <= 113 KB) keeps two CTAs resident per SM, so one
// CTA's barrier-bound phases overlap the other's transport; NCOL = 128 (512
// threads) takes wider planes.  (Pass 0 uses all 4 NCOL threads: 4 per column
// in H1, SEG-column tasks in H2.)
constexpr int S4_SMEM_MAX = 227 * 1024;
constexpr int S4_SMEM_2CTA = 113 * 1024;

struct Score4Geom {
    int h, n_bins, pad, C, groups, cpg;
    int WPP;   // pass-0 column-word row pitch (uint4)
    int S;     // pass-1 stream rows h + 2r
    int n0;    // pass-0 chunks ceil(h / T)
    int fref;  // 1: reference selected in-kernel (every pixel a sample)
    int nsamp;
    uint32_t moff;  // -4 * 0x4B000000 (mod 2^32): magic-float -> G-table byte offset
    int o_sb, o_sa, o_gt, o_xmap, o_rmap, o_stab, o_scale, o_sv, o_alias, total;
    // inside the alias region (offsets from o_alias)
    int a_chp, a_cnt, a_qm, a_lo, a_hi, a_pj;
};

__device__ __forceinline__ float rcp_approx4(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// fp32 shared load at a 32-bit shared address plus a constant byte offset
template <int OFF>
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF));
    return v;
}

// H2 segment: smallest odd length >= 3 whose tasks fit the consumer threads
__host__ __device__ constexpr int s4_seg(int t, int w, int ncol) {
    int s = 3;
    while (t * (ncol / w) * ((w + s - 1) / s) > 3 * ncol) s += 2;
    return s;
}
__host__ __device__ constexpr int s4_rounds(int t2) {
    int r = 0;
    while ((1 << r) < t2 + 1) ++r;
    return r;
}

// thermometer words of bin b (lane j of word q = [b <= 4q + j]) by ALU: see
// score6.cu's thermo6
__device__ __forceinline__ uint4 thermo4(int b) {
    const int s = 8 * b;
    return make_uint4(__funnelshift_lc(0u, 0x01010101u, s),
                      __funnelshift_lc(0u, 0x01010101u, max(s - 32, 0)),
                      __funnelshift_lc(0u, 0x01010101u, max(s - 64, 0)),
                      __funnelshift_lc(0u, 0x01010101u, max(s - 96, 0)));
}

template <int T, int W, int NCOL>
static void score4_layout(Score4Geom& g) {
    constexpr int CPB = NCOL / W;
    constexpr int T2 = T * T;
    constexpr int SEG = s4_seg(T, W, NCOL);
    constexpr int NSEG = (W + SEG - 1) / SEG;
    const int R = T / 2;
    // row pitch with consecutive H2 tasks on consecutive 16-byte bank groups
    int wpp = W + 2 * R;
    while ((wpp - NSEG * SEG) % 8 != 0) ++wpp;
    g.WPP = wpp;
    int off = 0;
    auto take = [&](long long bytes) {
        const int o = off;
        off = (int)((off + bytes + 15) & ~15LL);
        return o;
    };
    const int n_chunks = (g.S + T - 1) / T;
    g.o_sb = take((long long)CPB * g.h * W);
    g.o_sa = take((long long)CPB * g.h * W * 16);
    g.o_gt = take((long long)CPB * 16 * (T2 + 1) * 4);
    g.o_xmap = take((long long)(W + 2 * R) * 4);
    g.o_rmap = take((long long)n_chunks * T * 4);
    g.o_stab = take((long long)g.h * 8);
    g.o_scale = take((long long)CPB * 4);
    g.o_sv = take((long long)CPB * 16 * 4);
    // alias region: pass 0 (CHp) | search (cnt, qm, lo, hi) + PJ | pass 1 (Vb)
    int a = 0;
    auto atake = [&](long long bytes) {
        const int o = a;
        a = (int)((a + bytes + 15) & ~15LL);
        return o;
    };
    g.a_chp = atake((long long)2 * T * CPB * g.WPP * 16);  // pass-0 H2 staging: 2T padded rows
    const int pass0 = a;
    a = 0;
    g.a_cnt = atake((long long)(4 * NCOL / 32) * 8 * 4);  // per-warp search counts
    g.a_qm = atake((long long)CPB * 16);
    g.a_lo = atake((long long)CPB * 16 * 4);
    g.a_hi = atake((long long)CPB * 16 * 4);
    g.a_pj = atake((long long)CPB * (T2 + 1) * 4);
    const int tables = a;
    const long long vb = (long long)T * CPB * 16 * W * 4;
    long long alias = vb;
    if (pass0 > alias) alias = pass0;
    if (tables > alias) alias = tables;
    g.o_alias = take(alias);
    g.total = off;
}

template <int T, int W, int NCOL>
__global__ void __launch_bounds__(4 * NCOL, NCOL == 64 ? 2 : 1)
k_score4(const uint8_t* __restrict__ bins, const float* __restrict__ lo,
         const float* __restrict__ hi, const int32_t* __restrict__ Vref, const Score4Geom g,
         float* __restrict__ partial) {
    constexpr int S4_THREADS = 4 * NCOL;
    constexpr int R = T / 2;
    constexpr int T2 = T * T;
    constexpr int GP = T2 + 1;     // G-table length per bin
    constexpr int CPB = NCOL / W;  // channel slots: CPB * W = NCOL columns per CTA pass
    constexpr int SEG = s4_seg(T, W, NCOL);
    constexpr int NSEG = (W + SEG - 1) / SEG;
    constexpr int TPS = S4_THREADS / CPB;  // search threads per slot (whole warps)
    constexpr int ROUNDS = s4_rounds(T2);
    static_assert(TPS % 32 == 0, "search warps must not straddle slots");
    extern __shared__ __align__(16) uint8_t sm[];
    uint8_t* const sb = sm + g.o_sb;
    uint4* const SA4 = reinterpret_cast<uint4*>(sm + g.o_sa);
    float* const GT = reinterpret_cast<float*>(sm + g.o_gt);
    int* const xmap = reinterpret_cast<int*>(sm + g.o_xmap);
    int* const rmap = reinterpret_cast<int*>(sm + g.o_rmap);
    int2* const stab = reinterpret_cast<int2*>(sm + g.o_stab);
    float* const sscale = reinterpret_cast<float*>(sm + g.o_scale);
    int* const sV = reinterpret_cast<int*>(sm + g.o_sv);
    uint8_t* const al = sm + g.o_alias;
    uint4* const CHp = reinterpret_cast<uint4*>(al + g.a_chp);
    uint32_t* const cnt = reinterpret_cast<uint32_t*>(al + g.a_cnt);
    uint8_t* const qm8 = al + g.a_qm;
    const uint32_t* const qm = reinterpret_cast<const uint32_t*>(al + g.a_qm);
    int* const blo = reinterpret_cast<int*>(al + g.a_lo);
    int* const bhi = reinterpret_cast<int*>(al + g.a_hi);
    float* const sPJ = reinterpret_cast<float*>(al + g.a_pj);
    float* const Vb = reinterpret_cast<float*>(al);

    const int tid = threadIdx.x;
    const int h = g.h;
    const int hw = h * W;
    const int img = blockIdx.x / g.groups, cgi = blockIdx.x % g.groups;
    const int c_begin = cgi * g.cpg, c_end = min(g.C, c_begin + g.cpg);
    float* const part = partial + ((int64_t)img * g.groups + cgi) * hw;
    const int n_chunks = (g.S + T - 1) / T;

    // ---- per-CTA tables: padded-x map, pass-1 row map, pass-0 slide rows
    for (int p = tid; p < W + 2 * R; p += S4_THREADS) xmap[p] = map_coord(p - R, W, g.pad);
    for (int s = tid; s < n_chunks * T; s += S4_THREADS)
        rmap[s] = s < g.S ? map_coord(s - R, h, g.pad) : 0;
    for (int e = tid; e < h; e += S4_THREADS)
        stab[e] = e == 0 ? make_int2(0, 0)
                         : make_int2(map_coord(e + R, h, g.pad) * W,
                                     map_coord(e - 1 - R, h, g.pad) * W);
    __syncthreads();

    // ---- pass-1 role: thread (slot cs, group grp, column x)
    const int cs = tid / (4 * W);
    const int grp = (tid / W) & 3;
    const int grp4 = grp * 4;
    const bool g1 = (grp & 1) != 0, g2 = (grp & 2) != 0;
    const int x = tid % W;

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
                const uint4* s4 = reinterpret_cast<const uint4*>(bins + plane * hw);
                uint4* d4 = reinterpret_cast<uint4*>(dst);
                for (int i = tid; i < hw / 16; i += S4_THREADS) d4[i] = __ldg(s4 + i);
                if (!g.fref)
                    for (int i = tid; i < 16; i += S4_THREADS)
                        sV[k * 16 + i] = i < g.n_bins ? __ldg(Vref + plane * g.n_bins + i) : T2;
            } else {
                for (int i = tid; i < hw; i += S4_THREADS) dst[i] = 0;
                for (int i = tid; i < 16; i += S4_THREADS) sV[k * 16 + i] = T2;
            }
        }
        __syncthreads();

        // ---- pass 0: window counts of every pixel -> SA4, all warps.
        // (a) vertical windows (H1): four threads per column, each sliding over a
        //     quarter of the rows (one T-row start-up per quarter) -> SA4 in place
        {
            const int col = tid % NCOL, q = tid / NCOL;
            const int slot = col / W, x = col % W;
            const int y0 = q * h / 4, y1 = (q + 1) * h / 4;
            const uint8_t* pb = sb + slot * hw + x;
            uint4* dst = SA4 + slot * hw + x;
            if (y0 < y1) {
                uint4 cst = make_uint4(0, 0, 0, 0);
#pragma unroll 1
                for (int dy = -R; dy <= R; ++dy) {
                    const uint4 a = thermo4(pb[map_coord(y0 + dy, h, g.pad) * W]);
                    cst.x += a.x;
                    cst.y += a.y;
                    cst.z += a.z;
                    cst.w += a.w;
                }
                dst[y0 * W] = cst;
                // the next row's bin bytes are loaded before this row's store (which
                // the compiler cannot prove disjoint from them)
                int na = 0, nr = 0;
                if (y0 + 1 < y1) {
                    const int2 st = stab[y0 + 1];
                    na = pb[st.x];
                    nr = pb[st.y];
                }
                for (int y = y0 + 1; y < y1; ++y) {
                    const int ca = na, cr = nr;
                    if (y + 1 < y1) {
                        const int2 st = stab[y + 1];
                        na = pb[st.x];
                        nr = pb[st.y];
                    }
                    const uint4 a = thermo4(ca), r = thermo4(cr);
                    cst.x += a.x - r.x;
                    cst.y += a.y - r.y;
                    cst.z += a.z - r.z;
                    cst.w += a.w - r.w;
                    dst[y * W] = cst;
                }
            }
        }
        __syncthreads();
        // (b) row windows (H2), 2T rows at a time: copy the rows with their padded
        //     halo into CHp, then sliding sums over segments of SEG columns -> SA4
        for (int yb = 0; yb < h; yb += 2 * T) {
            const int nr = min(2 * T, h - yb);
            constexpr int PW = W + 2 * R;
            for (int idx = tid; idx < nr * CPB * PW; idx += S4_THREADS) {
                const int rc = idx / PW, pp = idx - rc * PW;  // rc = r * CPB + slot
                const int r = rc / CPB, slot = rc - r * CPB;
                CHp[rc * g.WPP + pp] = SA4[(slot * h + yb + r) * W + xmap[pp]];
            }
            __syncthreads();
            for (int task = tid; task < nr * CPB * NSEG; task += S4_THREADS) {
                const int rc = task / NSEG;
                const int x0 = (task - rc * NSEG) * SEG;
                const int r = rc / CPB, slot = rc - r * CPB;
                const uint4* src = CHp + rc * g.WPP + x0;
                uint4* dst = SA4 + (slot * h + yb + r) * W + x0;
                uint4 sum = make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int pq = 0; pq < T; ++pq) {
                    const uint4 v = src[pq];
                    sum.x += v.x;
                    sum.y += v.y;
                    sum.z += v.z;
                    sum.w += v.w;
                }
                dst[0] = sum;
                const int nn = x0 + SEG <= W ? SEG : W - x0;
#pragma unroll
                for (int k = 1; k < SEG; ++k) {
                    if (k >= nn) break;
                    const uint4 a = src[k + 2 * R], rr = src[k - 1];
                    sum.x += a.x - rr.x;
                    sum.y += a.y - rr.y;
                    sum.z += a.z - rr.z;
                    sum.w += a.w - rr.w;
                    dst[k] = sum;
                }
            }
            __syncthreads();
        }

        if (g.fref) {
            // ---- reference: smallest v with #{samples: A_i <= v} >= S - m, all bins at once
            const int c0 = g.nsamp - (g.nsamp - 1) / 2;
            if (tid < CPB * 16) {
                const int k = tid >> 4, i = tid & 15;
                const int top = (i < g.n_bins - 1 && sscale[k] != 0.f) ? 0 : T2;
                blo[tid] = top;
                bhi[tid] = T2;
                qm8[tid] = (uint8_t)((top + T2) >> 1);
            }
            __syncthreads();
            const int k = tid / TPS, lt = tid - k * TPS;
            constexpr int WPS = TPS / 32;  // search warps per slot
            const uint4* sa = SA4 + (size_t)k * g.nsamp;
#pragma unroll 1
            for (int r = 0; r < ROUNDS; ++r) {
                uint32_t Q[4], acc[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                for (int q = 0; q < 4; ++q) Q[q] = 0x80808080u | qm[k * 4 + q];
                for (int s = lt; s < g.nsamp; s += TPS) {
                    const uint4 v = sa[s];
                    acc[0] += __umulhi((Q[0] - v.x) & 0x80808080u, 1u << 25);
                    acc[1] += __umulhi((Q[1] - v.y) & 0x80808080u, 1u << 25);
                    acc[2] += __umulhi((Q[2] - v.z) & 0x80808080u, 1u << 25);
                    acc[3] += __umulhi((Q[3] - v.w) & 0x80808080u, 1u << 25);
                }
                // per-warp sums of the 16-bit count fields (no shared atomics)
                uint32_t* cp = cnt + (tid >> 5) * 8;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t ev = __reduce_add_sync(0xffffffffu, acc[q] & 0x00FF00FFu);
                    const uint32_t od = __reduce_add_sync(0xffffffffu, (acc[q] >> 8) & 0x00FF00FFu);
                    if ((tid & 31) == 0) {
                        cp[2 * q] = ev;
                        cp[2 * q + 1] = od;
                    }
                }
                __syncthreads();
                if (tid < CPB * 16) {
                    const int kk = tid >> 4, i = tid & 15, j = i & 3, q = i >> 2;
                    uint32_t word = 0;  // fields stay < 65536: nsamp < 65536
#pragma unroll
                    for (int w = 0; w < WPS; ++w) word += cnt[(kk * WPS + w) * 8 + 2 * q + (j & 1)];
                    const int count = (int)((j >> 1) ? word >> 16 : word & 0xFFFFu);
                    int a = blo[tid], bnd = bhi[tid];
                    const int mid = (a + bnd) >> 1;
                    if (count >= c0) bnd = mid; else a = mid + 1;
                    blo[tid] = a;
                    bhi[tid] = bnd;
                    qm8[tid] = (uint8_t)((a + bnd) >> 1);
                }
                __syncthreads();
            }
            if (tid < CPB * 16) sV[tid] = blo[tid];
            __syncthreads();
        }
        // ---- PJ = prefix of J, then G_i(v) for every bin and count
        for (int k = 0; k < CPB; ++k) {
            float* pjk = sPJ + k * GP;
            const int* V = sV + k * 16;
            for (int q = tid; q < T2; q += S4_THREADS) {
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
            float* pjk = sPJ + k * GP;
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
        for (int idx = tid; idx < CPB * 16 * GP; idx += S4_THREADS) {
            const int ki = idx / GP, v = idx - ki * GP;
            const int k = ki >> 4, i = ki & 15;
            const float* pjk = sPJ + k * GP;
            float vm = 0.f, d = 0.f;
            if (i < g.n_bins) {
                const int vmi = i > 0 ? sV[k * 16 + i - 1] : 0;
                vm = (float)vmi;
                d = 2.f * ((float)i * vm - pjk[vmi]);
            }
            const float fv = (float)v;
            const float nu = fmaf((float)i, fv, -pjk[v]);
            GT[idx] = fv < vm ? nu : d - nu;
        }
        __syncthreads();

        // ---- pass 1: transport (consumers) and own-bin box (all warps)
        float ring[T][4];  // E of the last T stream rows (registers: the row loop is unrolled)
        float vs[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            vs[j] = 0.f;
#pragma unroll
            for (int q = 0; q < T; ++q) ring[q][j] = 0.f;
        }
        // G-table address of count b = gaddr + 4 * magic(b), magic(b) = 0x4B000000 + b
        // (the float 2^23 + b), so the byte -> float PRMT result indexes the table directly
        // (g.moff = -4 * 0x4B000000 arrives as a parameter so that ptxas keeps it
        // folded into gaddr instead of re-adding it per load)
        const uint32_t gaddr =
            (uint32_t)__cvta_generic_to_shared(GT + (cs * 16 + grp4) * GP) + g.moff;
        const uint4* const sacol = SA4 + cs * hw + x;
        // box-phase task -> (row in chunk, column): interior columns first, the 2R
        // border columns (padded taps) last, so only the last warps take the xmap path
        constexpr int NI = W - 2 * R;
        constexpr int MAXA = (T * W + S4_THREADS - 1) / S4_THREADS;  // box tasks per thread
        auto a_task = [&](int task, int& rho, int& ax) {
            if (task < T * NI) {
                rho = task / NI;
                ax = R + task - rho * NI;
            } else {
                const int b = task - T * NI;
                constexpr int NB = 2 * R > 0 ? 2 * R : 1;  // (T = 1: no border)
                rho = b / NB;
                const int j = b - rho * NB;
                ax = j < R ? j : W - 2 * R + j;
            }
        };
        for (int c = 0; c < n_chunks; ++c) {
            const int s0 = c * T;
            // partial-map values of this chunk's box tasks, fetched before the
            // transport so their latency hides behind it
            float pold[MAXA];
#pragma unroll
            for (int q = 0; q < MAXA; ++q) {
                const int task = tid + q * S4_THREADS;
                pold[q] = 0.f;
                if (task < T * W) {
                    int rho, ax;
                    a_task(task, rho, ax);
                    const int y = s0 + rho - 2 * R;
                    if (y >= 0 && y < h) pold[q] = part[y * W + ax];
                }
            }
            {
                // count rows loaded two stream rows ahead of their transport
                uint4 vq0 = sacol[rmap[s0] * W];
                uint4 vq1 = T > 1 ? sacol[rmap[s0 + 1] * W] : vq0;
#pragma unroll
                for (int rho = 0; rho < T; ++rho) {
                    const uint4 v = vq0;
                    vq0 = vq1;
                    if (rho + 2 < T) vq1 = sacol[rmap[s0 + rho + 2] * W];
                    // (word, prev) = words grp, grp - 1 (0 for grp 0): branch-free selects
                    const uint32_t wlo = g1 ? v.y : v.x, whi = g1 ? v.w : v.z;
                    const uint32_t plo = g1 ? v.x : 0u, phi = g1 ? v.z : v.y;
                    const uint32_t word = g2 ? whi : wlo, prev = g2 ? phi : plo;
                    float E[4] = {0.f, 0.f, 0.f, 0.f};
                    {
                        uint32_t ma = __byte_perm(prev, 0x4B000000u, 0x7653);
                        uint32_t aa = gaddr + 4u * ma;
#define S4_E(J)                                                                 \
    {                                                                           \
        const uint32_t mb = __byte_perm(word, 0x4B000000u, 0x7650 + J);         \
        const uint32_t ab = gaddr + 4u * mb;                                    \
        const float gb = lds_f32<J * GP * 4>(ab);                               \
        const float ga = lds_f32<J * GP * 4>(aa);                               \
        const float pc = __uint_as_float(mb) - __uint_as_float(ma);             \
        E[J] = (gb - ga) * rcp_approx4(fmaxf(pc, 1.f));                         \
        ma = mb;                                                                \
        aa = ab;                                                                \
    }
                        S4_E(0) S4_E(1) S4_E(2) S4_E(3)
#undef S4_E
                    }
                    // the previous row's vertical sums are stored only now, after
                    // this row's loads (a store before them would keep the compiler
                    // from issuing them early: it cannot prove the two disjoint)
                    if (rho >= 1 && s0 + rho - 1 >= 2 * R) {
                        float* vb = Vb + (((rho - 1) * CPB + cs) * 16 + grp4) * W + x;
#pragma unroll
                        for (int j = 0; j < 4; ++j) vb[j * W] = vs[j];
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
                }
                if (s0 + T - 1 >= 2 * R) {
                    float* vb = Vb + (((T - 1) * CPB + cs) * 16 + grp4) * W + x;
#pragma unroll
                    for (int j = 0; j < 4; ++j) vb[j * W] = vs[j];
                }
            }
            __syncthreads();  // Vb complete
#pragma unroll
            for (int q = 0; q < MAXA; ++q) {
                const int task = tid + q * S4_THREADS;
                if (task >= T * W) continue;
                int rho, ax;
                a_task(task, rho, ax);
                const int y = s0 + rho - 2 * R;
                if (y < 0 || y >= h) continue;
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < CPB; ++k) {
                    const float scale = sscale[k];
                    if (scale == 0.f) continue;
                    const int bb = sb[k * hw + y * W + ax];
                    const float* vb = Vb + ((rho * CPB + k) * 16 + bb) * W;
                    float f = 0.f;
                    if (ax >= R && ax + R < W) {
#pragma unroll
                        for (int d = -R; d <= R; ++d) f += vb[ax + d];
                    } else {
#pragma unroll
                        for (int d = 0; d < T; ++d) f += vb[xmap[ax + d]];
                    }
                    acc = fmaf(f, scale, acc);
                }
                part[y * W + ax] = pold[q] + acc;
            }
            __syncthreads();  // Vb free
        }
    }
}

int sample_stride(int h, int w, int budget);

template <int T, int W, int NCOL>
static int s4_total(Score4Geom& g) {
    score4_layout<T, W, NCOL>(g);
    return g.total;
}

static int score4_plan(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                       int pad, int budget, bool has_ref, Score4Geom* out, size_t* smem_out,
                       int* ncol_out) {
    if (t < 1 || t > 11 || (t & 1) == 0 || n_bins < 1 || n_bins > 16) return QFCA_ERR_UNSUPPORTED;
    if (w != 32 && w != 64 && w != 128) return QFCA_ERR_UNSUPPORTED;
    if (h < 1 || (int64_t)h * w > (1 << 20) || ((int64_t)h * w) % 16) return QFCA_ERR_UNSUPPORTED;
    if (pad != QFCA_PAD_REFLECT && pad != QFCA_PAD_WRAP) return QFCA_ERR_UNSUPPORTED;
    Score4Geom g;
    memset(&g, 0, sizeof(g));
    g.h = h; g.n_bins = n_bins; g.pad = pad; g.C = C;
    g.S = h + 2 * (t / 2);
    g.n0 = (h + t - 1) / t;
    g.nsamp = h * w;
    g.moff = 0u - 4u * 0x4B000000u;
    // NCOL = 64 (two CTAs per SM) when the plane is narrow enough and fits, else 128
    int ncol = 0;
    size_t bytes = 0;
    for (int pass = 0; pass < 2 && !ncol; ++pass) {
        const int nc = pass == 0 ? 64 : 128;
        if (nc < w) continue;
        if (!has_ref) {
            // in-kernel reference: every pixel must be a sample (stride 1), counts
            // must fit the packed compare (T^2 <= 126) and the 8/16-bit counters
            if (t * t > 126 || budget < 1 || !(pad == QFCA_PAD_WRAP || h > 1)) return QFCA_ERR_UNSUPPORTED;
            if (sample_stride(h, w, budget) != 1) return QFCA_ERR_UNSUPPORTED;
            const int tps = 4 * nc / (nc / w);
            if (g.nsamp >= 65536 || (g.nsamp + tps - 1) / tps > 255) continue;
            g.fref = 1;
        }
        Score4Geom gg = g;
        switch (t * 100000 + w * 1000 + nc) {
#define S4C(TT, WW, NC) case TT * 100000 + WW * 1000 + NC: bytes = s4_total<TT, WW, NC>(gg); break;
            S4C(1, 32, 64) S4C(1, 64, 64) S4C(3, 32, 64) S4C(3, 64, 64) S4C(5, 32, 64)
            S4C(5, 64, 64) S4C(7, 32, 64) S4C(7, 64, 64) S4C(9, 32, 64) S4C(9, 64, 64)
            S4C(11, 32, 64) S4C(11, 64, 64)
            S4C(1, 32, 128) S4C(1, 64, 128) S4C(1, 128, 128) S4C(3, 32, 128) S4C(3, 64, 128)
            S4C(3, 128, 128) S4C(5, 32, 128) S4C(5, 64, 128) S4C(5, 128, 128) S4C(7, 32, 128)
            S4C(7, 64, 128) S4C(7, 128, 128) S4C(9, 32, 128) S4C(9, 64, 128) S4C(9, 128, 128)
            S4C(11, 32, 128) S4C(11, 64, 128) S4C(11, 128, 128)
#undef S4C
            default: return QFCA_ERR_UNSUPPORTED;
        }
        if (bytes <= (size_t)(nc == 64 ? S4_SMEM_2CTA : S4_SMEM_MAX)) {
            ncol = nc;
            g = gg;
        }
    }
    if (!ncol) return QFCA_ERR_UNSUPPORTED;
    const int cpb = ncol / w;
    int groups = groups_hint;
    if (groups <= 0) groups = balanced_groups(images, C, cpb, ncol == 64 ? 2 : 1);
    groups = groups < 1 ? 1 : (groups > C ? C : groups);
    // whole batches per group
    g.cpg = ((C + groups - 1) / groups + cpb - 1) / cpb * cpb;
    g.groups = (C + g.cpg - 1) / g.cpg;
    *out = g;
    *smem_out = bytes;
    *ncol_out = ncol;
    return QFCA_OK;
}

int score4_query(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                 int pad, int budget, int want_fref, int* fref) {
    Score4Geom g;
    size_t smem;
    int ncol;
    if (score4_plan(h, w, n_bins, t, C, images, groups_hint, pad, budget, want_fref == 0, &g,
                    &smem, &ncol) != QFCA_OK)
        return -1;
    if (fref) *fref = g.fref;
    return g.groups;
}

int launch_score4(const void* bins, int bins_bytes, const float* lo, const float* hi,
                  const int32_t* V, int64_t images, int C, int h, int w, int n_bins, int t,
                  int pad, int budget, int groups, float* partial, cudaStream_t st) {
    if (bins_bytes != 1) return QFCA_ERR_UNSUPPORTED;
    Score4Geom g;
    size_t smem;
    int ncol;
    int rc = score4_plan(h, w, n_bins, t, C, images, groups, pad, budget, V != nullptr, &g,
                         &smem, &ncol);
    if (rc != QFCA_OK) return rc;
    if (groups > 0 && g.groups != groups) return QFCA_ERR_ARG;
    void (*kern)(const uint8_t*, const float*, const float*, const int32_t*, const Score4Geom,
                 float*) = nullptr;
    switch (t * 100000 + w * 1000 + ncol) {
#define S4K(TT, WW, NC) case TT * 100000 + WW * 1000 + NC: kern = k_score4<TT, WW, NC>; break;
        S4K(1, 32, 64) S4K(1, 64, 64) S4K(3, 32, 64) S4K(3, 64, 64) S4K(5, 32, 64)
        S4K(5, 64, 64) S4K(7, 32, 64) S4K(7, 64, 64) S4K(9, 32, 64) S4K(9, 64, 64)
        S4K(11, 32, 64) S4K(11, 64, 64)
        S4K(1, 32, 128) S4K(1, 64, 128) S4K(1, 128, 128) S4K(3, 32, 128) S4K(3, 64, 128)
        S4K(3, 128, 128) S4K(5, 32, 128) S4K(5, 64, 128) S4K(5, 128, 128) S4K(7, 32, 128)
        S4K(7, 64, 128) S4K(7, 128, 128) S4K(9, 32, 128) S4K(9, 64, 128) S4K(9, 128, 128)
        S4K(11, 32, 128) S4K(11, 64, 128) S4K(11, 128, 128)
#undef S4K
        default: return QFCA_ERR_UNSUPPORTED;
    }
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100) !=
            cudaSuccess)
        return QFCA_ERR_CUDA;
    const int64_t grid = images * g.groups;
    kern<<<(unsigned)grid, 4 * ncol, smem, st>>>((const uint8_t*)bins, lo, hi, V, g, partial);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
