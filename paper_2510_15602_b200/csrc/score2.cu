// score2.cu -- K4 v2: the fused scoring kernel, specialised for the default
// family (uint8 bins, compile-time T <= 15, all bins of a row in one pass).
//
// Same mathematics as score.cu (see its header) -- exact integer window
// counts, closed-form Alg. 1, exact sliding box sums -- with a thread mapping
// chosen for instruction count and on-chip traffic:
//
//   thread (slot cs, bin group g, column x): 4 bins i = 4g..4g+3 of column x
//   of one channel; CPB channels ("slots") of one image share the CTA.
//
//   H1  vertical window counts as *thermometer* words: 8-bit lane j holds
//       #{rows of the column window with bin <= 4g+j} (table lookup per bin);
//       one column tracker per thread slides down the row stream.
//   H2  horizontal window: a (row, slot, group, segment) task slides the padded
//       row of column words -> A_{4g+j}(y,x) directly (cumulative counts; no
//       cross-word prefix; A_{4g-1} is lane 3 of group g-1).
//   E   per thread, per row, 4 bins: E_i = (G_i(A_i) - G_i(A_{i-1})) / P_i in
//       fp32 from exact small integers (byte -> float by PRMT magic, one
//       MUFU.RCP); the vertical box keeps a T-row ring of E in REGISTERS (row
//       loop unrolled by T, static slots), re-anchored every T rows.
//   A   own-bin horizontal box from the per-row V planes, slots summed in
//       fixed order, one RMW of the group partial per pixel; runs in the same
//       phase as the next chunk's H1 (no dependency between them).
//
// Shared-memory offsets are computed on the host and passed as kernel
// parameters (no runtime layout arithmetic, no local-memory arrays).
#include <string.h>

#include "common.cuh"

namespace qfca {

constexpr int S2_THREADS = 512;

struct Score2Geom {
    int h, w, n_bins, pad, C, groups, cpg;
    int G;     // bin groups of 4 (ceil(N / 4))
    int CPB;   // channels per CTA pass
    int WP;    // padded row length w + 2r
    int WPS;   // skewed storage length of a padded row
    int S;     // stream rows h + 2r
    int seg;   // H2 segment length
    int nseg;  // H2 segments per row
    int fastW; // compile-time-width variant in use (0 = runtime geometry)
    // fused reference selection (pass 0): sample grid of quantize.py:109-116
    int fref, stride, nsx, nsamp, sp;  // sp = nsamp rounded up to 4
    // shared-memory byte offsets
    int o_bins, o_pj, o_vd, o_stab, o_chp, o_wh, o_vb, o_xmap, o_scale, o_th, o_sv, o_sa, total;
};

constexpr int S2_MAXSEG = 33;  // longest H2 segment the unrolled loop covers

// H2 segment length: as few segments per (row, slot, group) as keep every
// thread busy, rounded up to odd (distinct banks across a warp's segments)
__host__ __device__ constexpr int s2_seg_rows(int rows, int w) {
    return ((w + ((S2_THREADS / rows) > 0 ? (S2_THREADS / rows) : 1) - 1) /
            ((S2_THREADS / rows) > 0 ? (S2_THREADS / rows) : 1)) | 1;
}
__host__ __device__ constexpr int s2_seg(int t, int w) {  // fixed-width: CPB*G = 512/w
    return s2_seg_rows(t * (S2_THREADS / w), w);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int T>
static void score2_layout(Score2Geom& g) {
    int off = 0;
    auto take = [&](long long bytes) {
        const int o = off;
        off = (int)((off + bytes + 15) & ~15LL);
        return o;
    };
    const int np = g.G * 4;
    g.o_bins = take((long long)g.CPB * g.h * g.w);
    g.o_pj = take((long long)g.CPB * (T * T + 1) * 4);
    g.o_vd = take((long long)g.CPB * np * 2 * 4);
    g.o_stab = take((long long)((g.S + T - 1) / T) * T * 16);
    g.o_chp = take((long long)T * g.CPB * g.G * g.WP * 4);
    g.o_wh = take((long long)T * g.CPB * g.G * g.w * 4);
    // the sample store (pass 0 only) and the V rows (pass 1 only) share space
    const long long vb_bytes = (long long)T * g.CPB * np * g.w * 4;
    const long long sa_bytes = g.fref ? (long long)g.CPB * np * g.sp : 0;
    g.o_vb = take(vb_bytes > sa_bytes ? vb_bytes : sa_bytes);
    g.o_sa = g.o_vb;
    g.o_xmap = take((long long)g.WP * 4);
    g.o_scale = take((long long)g.CPB * 4);
    g.o_th = take((long long)256 * g.G * 4);
    g.o_sv = take((long long)g.CPB * np * 4);
    g.total = off;
}

// W > 0: compile-time plane width (32 / 64 / 128) with 4 bin groups (N <= 16),
// so all index arithmetic folds to shifts; W == 0: runtime geometry.
template <int T, int W>
__global__ void __launch_bounds__(S2_THREADS, 1)
k_score2(const uint8_t* __restrict__ bins, const float* __restrict__ lo,
         const float* __restrict__ hi, const int32_t* __restrict__ Vref, const Score2Geom g,
         float* __restrict__ partial) {
    constexpr int R = T / 2;
    constexpr int T2 = T * T;
    static_assert(W == 0 || (S2_THREADS % (4 * W)) == 0, "W must divide the CTA");
    extern __shared__ __align__(16) uint8_t sm[];
    uint8_t* const sb = sm + g.o_bins;
    float* const sPJ = reinterpret_cast<float*>(sm + g.o_pj);
    float* const sVD = reinterpret_cast<float*>(sm + g.o_vd);
    int4* const stab = reinterpret_cast<int4*>(sm + g.o_stab);
    uint32_t* const CHp = reinterpret_cast<uint32_t*>(sm + g.o_chp);
    uint32_t* const WH = reinterpret_cast<uint32_t*>(sm + g.o_wh);
    float* const Vb = reinterpret_cast<float*>(sm + g.o_vb);
    int* const xmap = reinterpret_cast<int*>(sm + g.o_xmap);
    float* const sscale = reinterpret_cast<float*>(sm + g.o_scale);
    uint32_t* const TH = reinterpret_cast<uint32_t*>(sm + g.o_th);
    int* const sV = reinterpret_cast<int*>(sm + g.o_sv);
    uint8_t* const SA = sm + g.o_sa;

    const int tid = threadIdx.x;
    const int w = W ? W : g.w;
    const int G = W ? 4 : g.G;  // a multiple of 4: GQ quads of groups
    const int GQ = G / 4;
    const int CPB = W ? S2_THREADS / (4 * W) : g.CPB;
    const int h = g.h, NP = G * 4;
    const int per_slot = G * w;
    const int cs = tid / per_slot;
    const int gx = tid - cs * per_slot;
    const int grp = gx / w;
    const int grp4 = grp * 4;
    const int x = gx - grp * w;
    const bool active = cs < CPB;
    const int img = blockIdx.x / g.groups, cg = blockIdx.x % g.groups;
    const int c_begin = cg * g.cpg, c_end = min(g.C, c_begin + g.cpg);
    const int hw = h * w;
    float* const part = partial + ((int64_t)img * g.groups + cg) * hw;

    // ---- per-CTA tables: stream rows, padded-x map, thermometer words
    // stab[s] = {row offset entering the column window, row offset leaving it,
    //            -1 (slide) or the E row to recount from scratch,
    //            sample-row base index (fused reference) or -1}
    const int n_chunks = (g.S + T - 1) / T;
    for (int s = tid; s < n_chunks * T; s += S2_THREADS) {
        if (s >= g.S) {  // padding rows of the last chunk: tracker stays put
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
        stab[s] = make_int4(add * w, rem * w, recount, samp);
    }
    for (int p = tid; p < g.WP; p += S2_THREADS) xmap[p] = map_coord(p - R, w, g.pad);
    for (int idx = tid; idx < 256 * G; idx += S2_THREADS) {
        const int b = idx / G, q = idx % G, d = b - 4 * q;  // lane j = [b <= 4q + j]
        TH[idx] = d <= 0 ? 0x01010101u : (d < 4 ? (0x01010101u << (8 * d)) : 0u);
    }
    __syncthreads();

    // ---- H1 role: thread (slot hcs, quad hq, column hx) tracks 4 group words
    const int h1_threads = CPB * GQ * w;
    const bool h1_act = tid < h1_threads;
    const int hx = tid % w, hq = (tid / w) % GQ, hcs = h1_act ? tid / (w * GQ) : 0;
    // padded positions (outside [R, R + w)) that column hx feeds
    int halo0 = -1, halo1 = -1;
    if (h1_act) {
        for (int j = 0; j < 2 * R; ++j) {
            const int p = j < R ? j : w + j;
            if (xmap[p] == hx) {
                if (halo0 < 0) halo0 = p;
                else if (halo1 < 0) halo1 = p;
            }
        }
    }
    // a padded column can feed > 2 halo slots only for planes narrower than R
    const bool many_halo = w <= R;
    const uint8_t* const hbx = sb + hcs * hw + hx;
    const uint4* const th4 = reinterpret_cast<const uint4*>(TH) + hq;
    uint4* const chq = reinterpret_cast<uint4*>(CHp) + hcs * g.WP * GQ + hq;
    // ---- A role: the threads without an H1 column share the A phase
    const int a_threads = S2_THREADS - h1_threads;
    const int a_rows = a_threads / w;
    const int a_t = tid - h1_threads;
    const int a_x = a_t % w, a_r0 = a_t / w;
    const bool a_act = a_t >= 0 && a_t < a_rows * w;

    // ---- E role: thread (slot cs, group grp, column x)
    // sample column of x (fused reference), -1 if not on the grid
    const int xsamp = (g.fref && x % g.stride == 0) ? x / g.stride : -1;
    const int cs_ = active ? cs : 0;
    const float* const pj = sPJ + cs_ * (T2 + 1);
    // H2 task geometry: odd segment length keeps the lanes of a warp on
    // distinct banks
    const int seg = W ? s2_seg(T, W) : g.seg;
    const int nseg = (w + seg - 1) / seg;

    // H1 for the T stream rows of chunk starting at s0 (column trackers)
    uint4 cst = make_uint4(0, 0, 0, 0);  // 4 thermometer words
    auto h1_chunk = [&](int s0) {
#pragma unroll
        for (int rho = 0; rho < T; ++rho) {
            const int4 st = stab[s0 + rho];
            if (st.z < 0) {
                const uint4 a = th4[hbx[st.x] * GQ], r = th4[hbx[st.y] * GQ];
                cst.x += a.x - r.x;
                cst.y += a.y - r.y;
                cst.z += a.z - r.z;
                cst.w += a.w - r.w;
            } else {
                cst = make_uint4(0, 0, 0, 0);
#pragma unroll 1
                for (int dy = -R; dy <= R; ++dy) {
                    const uint4 a = th4[hbx[map_coord(st.z + dy, h, g.pad) * w] * GQ];
                    cst.x += a.x;
                    cst.y += a.y;
                    cst.z += a.z;
                    cst.w += a.w;
                }
            }
            uint4* row = chq + rho * CPB * g.WP * GQ;
            row[(hx + R) * GQ] = cst;
            if (halo0 >= 0) row[halo0 * GQ] = cst;
            if (halo1 >= 0) row[halo1 * GQ] = cst;
            if (many_halo) {
                for (int j = 0; j < 2 * R; ++j) {
                    const int p = j < R ? j : w + j;
                    if (xmap[p] == hx) row[p * GQ] = cst;
                }
            }
        }
    };
    // H2 for the chunk starting at s0; only_samples: just the sample rows.
    // Task = (row, slot, quad, segment): uint4 sliding window along the row.
    auto h2_chunk = [&](int s0, bool only_samples) {
        const int ntask = T * CPB * GQ * nseg;
        for (int task = tid; task < ntask; task += S2_THREADS) {
            const int rq = task / nseg;  // (rho * CPB + cs) * GQ + q
            const int x0 = (task - rq * nseg) * seg;
            const int rc = rq / GQ, q = rq - rc * GQ;
            if (only_samples && stab[s0 + rc / CPB].w < 0) continue;
            const uint4* src = reinterpret_cast<const uint4*>(CHp) + (rc * g.WP + x0) * GQ + q;
            uint4* dst = reinterpret_cast<uint4*>(WH) + (rc * w + x0) * GQ + q;
            uint4 sum = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int p = 0; p < T; ++p) {
                const uint4 v = src[p * GQ];
                sum.x += v.x;
                sum.y += v.y;
                sum.z += v.z;
                sum.w += v.w;
            }
            dst[0] = sum;
            const int kend = min(seg, w - x0);
            if (kend == seg && seg <= S2_MAXSEG) {
#pragma unroll
                for (int k = 1; k < S2_MAXSEG; ++k) {
                    if (k < seg) {
                        const uint4 a = src[(k + 2 * R) * GQ], r = src[(k - 1) * GQ];
                        sum.x += a.x - r.x;
                        sum.y += a.y - r.y;
                        sum.z += a.z - r.z;
                        sum.w += a.w - r.w;
                        dst[k * GQ] = sum;
                    }
                }
            } else {
                for (int k = 1; k < kend; ++k) {
                    const uint4 a = src[(k + 2 * R) * GQ], r = src[(k - 1) * GQ];
                    sum.x += a.x - r.x;
                    sum.y += a.y - r.y;
                    sum.z += a.z - r.z;
                    sum.w += a.w - r.w;
                    dst[k * GQ] = sum;
                }
            }
        }
    };
    // group words of (stream row rho, slot cs, column x): this group and the previous one
    auto wh_words = [&](int rho, uint32_t& word, uint32_t& prev) {
        const uint4 v = reinterpret_cast<const uint4*>(WH)[((rho * CPB + cs) * w + x) * GQ +
                                                           (grp >> 2)];
        const int gl = grp & 3;
        word = gl == 0 ? v.x : gl == 1 ? v.y : gl == 2 ? v.z : v.w;
        prev = gl == 1 ? v.x : gl == 2 ? v.y : gl == 3 ? v.z : 0u;
        if (gl == 0 && grp > 0)
            prev = reinterpret_cast<const uint4*>(WH)[((rho * CPB + cs) * w + x) * GQ +
                                                     (grp >> 2) - 1].w;
    };

    for (int cb = c_begin; cb < c_end; cb += CPB) {
        // ---- load the slot channels: bins planes, reference tables
        __syncthreads();
        for (int k = 0; k < CPB; ++k) {
            const int c = cb + k;
            const int64_t plane = (int64_t)img * g.C + c;
            if (tid == 0) {
                float sc = 0.f;  // w_c / T^2; 0 marks an empty or degenerate slot
                if (c < c_end && hi[plane] > lo[plane])
                    sc = (float)(((double)hi[plane] - (double)lo[plane]) / (double)g.n_bins /
                                 (double)T2);
                sscale[k] = sc;
            }
            uint8_t* dst = sb + k * hw;
            if (c < c_end) {
                const uint8_t* src = bins + plane * hw;
                if ((hw & 15) == 0) {
                    const uint4* s4 = reinterpret_cast<const uint4*>(src);
                    uint4* d4 = reinterpret_cast<uint4*>(dst);
                    for (int i = tid; i < hw / 16; i += S2_THREADS) d4[i] = __ldg(s4 + i);
                } else {
                    for (int i = tid; i < hw; i += S2_THREADS) dst[i] = src[i];
                }
                if (!g.fref)
                    for (int i = tid; i < NP; i += S2_THREADS)
                        sV[k * NP + i] = i < g.n_bins ? __ldg(Vref + plane * g.n_bins + i) : T2;
            } else {
                for (int i = tid; i < hw; i += S2_THREADS) dst[i] = 0;
                for (int i = tid; i < NP; i += S2_THREADS) sV[k * NP + i] = T2;
            }
        }
        __syncthreads();
        if (g.fref) {
            // ---- pass 0: the global reference, fused (quantize.py:150-200).  The
            // window counts at the stride-grid samples come from the same trackers;
            // V_i = the (S-1-m)-th smallest A_i over the samples (reference.cu).
            // phases: [H1(ch) + gather(ch-1)] | H2(ch, sample rows only)
            for (int ch = 0; ch <= n_chunks; ++ch) {
                const int s0 = ch * T;
                if (ch < n_chunks && h1_act) h1_chunk(s0);
                if (ch > 0 && active && xsamp >= 0) {
                    const int ps0 = s0 - T;
                    uint8_t* sa = SA + (cs * NP + grp4) * g.sp + xsamp;
#pragma unroll
                    for (int rho = 0; rho < T; ++rho) {
                        const int si = stab[ps0 + rho].w;
                        if (si < 0) continue;
                        uint32_t word, prev;
                        wh_words(rho, word, prev);
#pragma unroll
                        for (int j = 0; j < 4; ++j) sa[j * g.sp + si] = (word >> (8 * j)) & 0xff;
                    }
                }
                __syncthreads();
                if (ch == n_chunks) break;
                h2_chunk(s0, true);
                __syncthreads();
            }
            // pad each sample row with values above any query (packed compares)
            for (int idx = tid; idx < CPB * NP * (g.sp - g.nsamp); idx += S2_THREADS) {
                const int row = idx / (g.sp - g.nsamp), k = idx % (g.sp - g.nsamp);
                SA[row * g.sp + g.nsamp + k] = 127;
            }
            __syncthreads();
            {  // one warp per (slot, bin): smallest v with #{A <= v} >= S - m
                const int warp = tid >> 5, lane = tid & 31;
                const int c0 = g.nsamp - (g.nsamp - 1) / 2;
                for (int task = warp; task < CPB * NP; task += S2_THREADS / 32) {
                    const int k = task / NP, i = task % NP;
                    int res = T2;
                    if (i < g.n_bins - 1 && sscale[k] != 0.f) {
                        const uint32_t* row = reinterpret_cast<const uint32_t*>(SA + task * g.sp);
                        int a = 0, b = T2;
                        while (a < b) {
                            const int mid = (a + b) >> 1;
                            const uint32_t q = 0x80808080u | ((uint32_t)mid * 0x01010101u);
                            int cnt = 0;
                            for (int wi = lane; wi < g.sp / 4; wi += 32)
                                cnt += __popc((q - row[wi]) & 0x80808080u);
                            cnt = warp_sum_i(cnt);
                            if (cnt >= c0) b = mid; else a = mid + 1;
                        }
                        res = a;
                    }
                    if (lane == 0) sV[task] = res;
                }
            }
            __syncthreads();
        }
        for (int k = 0; k < CPB; ++k) {
            float* pjk = sPJ + k * (T2 + 1);
            const int* V = sV + k * NP;
            for (int q = tid; q < T2; q += S2_THREADS) {  // J_q = min{i : V_i > q}
                int a = 0, b = g.n_bins - 1;
                while (a < b) {
                    const int mid = (a + b) >> 1;
                    if (V[mid] > q) b = mid; else a = mid + 1;
                }
                pjk[q + 1] = (float)a;
            }
        }
        __syncthreads();
        if (tid < 32 * CPB) {  // one warp per slot: PJ = inclusive prefix of J
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
        for (int idx = tid; idx < CPB * NP; idx += S2_THREADS) {
            const int k = idx / NP, i = idx % NP;
            float vm = 0.f, d = 0.f;
            if (i < g.n_bins) {
                const int vmi = i > 0 ? sV[k * NP + i - 1] : 0;
                vm = (float)vmi;
                d = 2.f * ((float)i * vm - sPJ[k * (T2 + 1) + vmi]);
            }
            sVD[(k * NP + i) * 2] = vm;
            sVD[(k * NP + i) * 2 + 1] = d;
        }
        __syncthreads();

        float Vm[4], Dv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            Vm[j] = sVD[(cs_ * NP + grp4 + j) * 2];
            Dv[j] = sVD[(cs_ * NP + grp4 + j) * 2 + 1];
        }
        float ring[T][4];
        float vs[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            vs[j] = 0.f;
#pragma unroll
            for (int q = 0; q < T; ++q) ring[q][j] = 0.f;
        }

        // the stream is padded to whole chunks of T rows (stab mode 2 = no move)
        for (int ch = 0; ch <= n_chunks; ++ch) {
            const int s0 = ch * T;
            // ---- phase 1: H1 of chunk ch  +  A of chunk ch-1
            if (ch < n_chunks && h1_act) h1_chunk(s0);
            if (ch > 0 && a_act) {
                const int ps0 = s0 - T;
                for (int rho = a_r0; rho < T; rho += a_rows) {
                    const int y = ps0 + rho - 2 * R;
                    if (y < 0 || y >= h) continue;
                    float acc = 0.f;
                    for (int k = 0; k < CPB; ++k) {
                        const float scale = sscale[k];
                        if (scale == 0.f) continue;
                        const int b = sb[k * hw + y * w + a_x];
                        const float* vb = Vb + ((rho * CPB + k) * NP + b) * w;
                        float f = 0.f;
                        if (a_x >= R && a_x + R < w) {
#pragma unroll
                            for (int d = -R; d <= R; ++d) f += vb[a_x + d];
                        } else {
#pragma unroll
                            for (int d = 0; d < T; ++d) f += vb[xmap[a_x + d]];
                        }
                        acc = fmaf(f, scale, acc);
                    }
                    part[y * w + a_x] += acc;
                }
            }
            __syncthreads();
            if (ch == n_chunks) break;
            // ---- phase 2: H2, horizontal windows of the column words
            h2_chunk(s0, false);
            __syncthreads();
            // ---- phase 3: E, closed-form transport + register ring + vertical box
            if (active) {
#pragma unroll
                for (int rho = 0; rho < T; ++rho) {
                    uint32_t word, prev;
                    wh_words(rho, word, prev);
                    // the group has mass in this window iff A_{4g+3} > A_{4g-1};
                    // groups empty across the whole warp contribute E = 0
                    const bool mass = (word >> 24) != (prev >> 24);
                    if (__any_sync(__activemask(), mass)) {
                        // byte -> float by exponent magic: 0x4B0000bb = 2^23 + b
                        const uint32_t ma = __byte_perm(prev, 0x4B000000u, 0x7653);
                        float af = __uint_as_float(ma) - 8388608.0f;
                        float pja = pj[ma - 0x4B000000u];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t mbits = __byte_perm(word, 0x4B000000u, 0x7650 + j);
                            const float bf = __uint_as_float(mbits) - 8388608.0f;
                            const float pjb = pj[mbits - 0x4B000000u];
                            const float fi = (float)(grp4 + j);
                            const float nua = fmaf(fi, af, -pja);  // -u(a)
                            const float nub = fmaf(fi, bf, -pjb);  // -u(b)
                            const float ga = af < Vm[j] ? nua : Dv[j] - nua;
                            const float gb = bf < Vm[j] ? nub : Dv[j] - nub;
                            const float pc = bf - af;
                            // pc == 0 -> gb == ga exactly -> E == 0
                            const float E = (gb - ga) * rcp_approx(fmaxf(pc, 1.f));
                            vs[j] += E - ring[rho][j];
                            ring[rho][j] = E;
                            af = bf;
                            pja = pjb;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            vs[j] -= ring[rho][j];
                            ring[rho][j] = 0.f;
                        }
                    }
                    if (rho == T - 1) {  // re-anchor: exact sum of the ring
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            float s = ring[0][j];
#pragma unroll
                            for (int q = 1; q < T; ++q) s += ring[q][j];
                            vs[j] = s;
                        }
                    }
                    if (s0 + rho >= 2 * R) {
                        float* vb = Vb + ((rho * CPB + cs) * NP + grp4) * w + x;
#pragma unroll
                        for (int j = 0; j < 4; ++j) vb[j * w] = vs[j];
                    }
                }
            }
            __syncthreads();
        }
    }
}

template <int T>
static int score2_plan_t(Score2Geom& g) {
    score2_layout<T>(g);
    return g.total;
}

int sample_stride(int h, int w, int budget);

// fused_ref: compute the median-quan reference inside the kernel (pass 0) when
// possible -- T^2 <= 126 (packed u8 compares), reflect with h, w > 1 or wrap
// (pad_plane's edge fallback for size-1 axes differs from _map_coord), and the
// sample store fits shared memory.
static int score2_plan(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                       int pad, int budget, bool fused_ref, Score2Geom* out, size_t* smem_out) {
    if (t < 1 || t > 15 || (t & 1) == 0) return QFCA_ERR_UNSUPPORTED;
    if (n_bins > 256) return QFCA_ERR_UNSUPPORTED;
    if ((int64_t)h * w > (1 << 24)) return QFCA_ERR_UNSUPPORTED;
    Score2Geom g;
    memset(&g, 0, sizeof(g));
    g.h = h; g.w = w; g.n_bins = n_bins; g.pad = pad; g.C = C;
    g.fref = fused_ref && t * t <= 126 && budget >= 1 &&
             (pad == QFCA_PAD_WRAP || (h > 1 && w > 1)) ? 1 : 0;
    if (g.fref) {
        g.stride = sample_stride(h, w, budget);
        g.nsx = (w + g.stride - 1) / g.stride;
        g.nsamp = ((h + g.stride - 1) / g.stride) * g.nsx;
        g.sp = (g.nsamp + 3) & ~3;
    }
    // compile-time-width variant: w in {32, 64, 128}, 4 groups (N <= 16)
    const bool fast = n_bins <= 16 && (w == 32 || w == 64 || w == 128);
    g.fastW = fast ? w : 0;
    g.G = fast ? 4 : ((n_bins + 15) / 16) * 4;  // whole quads of 4-bin groups
    const int per = g.G * w;
    if (per > S2_THREADS || w < 4) return QFCA_ERR_UNSUPPORTED;
    g.CPB = S2_THREADS / per;
    if (g.CPB > 8) g.CPB = 8;
    const int r = t / 2;
    g.WP = w + 2 * r;
    g.WPS = g.WP | 1;  // odd row stride
    g.S = h + 2 * r;
    size_t bytes = 0;
    for (;;) {
        // H2 segments: one task per thread where possible (kernel recomputes
        // the same value at compile time for the fixed-width variants)
        g.seg = g.fastW ? s2_seg(t, w) : s2_seg_rows(t * g.CPB * g.G, w);
        if (g.seg > w) g.seg = w;
        g.nseg = (w + g.seg - 1) / g.seg;
        switch (t) {
#define QFCA_S2_CASE(TT) case TT: bytes = score2_plan_t<TT>(g); break;
            QFCA_S2_CASE(1) QFCA_S2_CASE(3) QFCA_S2_CASE(5) QFCA_S2_CASE(7)
            QFCA_S2_CASE(9) QFCA_S2_CASE(11) QFCA_S2_CASE(13) QFCA_S2_CASE(15)
#undef QFCA_S2_CASE
        }
        if (bytes <= 225 * 1024) break;
        if (g.fref) {  // keep the fast variant, compute the reference outside
            g.fref = 0;
            continue;
        }
        if (g.fastW) {  // the fixed-width variant needs its full slot count
            g.fastW = 0;
            g.G = ((n_bins + 15) / 16) * 4;
            g.CPB = S2_THREADS / (g.G * w);
            if (g.CPB > 8) g.CPB = 8;
            continue;
        }
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

// groups the v2 kernel would use (-1: not applicable); *fref = fused reference
int score2_query(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                 int pad, int budget, int want_fref, int* fref) {
    Score2Geom g;
    size_t smem;
    if (score2_plan(h, w, n_bins, t, C, images, groups_hint, pad, budget, want_fref != 0, &g,
                    &smem) != QFCA_OK)
        return -1;
    if (fref) *fref = g.fref;
    return g.groups;
}

// V == nullptr: the reference is selected inside the kernel (needs fref).
int launch_score2(const void* bins, int bins_bytes, const float* lo, const float* hi,
                  const int32_t* V, int64_t images, int C, int h, int w, int n_bins, int t,
                  int pad, int budget, int groups, float* partial, cudaStream_t st) {
    if (bins_bytes != 1) return QFCA_ERR_UNSUPPORTED;
    if (pad != QFCA_PAD_REFLECT && pad != QFCA_PAD_WRAP) return QFCA_ERR_UNSUPPORTED;
    Score2Geom g;
    size_t smem;
    int rc = score2_plan(h, w, n_bins, t, C, images, groups, pad, budget, V == nullptr, &g,
                         &smem);
    if (rc != QFCA_OK) return rc;
    if (groups > 0 && g.groups != groups) return QFCA_ERR_ARG;
    if (V == nullptr && !g.fref) return QFCA_ERR_UNSUPPORTED;
    const int64_t grid = images * g.groups;
    void (*kern)(const uint8_t*, const float*, const float*, const int32_t*, const Score2Geom,
                 float*) = nullptr;
#define QFCA_S2_PICK(TT)                                                       \
    case TT:                                                                   \
        kern = g.fastW == 128 ? k_score2<TT, 128>                              \
             : g.fastW == 64  ? k_score2<TT, 64>                               \
             : g.fastW == 32  ? k_score2<TT, 32> : k_score2<TT, 0>;            \
        break;
    switch (t) {
        QFCA_S2_PICK(1) QFCA_S2_PICK(3) QFCA_S2_PICK(5) QFCA_S2_PICK(7)
        QFCA_S2_PICK(9) QFCA_S2_PICK(11) QFCA_S2_PICK(13) QFCA_S2_PICK(15)
        default: return QFCA_ERR_UNSUPPORTED;
    }
#undef QFCA_S2_PICK
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return QFCA_ERR_CUDA;
    kern<<<(unsigned)grid, S2_THREADS, smem, st>>>((const uint8_t*)bins, lo, hi, V, g, partial);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
