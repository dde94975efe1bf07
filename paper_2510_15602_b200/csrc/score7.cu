// score7.cu -- K4 v7: the fused scoring kernel for LARGE patch sizes (T = 17..65)
// on 128-wide planes / tiles (configs[3]'s patch sweep at 1024^2).
//
// v6 keeps the vertical box of the transport errors E in a T-row register ring
// and gathers the own-bin horizontal box with T taps: both scale with T.  v7
// keeps no T-row state at all.  Same closed-form transport (score2.cu's fp32
// G_i, rcp.approx; bit-identical E for the same counts) and the same window
// counts, but the association is an exact 2D prefix (summed-area table) of E
// over the reflect-padded window-centre grid, evaluated incrementally:
//
//   Q_i(s, p) = sum_{s' <= s, p' <= p} E_i(centre(s'), column(p'))     (fp64)
//   score(y, x) = Q_b(y+2R, x+2R) - Q_b(y+2R, x-1) - Q_b(y-1, x+2R) + Q_b(y-1, x-1)
//
// with b = bin(y, x).  The stream walks the padded centre rows s = 0 .. h+2R-1
// once; after row s the CTA holds the row Q(s, .) of all 16 bins; a pixel
// whose window starts at s + 1 snapshots the first difference of its own bin,
// a pixel whose window ends at s subtracts it (per-pixel snapshots in a ring of
// 2R + 2 rows).  Every cost per (channel, pixel) is independent of T:
//
//   phase RW  row windows of the thermometer counts (8-bit lanes, one warp per
//             row: warp prefix scan over the padded row, window = difference of
//             two prefix words) -> per-SM scratch in L2 (word-major rows);
//   phase 4   per stream row: the vertical window counts slide by one row in
//             registers (16-bit lanes: add the entering row's windows, remove
//             the leaving row's), E of the thread's 4 bins from the shared
//             prefix table PJ (the G values computed, not tabulated: 16 x (T^2
//             + 1) floats do not fit), E row -> shared memory; one warp per bin
//             scans the row (fp64, registers keep Q for its columns) and
//             publishes Q(s, .); bin groups 2 / 3 (rare mass, light E) take the
//             snapshots and the finished pixels.
// The reference comes from K3 (reference.cu).  fp64 prefixes: the result is the
// reference's own fp64 SAT association (scoring.py:218-232) up to summation
// order, far inside the 1e-4 bar.
#include <string.h>

#include "common.cuh"

namespace qfca {

constexpr int S7_THREADS = 512;
constexpr int S7_W = 128;
constexpr int S7_EST = S7_W + 2;  // E row stride (conflict-free stores)
constexpr int S7_SMEM_MAX = 227 * 1024;
constexpr int S7_GT_MAXT = 43;  // largest T whose 16 x (T^2 + 1) G table is built
constexpr int S7_NFL = 4;       // stream rows between fp32 -> fp64 prefix flushes

struct Score7Geom {
    int h, n_bins, pad, C, groups, cpg;
    int S;      // stream rows h + 2R
    int nsnap;  // snapshot rows 2R + 2
    // in-kernel reference (median-quan, quantize.py:150-200): sample grid
    int fref, stride, nsy, nsx, nsamp, srow;
    int o_sb, o_pj, o_gt, o_erow, o_qrow, o_qf, o_prow, o_snap, o_sa, o_xmap, o_stab, o_misc, total;
    int gt;         // 1: the G_i(v) table (T <= 43 and it fits), else G from PJ
    int passes;     // bin passes: 16 lanes each, 15 new bins after the first (N <= 256)
    uint32_t moff;  // G-table address of the magic float 2^23 + v is base + 4 v
};

__device__ __forceinline__ float rcp_approx7(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// thermometer words of bin b (lane j of word q = [b <= 4q + j]) by ALU: see
// score6.cu's thermo6
__device__ __forceinline__ uint4 thermo7(int b, int tb) {  // lanes: bins tb .. tb + 15
    const int s = 8 * (b - tb);
    return make_uint4(__funnelshift_lc(0u, 0x01010101u, max(s, 0)),
                      __funnelshift_lc(0u, 0x01010101u, max(s - 32, 0)),
                      __funnelshift_lc(0u, 0x01010101u, max(s - 64, 0)),
                      __funnelshift_lc(0u, 0x01010101u, max(s - 96, 0)));
}
__device__ __forceinline__ uint32_t smid7() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

template <int T, bool GT>
static void score7_layout(Score7Geom& g) {
    constexpr int R = T / 2;
    constexpr int WP = S7_W + 2 * R;
    int off = 0;
    auto take = [&](long long bytes) {
        const int o = off;
        off = (int)((off + bytes + 15) & ~15LL);
        return o;
    };
    g.o_sb = take((long long)g.h * S7_W);
    // one region, three lives: the RW phase's prefix rows, then the sample
    // store (fref), then the phase-4 tables and rows
    const int ubase = off;
    g.o_pj = take((long long)(T * T + 1) * 4);
    g.o_gt = GT ? take(16LL * (T * T + 1) * 4) : 0;
    g.o_qrow = take(16LL * WP * 8);
    g.o_qf = take(16LL * WP * 4);
    g.o_snap = take((long long)g.nsnap * S7_W * 8);
    const int p4end = off;
    g.o_prow = ubase;  // one padded prefix row per warp (RW phase)
    g.o_sa = ubase;
    long long uend = p4end;
    const long long prb = 16LL * WP * 16;
    if (ubase + prb > uend) uend = ubase + prb;
    if (g.fref) {
        const long long sab = (long long)g.srow * 16 * 2;
        if (ubase + sab > uend) uend = ubase + sab;
    }
    off = (int)((uend + 15) & ~15LL);
    g.o_erow = take(16LL * S7_EST * 4);
    g.o_xmap = take((long long)WP * 4);
    g.o_stab = take((long long)(g.S + 1) * 16);
    g.o_misc = take(2048);  // scale, V[256], (vm, d) of the pass's 16 bins
    g.total = off;
}

template <int T, bool GT>
__global__ void __launch_bounds__(S7_THREADS, 1)
k_score7(const uint8_t* __restrict__ bins, const float* __restrict__ lo,
         const float* __restrict__ hi, const int32_t* __restrict__ Vref, const Score7Geom g,
         uint32_t* __restrict__ scratch, float* __restrict__ partial) {
    constexpr int W = S7_W;
    constexpr int R = T / 2;
    constexpr int T2 = T * T;
    constexpr int WP = W + 2 * R;             // padded columns
    constexpr int CPL = (WP + 31) / 32;       // padded columns per lane (scans)
    constexpr int EST = S7_EST;
    constexpr int GP = T2 + 1;
    constexpr uint32_t FULL = 0xffffffffu;
    extern __shared__ __align__(16) uint8_t sm[];
    uint8_t* const sb = sm + g.o_sb;
    float* const sPJ = reinterpret_cast<float*>(sm + g.o_pj);
    float* const Erow = reinterpret_cast<float*>(sm + g.o_erow);     // [16][EST]
    double* const Qrow = reinterpret_cast<double*>(sm + g.o_qrow);   // [16][WP] (flushed)
    float* const Qf = reinterpret_cast<float*>(sm + g.o_qf);         // [16][WP] (recent)
    uint4* const Prow = reinterpret_cast<uint4*>(sm + g.o_prow);     // [16 warps][WP]
    double* const snap = reinterpret_cast<double*>(sm + g.o_snap);   // [nsnap][W]
    int* const xmap = reinterpret_cast<int*>(sm + g.o_xmap);
    int4* const stab = reinterpret_cast<int4*>(sm + g.o_stab);        // per stream row
    uint16_t* const SA = reinterpret_cast<uint16_t*>(sm + g.o_sa);     // [16][srow] (fref)
    float* const sscale = reinterpret_cast<float*>(sm + g.o_misc);    // [1]
    int* const sV = reinterpret_cast<int*>(sm + g.o_misc + 16);         // [256]
    float* const svm = reinterpret_cast<float*>(sm + g.o_misc + 1040);  // [16] (pass)
    float* const sd = reinterpret_cast<float*>(sm + g.o_misc + 1104);   // [16] (pass)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int h = g.h;
    const int hw = h * W;
    const int img = blockIdx.x / g.groups, cgi = blockIdx.x % g.groups;
    const int c_begin = cgi * g.cpg, c_end = min(g.C, c_begin + g.cpg);
    float* const part = partial + ((int64_t)img * g.groups + cgi) * hw;
    uint32_t* const scr = scratch + (size_t)smid7() * (size_t)h * 4 * W;

    // ---- per-CTA tables
    for (int p = tid; p < WP; p += S7_THREADS) xmap[p] = map_coord(p - R, W, g.pad);
    // stream row s = padded centre row, centre c = map(s - R).  For h >= 2 the
    // centre moves by one row (mod h for wrap) at every s >= 1, so the window
    // slides: (.z, .w) = scratch offsets of the entering / leaving row; entry
    // S is a harmless pad for the one-ahead prefetch
    for (int s = tid; s <= g.S; s += S7_THREADS) {
        int add = 0, rem = 0;
        const int c = map_coord(s - R, h, g.pad);
        if (s > 0 && s < g.S) {
            const int cp = map_coord(s - 1 - R, h, g.pad);
            if (c == cp - 1) { add = map_coord(c - R, h, g.pad); rem = map_coord(cp + R, h, g.pad); }
            else { add = map_coord(c + R, h, g.pad); rem = map_coord(cp - R, h, g.pad); }
        }
        stab[s] = make_int4(c, 1, add * 4 * W, rem * 4 * W);
    }
    __syncthreads();

    // phase-4 roles: thread (column x, bin group grp), the 4 groups of a column
    // in adjacent lanes (warp = 8 columns: balanced E work per warp, the
    // group-below count is one shuffle away); scan roles: warp = bin
    const int grp = tid & 3, x = tid >> 2;
    int scol[CPL];  // the columns this scan lane reads: padded p = lane * CPL + k
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
        const int p = lane * CPL + k;
        scol[k] = p < WP ? xmap[p] : 0;
    }
    // row windows in the scratch: [row][x][4 words], word q = bins 4q .. 4q+3
    const uint32_t* const rwt = scr + x * 4 + grp;

    for (int c = c_begin; c < c_end; ++c) {
        const int64_t plane = (int64_t)img * g.C + c;
        if (tid == 0) {
            float sc = 0.f;
            if (hi[plane] > lo[plane])
                sc = (float)(((double)hi[plane] - (double)lo[plane]) / (double)g.n_bins /
                             (double)T2);
            sscale[0] = sc;
        }
        for (int i = tid; i < 256; i += S7_THREADS)
            sV[i] = (i < g.n_bins && !g.fref) ? __ldg(Vref + plane * g.n_bins + i) : T2;
        for (int i = tid; i < hw / 16; i += S7_THREADS)
            reinterpret_cast<uint4*>(sb)[i] = __ldg(reinterpret_cast<const uint4*>(bins + plane * hw) + i);
        __syncthreads();
        const float scale = sscale[0];
        if (scale == 0.f) {  // degenerate channel (scoring.py:265-266)
            __syncthreads();
            continue;
        }

        // ======== phase RW: row windows of every plane row -> scratch, one warp per
        // row, thermometer lanes of the pass's bins tb .. tb + 15
        auto rw_phase = [&](int tb) {
        for (int y = warp; y < h; y += S7_THREADS / 32) {
            const uint8_t* const brow = sb + y * W;
            uint4 pre[CPL];
            uint4 run = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                const int p = lane * CPL + k;
                const uint4 v = p < WP ? thermo7(brow[scol[k]], tb) : make_uint4(0, 0, 0, 0);
                run.x += v.x; run.y += v.y; run.z += v.z; run.w += v.w;
                pre[k] = run;
            }
            // exclusive scan of the lane totals (8-bit lanes stay <= WP <= 255: exact)
            uint4 off = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t ax = __shfl_up_sync(FULL, off.x, o), ay = __shfl_up_sync(FULL, off.y, o);
                const uint32_t az = __shfl_up_sync(FULL, off.z, o), aw = __shfl_up_sync(FULL, off.w, o);
                if (lane >= o) { off.x += ax; off.y += ay; off.z += az; off.w += aw; }
            }
            off.x -= run.x; off.y -= run.y; off.z -= run.z; off.w -= run.w;
            uint4* const pr = Prow + warp * WP;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                const int p = lane * CPL + k;
                if (p < WP)
                    pr[p] = make_uint4(pre[k].x + off.x, pre[k].y + off.y, pre[k].z + off.z,
                                       pre[k].w + off.w);
            }
            __syncwarp();
            uint4* const dst = reinterpret_cast<uint4*>(scr + (size_t)y * 4 * W);
#pragma unroll
            for (int k = 0; k < W / 32; ++k) {
                const int xx = lane + 32 * k;
                const uint4 a = pr[xx + 2 * R];
                const uint4 b = xx > 0 ? pr[xx - 1] : make_uint4(0, 0, 0, 0);
                dst[xx] = make_uint4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
            }
            __syncwarp();
        }
        __syncthreads();  // scratch rows complete; the prefix rows' region is free
        };
        // ======== the reference (median-quan) from this plane's own window counts:
        // the cumulative counts A_i(s) at the stride-grid samples (reference.cu's
        // statistic: V_i = the (S-1-m)-th smallest A_i(s)) of the pass's lanes
        // klo .. 15 (lane 0 of a later pass is the previous pass's last bin)
        auto fref_pass = [&](int tb, int klo) {
            const int nsx = g.nsx, nsy = g.nsy, sd_ = g.stride;
            const int cols = 4 * nsx;
            const int nsub = max(1, S7_THREADS / cols);
            const int per = (nsy + nsub - 1) / nsub;
            if (tid < cols * nsub) {
                const int sub = tid / cols, r = tid % cols, jx = r >> 2, gq = r & 3;
                const uint32_t* const col = scr + (jx * sd_) * 4 + gq;
                uint16_t* const sa = SA + (size_t)(4 * gq) * g.srow;
                const int j0 = sub * per, j1 = min(nsy, j0 + per);
                uint32_t l16 = 0, h16 = 0;
                auto store = [&](int j) {
                    const int si = j * nsx + jx;
                    sa[si] = (uint16_t)(l16 & 0xFFFFu);
                    sa[g.srow + si] = (uint16_t)(h16 & 0xFFFFu);
                    sa[2 * g.srow + si] = (uint16_t)(l16 >> 16);
                    sa[3 * g.srow + si] = (uint16_t)(h16 >> 16);
                };
                if (sd_ == 2 && j0 < j1) {
                    // stride 2 (the 128^2 planes): a recount at the segment start,
                    // then two slides per sample row with the next row's four row
                    // windows loaded one sample row ahead
                    const int cy0 = j0 * 2;
#pragma unroll 8
                    for (int dy = -R; dy <= R; ++dy) {
                        const uint32_t w = col[(size_t)map_coord(cy0 + dy, h, g.pad) * 4 * W];
                        l16 += w & 0x00FF00FFu;
                        h16 += (w >> 8) & 0x00FF00FFu;
                    }
                    store(j0);
                    uint32_t a1 = 0, r1 = 0, a2 = 0, r2 = 0;
                    auto fetch = [&](int j) {  // centres 2j - 1, 2j: stream rows + R
                        const int4 s1 = stab[2 * j - 1 + R], s2 = stab[2 * j + R];
                        a1 = col[s1.z];
                        r1 = col[s1.w];
                        a2 = col[s2.z];
                        r2 = col[s2.w];
                    };
                    if (j0 + 1 < j1) fetch(j0 + 1);
                    for (int j = j0 + 1; j < j1; ++j) {
                        l16 += (a1 & 0x00FF00FFu) - (r1 & 0x00FF00FFu) + (a2 & 0x00FF00FFu) -
                               (r2 & 0x00FF00FFu);
                        h16 += ((a1 >> 8) & 0x00FF00FFu) - ((r1 >> 8) & 0x00FF00FFu) +
                               ((a2 >> 8) & 0x00FF00FFu) - ((r2 >> 8) & 0x00FF00FFu);
                        if (j + 1 < j1) fetch(j + 1);
                        store(j);
                    }
                } else
                for (int j = j0; j < j1; ++j) {
                    const int cy = j * sd_;
                    if (j == j0 || sd_ >= T) {
                        l16 = h16 = 0;
                        for (int dy = -R; dy <= R; ++dy) {
                            const uint32_t w = col[(size_t)map_coord(cy + dy, h, g.pad) * 4 * W];
                            l16 += w & 0x00FF00FFu;
                            h16 += (w >> 8) & 0x00FF00FFu;
                        }
                    } else {  // centres cy - stride + 1 .. cy: stream rows + R (slides)
                        for (int d = cy - sd_ + 1 + R; d <= cy + R; ++d) {
                            const int4 st = stab[d];
                            const uint32_t wa = col[st.z], wr = col[st.w];
                            l16 += (wa & 0x00FF00FFu) - (wr & 0x00FF00FFu);
                            h16 += ((wa >> 8) & 0x00FF00FFu) - ((wr >> 8) & 0x00FF00FFu);
                        }
                    }
                    store(j);
                }
            }
            // pad the sample rows so packed compares see values > any query
            const int padn = g.srow - g.nsamp;
            for (int idx = tid; idx < 16 * padn; idx += S7_THREADS)
                SA[(size_t)(idx / padn) * g.srow + g.nsamp + idx % padn] = 32767;
            __syncthreads();
            const int m = (g.nsamp - 1) / 2, c0 = g.nsamp - m;
            const int words = g.srow / 2;
            for (int bi = warp; bi < 16; bi += S7_THREADS / 32) {
                if (bi < klo || tb + bi >= g.n_bins) continue;
                const uint32_t* const row = reinterpret_cast<const uint32_t*>(SA + (size_t)bi * g.srow);
                int a = 0, b = T2;
                while (a < b) {  // smallest v with #{A <= v} >= c0
                    const int mid = (a + b) >> 1;
                    const uint32_t q = 0x80008000u | ((uint32_t)mid * 0x00010001u);
                    int cnt = 0;
                    for (int wi = lane; wi < words; wi += 32)
                        cnt += __popc((q - row[wi]) & 0x80008000u);
                    cnt = __reduce_add_sync(FULL, cnt);
                    if (cnt >= c0) b = mid; else a = mid + 1;
                }
                if (lane == 0) sV[tb + bi] = a;
            }
            __syncthreads();  // sV ready; the sample store is free again
        };
        // ======== tables: PJ = prefix of J (all bins); (V_{i-1}, D_i) and G_i of
        // the pass's bins tb .. tb + 15
        auto pass_tables = [&](int tb) {
        for (int qq = tid; qq < T2; qq += S7_THREADS) {
            int a = 0, bnd = g.n_bins - 1;
            while (a < bnd) {
                const int mid = (a + bnd) >> 1;
                if (sV[mid] > qq) bnd = mid; else a = mid + 1;
            }
            sPJ[qq + 1] = (float)a;
        }
        if (tid < W) snap[tid] = 0.0;  // row 0's window starts before the stream
        for (int i = tid; i < 16 * WP; i += S7_THREADS) Qrow[i] = 0.0;
        __syncthreads();
        if (warp == 0) {
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
        if (tid < 16) {
            const int i = tb + tid;
            float vm = 0.f, d = 0.f;
            if (i < g.n_bins) {
                const int vmi = i > 0 ? sV[i - 1] : 0;
                vm = (float)vmi;
                d = 2.f * ((float)i * vm - sPJ[vmi]);
            }
            svm[tid] = vm;
            sd[tid] = d;
        }
        __syncthreads();  // scratch rows, PJ, (vm, d) ready
        if (GT) {  // G_i(v) for every bin and count (score6.cu's table)
            float* const sG = reinterpret_cast<float*>(sm + g.o_gt);
            for (int idx = tid; idx < 16 * GP; idx += S7_THREADS) {
                const int j = idx / GP, v = idx - j * GP;
                const float fv = (float)v;
                const float nu = fmaf((float)(tb + j), fv, -sPJ[v]);
                sG[idx] = fv < svm[j] ? nu : sd[j] - nu;
            }
            __syncthreads();
        }
        };

        // ======== phase 4: stream the padded centre rows; scores the pixels whose
        // bin is in [bin_lo, bin_hi]
        auto phase4 = [&](int tb, int bin_lo, int bin_hi) {
            // this thread's 4 lanes: bins i = tb + 4 grp + j
            float vmj[4], dj[4], fi[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                vmj[j] = svm[grp * 4 + j];
                dj[j] = sd[grp * 4 + j];
                fi[j] = (float)(tb + grp * 4 + j);
            }
            // vertical window counts, 16-bit lanes: lo = lanes (4g, 4g+2), hi =
            // (4g+1, 4g+3); the count below the group (lane 4g-1) is the
            // neighbour lane's top lane
            uint32_t alo = 0, ahi = 0;
            uint32_t na = 0, nr = 0;  // entering / leaving row windows of row s (prefetched)
            // scan lane's running column prefixes Q(s, p) of bin `warp`: fp64 up to
            // the last flush + fp32 since (at most S7_NFL rows of row prefixes)
            double q[CPL];
            float qf[CPL];
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                q[k] = 0.0;
                qf[k] = 0.f;
            }
            const int xl = tid & (W - 1);  // snapshot / finish roles: tid < 2 W
            float pold = 0.f;
            const uint32_t gaddr =
                (uint32_t)__cvta_generic_to_shared(sm + g.o_gt) + grp * 4 * GP * 4 + g.moff;
            int sf = (g.nsnap - 2 * R) % g.nsnap;  // snapshot slot of row s - 2R
            {  // the first centre's window: all its rows
                const int c0 = stab[0].x;
#pragma unroll 8
                for (int dy = -R; dy <= R; ++dy) {
                    const uint32_t wa = rwt[(size_t)map_coord(c0 + dy, h, g.pad) * 4 * W];
                    alo += wa & 0x00FF00FFu;
                    ahi += (wa >> 8) & 0x00FF00FFu;
                }
                const int4 st = stab[1];
                na = rwt[st.z];
                nr = rwt[st.w];
            }
            const bool fin_warp = warp >= W / 32 && warp < 2 * W / 32;  // finished-pixel roles
            for (int s = 0; s < g.S; ++s) {
                // ---- vertical slide of the window counts (rows prefetched one ahead)
                if (s > 0) {
                    alo += (na & 0x00FF00FFu) - (nr & 0x00FF00FFu);
                    ahi += ((na >> 8) & 0x00FF00FFu) - ((nr >> 8) & 0x00FF00FFu);
                    const int4 st = stab[s + 1];
                    na = rwt[st.z];
                    nr = rwt[st.w];
                }
                // ---- E of the 4 bins (G from the shared PJ prefix table)
                const int a0 = (int)(alo & 0xFFFFu), a1 = (int)(ahi & 0xFFFFu),
                          a2 = (int)(alo >> 16), a3 = (int)(ahi >> 16);
                int a_1 = __shfl_up_sync(FULL, a3, 1);
                if (grp == 0) a_1 = 0;
                float E[4] = {0.f, 0.f, 0.f, 0.f};
                if (GT) {
                    {  // (every warp holds bin group 0, which has mass in nearly every
                       // window: no vote; a bin without mass gets E = 0 / 1 = 0)
                        const int av[5] = {a_1, a0, a1, a2, a3};
                        uint32_t ma = 0x4B000000u | (uint32_t)av[0];
                        uint32_t aa = gaddr + 4u * ma;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t mb = 0x4B000000u | (uint32_t)av[j + 1];
                            const uint32_t ab = gaddr + 4u * mb;
                            float gb, ga;
                            asm("ld.shared.f32 %0, [%1];" : "=f"(gb) : "r"(ab + j * GP * 4));
                            asm("ld.shared.f32 %0, [%1];" : "=f"(ga) : "r"(aa + j * GP * 4));
                            const float pc = __uint_as_float(mb) - __uint_as_float(ma);
                            E[j] = (gb - ga) * rcp_approx7(fmaxf(pc, 1.f));
                            ma = mb;
                            aa = ab;
                        }
                    }
                } else if (__any_sync(FULL, a3 != a_1)) {
                    const int av[5] = {a_1, a0, a1, a2, a3};
                    float pj[5];
#pragma unroll
                    for (int k = 0; k < 5; ++k) pj[k] = sPJ[av[k]];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float fa = (float)av[j], fb = (float)av[j + 1];
                        const float nua = fmaf(fi[j], fa, -pj[j]), nub = fmaf(fi[j], fb, -pj[j + 1]);
                        const float ga = fa < vmj[j] ? nua : dj[j] - nua;
                        const float gb = fb < vmj[j] ? nub : dj[j] - nub;
                        E[j] = (gb - ga) * rcp_approx7(fmaxf(fb - fa, 1.f));
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) Erow[(grp * 4 + j) * EST + x] = E[j];
                // partial map of the pixel that finishes at this row (fetched early)
                const int yf = s - 2 * R;
                if (fin_warp && yf >= 0 && yf < h) pold = part[yf * W + xl];
                __syncthreads();  // E row complete; the previous row's Q readers done
                // ---- one warp per bin: the padded E row's prefix (fp32 within the
                //      row), added to the fp64 running prefixes Q
                {
                    const float* const er = Erow + warp * EST;
                    float rp[CPL];
                    float run = 0.f;
#pragma unroll
                    for (int k = 0; k < CPL; ++k) {
                        const int p = lane * CPL + k;
                        run += p < WP ? er[scol[k]] : 0.f;
                        rp[k] = run;
                    }
                    float off = run;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const float u = __shfl_up_sync(FULL, off, o);
                        if (lane >= o) off += u;
                    }
                    off -= run;
                    double* const qr = Qrow + warp * WP;
                    float* const qfr = Qf + warp * WP;
                    const bool flush = (s % S7_NFL) == S7_NFL - 1;
#pragma unroll
                    for (int k = 0; k < CPL; ++k) {
                        const int p = lane * CPL + k;
                        qf[k] += rp[k] + off;
                        if (flush) {
                            q[k] += (double)qf[k];
                            qf[k] = 0.f;
                            if (p < WP) qr[p] = q[k];
                        }
                        if (p < WP) qfr[p] = qf[k];
                    }
                }
                __syncthreads();  // Q(s, .) published
                // ---- snapshots (pixels whose window starts at s + 1) and the
                //      pixels whose window ended at s
                // (slots: row y -> y mod nsnap; row s + 1's slot is row s - 2R's - 1)
                // D_b(s, x) = Q_b(s, x + 2R) - Q_b(s, x - 1), own bin b
                auto dwin = [&](int b) -> double {
                    const double* const qr = Qrow + b * WP;
                    const float* const qfr = Qf + b * WP;
                    const double d64 = qr[xl + 2 * R] - (xl > 0 ? qr[xl - 1] : 0.0);
                    const float d32 = qfr[xl + 2 * R] - (xl > 0 ? qfr[xl - 1] : 0.f);
                    return d64 + (double)d32;
                };
                if (tid < W) {
                    const int ys = s + 1;
                    if (ys < h) {
                        const int b = sb[ys * W + xl];
                        if (b >= bin_lo && b <= bin_hi)
                            snap[(sf == 0 ? g.nsnap - 1 : sf - 1) * W + xl] = dwin(b - tb);
                    }
                } else if (tid < 2 * W && yf >= 0 && yf < h) {
                    const int b = sb[yf * W + xl];
                    if (b >= bin_lo && b <= bin_hi) {
                        const double sc = dwin(b - tb) - snap[sf * W + xl];
                        part[yf * W + xl] = pold + fmaf((float)sc, scale, 0.f);
                    }
                }
                sf = sf + 1 == g.nsnap ? 0 : sf + 1;
            }
        };

        // ======== the channel: reference passes, then scoring passes (the last
        // reference pass's row windows are the first scoring pass's)
        const int npass = g.passes;
        if (g.fref)
            for (int p = 0; p < npass; ++p) {
                rw_phase(15 * p);
                fref_pass(15 * p, p > 0 ? 1 : 0);
            }
        for (int p = npass - 1; p >= 0; --p) {
            if (!(g.fref && p == npass - 1)) rw_phase(15 * p);
            pass_tables(15 * p);
            phase4(15 * p, p == 0 ? 0 : 15 * p + 1, min(15 * p + 15, g.n_bins - 1));
            __syncthreads();
        }
    }
}

int sample_stride(int h, int w, int budget);

template <int T>
static int s7_total(Score7Geom& g, bool gt) {
    if (gt) score7_layout<T, true>(g);
    else score7_layout<T, false>(g);
    return g.total;
}

static int nsmid7() {
    static int n = 0;
    if (n <= 0) {
        int dev = 0, sms = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 148;
        n = sms + 64;  // %smid < %nsmid; generous headroom for id gaps
    }
    return n;
}

static int score7_plan(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                       int pad, int budget, bool has_ref, Score7Geom* out, size_t* smem_out) {
    if (w != S7_W || t < 17 || t > 65 || (t & 1) == 0 || n_bins < 1 || n_bins > 256)
        return QFCA_ERR_UNSUPPORTED;
    if (h < 2 || h > 128 || (h * w) % 16) return QFCA_ERR_UNSUPPORTED;
    if (pad != QFCA_PAD_REFLECT && pad != QFCA_PAD_WRAP) return QFCA_ERR_UNSUPPORTED;
    Score7Geom g;
    memset(&g, 0, sizeof(g));
    g.h = h; g.n_bins = n_bins; g.pad = pad; g.C = C;
    g.S = h + 2 * (t / 2);
    g.nsnap = 2 * (t / 2) + 2;
    // pass p counts with lanes for bins 15p .. 15p + 15 (15 new bins after the first)
    g.passes = n_bins <= 16 ? 1 : 1 + (n_bins - 16 + 14) / 15;
    if (!has_ref) {  // in-kernel reference: the sample store must fit shared memory
        if (budget < 1) return QFCA_ERR_ARG;
        g.fref = 1;
        g.stride = sample_stride(h, w, budget);
        g.nsy = (h + g.stride - 1) / g.stride;
        g.nsx = (w + g.stride - 1) / g.stride;
        g.nsamp = g.nsy * g.nsx;
        g.srow = (g.nsamp + 3) & ~3;
        if (g.nsamp > 4096) return QFCA_ERR_UNSUPPORTED;
    }
    g.moff = 0u - 4u * 0x4B000000u;
    size_t bytes = 0;
    for (int gt = t <= S7_GT_MAXT ? 1 : 0; gt >= 0; --gt) {
        g.gt = gt;
        switch (t) {
#define S7C(TT) case TT: bytes = s7_total<TT>(g, gt != 0); break;
            S7C(17) S7C(19) S7C(21) S7C(23) S7C(25) S7C(27) S7C(29) S7C(31) S7C(33) S7C(35)
            S7C(37) S7C(39) S7C(41) S7C(43) S7C(45) S7C(47) S7C(49) S7C(51) S7C(53) S7C(55)
            S7C(57) S7C(59) S7C(61) S7C(63) S7C(65)
#undef S7C
            default: return QFCA_ERR_UNSUPPORTED;
        }
        if (bytes <= (size_t)S7_SMEM_MAX) break;
    }
    if (bytes > (size_t)S7_SMEM_MAX) return QFCA_ERR_UNSUPPORTED;
    int groups = groups_hint;
    if (groups <= 0) groups = balanced_groups(images, C, 1, 1);
    groups = groups < 1 ? 1 : (groups > C ? C : groups);
    g.cpg = (C + groups - 1) / groups;
    g.groups = (C + g.cpg - 1) / g.cpg;
    *out = g;
    *smem_out = bytes;
    return QFCA_OK;
}

int score7_query(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                 int pad, int budget, int want_fref, int* fref) {
    Score7Geom g;
    size_t smem;
    if (score7_plan(h, w, n_bins, t, C, images, groups_hint, pad, budget, want_fref == 0, &g,
                    &smem) != QFCA_OK)
        return -1;
    if (fref) *fref = g.fref;
    return g.groups;
}

int64_t score7_scratch_bytes(int h) { return (int64_t)nsmid7() * h * 4 * S7_W * 4; }

int launch_score7(const void* bins, int bins_bytes, const float* lo, const float* hi,
                  const int32_t* V, int64_t images, int C, int h, int w, int n_bins, int t,
                  int pad, int budget, int groups, void* scratch, int64_t scratch_bytes,
                  float* partial, cudaStream_t st) {
    if (bins_bytes != 1) return QFCA_ERR_UNSUPPORTED;
    if (!scratch || scratch_bytes < score7_scratch_bytes(h)) return QFCA_ERR_ARG;
    Score7Geom g;
    size_t smem;
    int rc = score7_plan(h, w, n_bins, t, C, images, groups, pad, budget, V != nullptr, &g, &smem);
    if (rc != QFCA_OK) return rc;
    if (groups > 0 && g.groups != groups) return QFCA_ERR_ARG;
    void (*kern)(const uint8_t*, const float*, const float*, const int32_t*, const Score7Geom,
                 uint32_t*, float*) = nullptr;
    switch (t) {
#define S7K(TT) case TT: kern = g.gt ? k_score7<TT, (TT <= S7_GT_MAXT)> : k_score7<TT, false>; break;
        S7K(17) S7K(19) S7K(21) S7K(23) S7K(25) S7K(27) S7K(29) S7K(31) S7K(33) S7K(35)
        S7K(37) S7K(39) S7K(41) S7K(43) S7K(45) S7K(47) S7K(49) S7K(51) S7K(53) S7K(55)
        S7K(57) S7K(59) S7K(61) S7K(63) S7K(65)
#undef S7K
        default: return QFCA_ERR_UNSUPPORTED;
    }
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return QFCA_ERR_CUDA;
    const int64_t grid = images * g.groups;
    kern<<<(unsigned)grid, S7_THREADS, smem, st>>>((const uint8_t*)bins, lo, hi, V, g,
                                                   (uint32_t*)scratch, partial);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
