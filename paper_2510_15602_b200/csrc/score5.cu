// score5.cu -- K4 v5: patch-size-independent fused scoring (any odd T with
// T^2 < 32768, N <= 16, planes of width 32 / 64 / 128).
//
// score3.cu / score4.cu keep 8-bit window counts and a T-row E ring in
// registers, so they stop at T = 15.  This kernel keeps every cost per
// (channel, pixel) independent of T -- the constant-time pooling of the
// north star -- and serves the patch-size sweep (BASELINE configs[3]):
//   * window counts in 16-bit thermometer lanes, one bin group of 4 bins per
//     sweep (lanes A_{4g-1}, A_{4g} .. A_{4g+3}); vertical sliding trackers
//     (producer warps, H1) and a row prefix scan (consumer warps, H2: the
//     window is a difference of two prefix words, modular 32-bit arithmetic is
//     exact);
//   * the T-row E ring of the vertical box lives in shared memory (one slot
//     per stream row mod T, re-anchored every T rows);
//   * the horizontal box of the own bin is a difference of two entries of a
//     per-row prefix over the padded row;
//   * the median-quan reference: per bin group, the window counts at the
//     sample positions, then a lock-step binary search with packed 16-bit
//     compares ((0x8000 | mid) - count has bit 15 set iff count <= mid).
// Same closed-form transport as score2.cu (fp32 G_i, rcp.approx).
// One channel per CTA pass; a pixel receives its channel's contribution in
// the sweep of its own bin group, so the partial map is updated once per
// channel in fixed channel order.
#include <string.h>

#include "common.cuh"

namespace qfca {

constexpr int S5_FULL0 = 3, S5_EMPTY0 = 5;  // named barriers (0 is __syncthreads)
constexpr int S5_SMEM_MAX = 227 * 1024;

struct Score5Geom {
    int h, t, r, n_bins, pad, C, groups, cpg;
    int WP;   // padded row length W + 2R
    int S;    // stream rows h + 2R
    int RC;   // stream rows per chunk
    int fref, stride, nsx, nsamp, rounds;
    int o_sb, o_chp, o_ring, o_vbp, o_pj, o_th, o_xmap, o_stab, o_misc, total;
};

__device__ __forceinline__ void bar_sync5(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive5(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float rcp_approx5(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int W>
static void score5_layout(Score5Geom& g) {
    int off = 0;
    auto take = [&](long long bytes) {
        const int o = off;
        off = (int)((off + bytes + 15) & ~15LL);
        return o;
    };
    const int n_chunks = (g.S + g.RC - 1) / g.RC;
    g.o_sb = take((long long)g.h * W);
    g.o_chp = take((long long)2 * g.RC * g.WP * 16);       // column words, double buffer
    // E ring [T][4][W] fp32 in pass 1; sample counts [nsamp] uint2 in pass 0
    const long long ring = (long long)g.t * 4 * W * 4;
    const long long sa = g.fref ? (long long)g.nsamp * 8 : 0;
    g.o_ring = take(ring > sa ? ring : sa);
    g.o_vbp = take((long long)g.RC * 4 * g.WP * 4);         // vertical sums -> row prefix
    g.o_pj = take((long long)(g.t * g.t + 1) * 4);
    g.o_th = take(256 * 16);
    g.o_xmap = take((long long)g.WP * 4);
    g.o_stab = take((long long)n_chunks * g.RC * 16);
    g.o_misc = take(1024);  // V, Vm/D, counters, scale
    g.total = off;
}

template <int W>
__global__ void __launch_bounds__(5 * W, 1)
k_score5(const uint8_t* __restrict__ bins, const float* __restrict__ lo,
         const float* __restrict__ hi, const int32_t* __restrict__ Vref, const Score5Geom g,
         float* __restrict__ partial) {
    constexpr int NT = 5 * W;   // threads
    constexpr int NC = 4 * W;   // consumers: (bin j of the group, column x)
    extern __shared__ __align__(16) uint8_t sm[];
    uint8_t* const sb = sm + g.o_sb;
    uint4* const CHp = reinterpret_cast<uint4*>(sm + g.o_chp);
    float* const ring = reinterpret_cast<float*>(sm + g.o_ring);
    uint2* const SA = reinterpret_cast<uint2*>(sm + g.o_ring);
    float* const Vbp = reinterpret_cast<float*>(sm + g.o_vbp);
    float* const sPJ = reinterpret_cast<float*>(sm + g.o_pj);
    uint4* const TH = reinterpret_cast<uint4*>(sm + g.o_th);
    int* const xmap = reinterpret_cast<int*>(sm + g.o_xmap);
    int4* const stab = reinterpret_cast<int4*>(sm + g.o_stab);
    int* const sV = reinterpret_cast<int*>(sm + g.o_misc);             // [16]
    float* const sVm = reinterpret_cast<float*>(sm + g.o_misc + 64);   // [16]
    float* const sD = reinterpret_cast<float*>(sm + g.o_misc + 128);   // [16]
    uint32_t* const cnt = reinterpret_cast<uint32_t*>(sm + g.o_misc + 192);  // [2][4]
    int* const blo = reinterpret_cast<int*>(sm + g.o_misc + 256);      // [4]
    int* const bhi = reinterpret_cast<int*>(sm + g.o_misc + 272);      // [4]
    uint32_t* const qm = reinterpret_cast<uint32_t*>(sm + g.o_misc + 288);  // [2] packed mids
    float* const sscale = reinterpret_cast<float*>(sm + g.o_misc + 304);

    const int tid = threadIdx.x;
    const bool is_p = tid >= NC;
    const int h = g.h, T = g.t, R = g.r, WP = g.WP, RC = g.RC;
    const int T2 = T * T;
    const int hw = h * W;
    const int img = blockIdx.x / g.groups, cgi = blockIdx.x % g.groups;
    const int c_begin = cgi * g.cpg, c_end = min(g.C, c_begin + g.cpg);
    float* const part = partial + ((int64_t)img * g.groups + cgi) * hw;
    const int n_chunks = (g.S + RC - 1) / RC;
    const int CHS = RC * WP;  // uint4 per CHp buffer

    // ---- per-CTA tables: stream-row slide plan, padded-x map
    for (int s = tid; s < n_chunks * RC; s += NT) {
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
        // w: sample-row index (pass 0), -1 if no sample row
        const int samp = (g.fref && e >= 0 && e < h && e % g.stride == 0) ? (e / g.stride) : -1;
        stab[s] = make_int4(add * W, rem * W, recount, samp);
    }
    for (int p = tid; p < WP; p += NT) xmap[p] = map_coord(p - R, W, g.pad);
    __syncthreads();

    // producer: column px; consumer: (bin j, column x)
    const int px = tid - NC;
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
    const int cj = tid / W, cx = tid % W;  // consumer bin slot, column
    int chalo0 = -1, chalo1 = -1;
    if (!is_p && !many_halo) {
        for (int j = 0; j < 2 * R; ++j) {
            const int p = j < R ? j : W + j;
            if (xmap[p] == cx) {
                if (chalo0 < 0) chalo0 = p;
                else if (chalo1 < 0) chalo1 = p;
            }
        }
    }
    const int warp = tid >> 5, lane = tid & 31;

    // H1 over one sweep: chunk c of stream rows into CHp[c & 1]
    uint4 cst = make_uint4(0, 0, 0, 0);
    auto h1_chunk = [&](int c) {
        uint4* base = CHp + (c & 1) * CHS;
        const uint8_t* col = sb + px;
        for (int rho = 0; rho < RC; ++rho) {
            const int4 st = stab[c * RC + rho];
            if (st.z < 0) {
                const uint4 a = TH[col[st.x]], r = TH[col[st.y]];
                cst.x += a.x - r.x;
                cst.y += a.y - r.y;
                cst.z += a.z - r.z;
            } else {
                cst = make_uint4(0, 0, 0, 0);
                for (int dy = -R; dy <= R; ++dy) {
                    const uint4 a = TH[col[map_coord(st.z + dy, h, g.pad) * W]];
                    cst.x += a.x;
                    cst.y += a.y;
                    cst.z += a.z;
                }
            }
            uint4* row = base + rho * WP;
            row[px + R] = cst;
            if (halo0 >= 0) row[halo0] = cst;
            if (halo1 >= 0) row[halo1] = cst;
            if (many_halo)
                for (int j = 0; j < 2 * R; ++j) {
                    const int p = j < R ? j : W + j;
                    if (xmap[p] == px) row[p] = cst;
                }
        }
    };
    auto produce = [&]() {
        for (int c = 0; c < n_chunks; ++c) {
            const int b = c & 1;
            if (c >= 2) bar_sync5(S5_EMPTY0 + b, NT);
            h1_chunk(c);
            bar_arrive5(S5_FULL0 + b, NT);
        }
    };
    // consumers: inclusive prefix of each chunk row of CHp[c & 1], in place
    // (one warp per row; uint32 lane words add modulo 2^32 exactly)
    auto scan_rows = [&](int c, bool samples_only) {
        uint4* base = CHp + (c & 1) * CHS;
        for (int rho = warp; rho < RC; rho += NC / 32) {
            if (samples_only && stab[c * RC + rho].w < 0) continue;
            uint4* row = base + rho * WP;
            uint32_t cx_ = 0, cy_ = 0, cz_ = 0;
            for (int b0 = 0; b0 < WP; b0 += 32) {
                const int p = b0 + lane;
                uint4 v = p < WP ? row[p] : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t ux = __shfl_up_sync(0xffffffffu, v.x, o);
                    const uint32_t uy = __shfl_up_sync(0xffffffffu, v.y, o);
                    const uint32_t uz = __shfl_up_sync(0xffffffffu, v.z, o);
                    if (lane >= o) { v.x += ux; v.y += uy; v.z += uz; }
                }
                v.x += cx_;
                v.y += cy_;
                v.z += cz_;
                if (p < WP) row[p] = v;
                cx_ = __shfl_sync(0xffffffffu, v.x, 31);
                cy_ = __shfl_sync(0xffffffffu, v.y, 31);
                cz_ = __shfl_sync(0xffffffffu, v.z, 31);
            }
        }
    };
    // window words of column x (padded x .. x + T - 1) from the row prefix
    auto window = [&](const uint4* row, int x) {
        const uint4 a = row[x + T - 1];
        const uint4 b = x > 0 ? row[x - 1] : make_uint4(0, 0, 0, 0);
        return make_uint4(a.x - b.x, a.y - b.y, a.z - b.z, 0u);
    };
    // lane k (0..4: A_{4g-1}, A_{4g}, .., A_{4g+3}) of the window words
    auto lane_of = [](const uint4& v, int k) -> uint32_t {
        const uint32_t w = k < 2 ? v.x : (k < 4 ? v.y : v.z);
        return (k & 1) ? (w >> 16) : (w & 0xFFFFu);
    };
    // thermometer table of bin group gg: lane k = [bin <= 4 gg - 1 + k]
    auto build_th = [&](int gg) {
        for (int b = tid; b < 256; b += NT) {
            uint32_t l[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) l[k] = b <= 4 * gg - 1 + k ? 1u : 0u;
            TH[b] = make_uint4(l[0] | (l[1] << 16), l[2] | (l[3] << 16), l[4], 0u);
        }
    };

    for (int c = c_begin; c < c_end; ++c) {
        const int64_t plane = (int64_t)img * g.C + c;
        __syncthreads();
        {
            const uint4* s4 = reinterpret_cast<const uint4*>(bins + plane * hw);
            uint4* d4 = reinterpret_cast<uint4*>(sb);
            for (int i = tid; i < hw / 16; i += NT) d4[i] = __ldg(s4 + i);
        }
        if (tid == 0) {
            float sc = 0.f;
            if (hi[plane] > lo[plane])
                sc = (float)(((double)hi[plane] - (double)lo[plane]) / (double)g.n_bins /
                             (double)T2);
            sscale[0] = sc;
        }
        if (!g.fref)
            for (int i = tid; i < 16; i += NT)
                sV[i] = i < g.n_bins ? __ldg(Vref + plane * g.n_bins + i) : T2;
        __syncthreads();
        const float scale = sscale[0];

        if (g.fref) {
            if (tid < 16) sV[tid] = T2;
            // ---- pass 0: per bin group, window counts at the samples, then the search
            const int c0 = g.nsamp - (g.nsamp - 1) / 2;
            for (int gg = 0; gg < 4 && 4 * gg < g.n_bins - 1 && scale != 0.f; ++gg) {
                __syncthreads();
                build_th(gg);
                __syncthreads();
                if (is_p) {
                    produce();
                } else {
                    for (int ch = 0; ch < n_chunks; ++ch) {
                        bar_sync5(S5_FULL0 + (ch & 1), NT);
                        scan_rows(ch, true);
                        asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
                        const uint4* base = CHp + (ch & 1) * CHS;
                        for (int rho = 0; rho < RC; ++rho) {
                            const int si = stab[ch * RC + rho].w;
                            if (si < 0) continue;
                            for (int sx = tid; sx < g.nsx; sx += NC) {
                                const uint4 v = window(base + rho * WP, sx * g.stride);
                                // lanes A_{4g} .. A_{4g+3}
                                SA[si * g.nsx + sx] =
                                    make_uint2((v.x >> 16) | (v.y << 16), (v.y >> 16) | (v.z << 16));
                            }
                        }
                        if (ch + 2 < n_chunks) bar_arrive5(S5_EMPTY0 + (ch & 1), NT);
                        else asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
                    }
                }
                __syncthreads();
                // lock-step search of the group's bins (16-bit packed compares)
                if (tid < 4) {
                    const int b = 4 * gg + tid;
                    const int top = b < g.n_bins - 1 ? 0 : T2;
                    blo[tid] = top;
                    bhi[tid] = T2;
                    reinterpret_cast<uint16_t*>(qm)[tid] = (uint16_t)((top + T2) >> 1);
                }
                if (tid < 8) cnt[tid] = 0;
                __syncthreads();
                for (int rd = 0; rd < g.rounds; ++rd) {
                    const int par = rd & 1;
                    const uint32_t Q0 = 0x80008000u | qm[0], Q1 = 0x80008000u | qm[1];
                    uint32_t a0 = 0, a1 = 0;
                    for (int s = tid; s < g.nsamp; s += NT) {
                        const uint2 u = SA[s];
                        a0 += __umulhi((Q0 - u.x) & 0x80008000u, 1u << 17);
                        a1 += __umulhi((Q1 - u.y) & 0x80008000u, 1u << 17);
                    }
                    a0 = __reduce_add_sync(0xffffffffu, a0);
                    a1 = __reduce_add_sync(0xffffffffu, a1);
                    if (lane == 0) {
                        atomicAdd(cnt + par * 4 + 0, a0 & 0xFFFFu);
                        atomicAdd(cnt + par * 4 + 1, a0 >> 16);
                        atomicAdd(cnt + par * 4 + 2, a1 & 0xFFFFu);
                        atomicAdd(cnt + par * 4 + 3, a1 >> 16);
                    }
                    __syncthreads();
                    if (tid < 4) {
                        const int count = (int)cnt[par * 4 + tid];
                        int a = blo[tid], bnd = bhi[tid];
                        const int mid = (a + bnd) >> 1;
                        if (count >= c0) bnd = mid; else a = mid + 1;
                        blo[tid] = a;
                        bhi[tid] = bnd;
                        reinterpret_cast<uint16_t*>(qm)[tid] = (uint16_t)((a + bnd) >> 1);
                        cnt[(par ^ 1) * 4 + tid] = 0;
                    }
                    __syncthreads();
                }
                if (tid < 4 && 4 * gg + tid < 16) sV[4 * gg + tid] = blo[tid];
                __syncthreads();
            }
            __syncthreads();
        }
        // ---- PJ = prefix of J, Vm / D per bin
        for (int q = tid; q < T2; q += NT) {
            int a = 0, bnd = g.n_bins - 1;
            while (a < bnd) {
                const int mid = (a + bnd) >> 1;
                if (sV[mid] > q) bnd = mid; else a = mid + 1;
            }
            sPJ[q + 1] = (float)a;
        }
        __syncthreads();
        if (tid < 32) {
            float carry = 0.f;
            if (lane == 0) sPJ[0] = 0.f;
            for (int base = 1; base <= T2; base += 32) {
                const int q = base + lane;
                float v = q <= T2 ? sPJ[q] : 0.f;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float u = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v += u;
                }
                v += carry;
                if (q <= T2) sPJ[q] = v;
                carry = __shfl_sync(0xffffffffu, v, 31);
            }
        }
        __syncthreads();
        if (tid < 16) {
            float vm = 0.f, d = 0.f;
            if (tid < g.n_bins) {
                const int vmi = tid > 0 ? sV[tid - 1] : 0;
                vm = (float)vmi;
                d = 2.f * ((float)tid * vm - sPJ[vmi]);
            }
            sVm[tid] = vm;
            sD[tid] = d;
        }
        __syncthreads();
        if (scale == 0.f) continue;  // degenerate channel: no contribution

        // ---- pass 1: one sweep per bin group
        for (int gg = 0; gg < 4 && 4 * gg < g.n_bins; ++gg) {
            __syncthreads();  // previous sweep's consumers are done with TH and the ring
            build_th(gg);
            for (int i = tid; i < T * 4 * W; i += NT) ring[i] = 0.f;
            __syncthreads();
            if (is_p) {
                produce();
            } else {
                const int b = 4 * gg + cj;
                const float fi = (float)b, Vm = sVm[b < 16 ? b : 15], Dv = sD[b < 16 ? b : 15];
                float vs = 0.f;
                int slot = 0;
                float* const rcol = ring + cj * W + cx;  // slot q at rcol[q * 4 * W]
                for (int ch = 0; ch < n_chunks; ++ch) {
                    bar_sync5(S5_FULL0 + (ch & 1), NT);
                    scan_rows(ch, false);
                    asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
                    const uint4* base = CHp + (ch & 1) * CHS;
                    for (int rho = 0; rho < RC; ++rho) {
                        const int s = ch * RC + rho;
                        if (s >= g.S) break;
                        const uint4 v = window(base + rho * WP, cx);
                        const uint32_t A = lane_of(v, cj + 1), Ap = lane_of(v, cj);
                        float E = 0.f;
                        if (A != Ap) {
                            const float bf = (float)A, af = (float)Ap;
                            const float nub = fmaf(fi, bf, -sPJ[A]);
                            const float nua = fmaf(fi, af, -sPJ[Ap]);
                            const float gb = bf < Vm ? nub : Dv - nub;
                            const float ga = af < Vm ? nua : Dv - nua;
                            E = (gb - ga) * rcp_approx5(bf - af);
                        }
                        float* const rs = rcol + slot * 4 * W;  // slot = s mod T
                        vs += E - *rs;
                        *rs = E;
                        if (++slot == T) {  // re-anchor the sliding sum
                            float t = 0.f;
                            for (int q = 0; q < T; ++q) t += rcol[q * 4 * W];
                            vs = t;
                            slot = 0;
                        }
                        if (s >= 2 * R) {
                            float* vrow = Vbp + (rho * 4 + cj) * WP;
                            vrow[cx + R] = vs;
                            if (chalo0 >= 0) vrow[chalo0] = vs;  // halo columns mapping here
                            if (chalo1 >= 0) vrow[chalo1] = vs;
                            if (many_halo)
                                for (int j = 0; j < 2 * R; ++j) {
                                    const int p = j < R ? j : W + j;
                                    if (xmap[p] == cx) vrow[p] = vs;
                                }
                        }
                    }
                    if (ch + 2 < n_chunks) bar_arrive5(S5_EMPTY0 + (ch & 1), NT);
                    asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");  // Vbp complete
                    // prefix of every (row, bin) line of Vbp (one warp per line)
                    for (int ln = warp; ln < RC * 4; ln += NC / 32) {
                        float* line = Vbp + ln * WP;
                        float carry = 0.f;
                        for (int b0 = 0; b0 < WP; b0 += 32) {
                            const int p = b0 + lane;
                            float val = p < WP ? line[p] : 0.f;
#pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const float u = __shfl_up_sync(0xffffffffu, val, o);
                                if (lane >= o) val += u;
                            }
                            val += carry;
                            if (p < WP) line[p] = val;
                            carry = __shfl_sync(0xffffffffu, val, 31);
                        }
                    }
                    asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
                    // A: pixels of this chunk whose bin is in the group
                    for (int task = tid; task < RC * W; task += NC) {
                        const int rho = task / W, x = task - rho * W;
                        const int y = ch * RC + rho - 2 * R;
                        if (y < 0 || y >= h) continue;
                        const int bb = sb[y * W + x] - 4 * gg;
                        if (bb < 0 || bb > 3) continue;
                        const float* line = Vbp + (rho * 4 + bb) * WP;
                        const float f = line[x + T - 1] - (x > 0 ? line[x - 1] : 0.f);
                        part[y * W + x] += f * scale;
                    }
                    asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");  // Vbp free
                }
            }
        }
    }
}

int sample_stride(int h, int w, int budget);

template <int W>
static int s5_total(Score5Geom& g) {
    score5_layout<W>(g);
    return g.total;
}

static int score5_plan(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                       int pad, int budget, bool has_ref, Score5Geom* out, size_t* smem_out) {
    if (t < 1 || (t & 1) == 0 || t * t >= 32768 || n_bins < 1 || n_bins > 16)
        return QFCA_ERR_UNSUPPORTED;
    if (w != 32 && w != 64 && w != 128) return QFCA_ERR_UNSUPPORTED;
    if (h < 1 || (int64_t)h * w > (1 << 20) || ((int64_t)h * w) % 16) return QFCA_ERR_UNSUPPORTED;
    if (pad != QFCA_PAD_REFLECT && pad != QFCA_PAD_WRAP) return QFCA_ERR_UNSUPPORTED;
    Score5Geom g;
    memset(&g, 0, sizeof(g));
    g.h = h; g.t = t; g.r = t / 2; g.n_bins = n_bins; g.pad = pad; g.C = C;
    g.WP = w + 2 * g.r;
    g.S = h + 2 * g.r;
    if (!has_ref) {
        if (budget < 1 || !(pad == QFCA_PAD_WRAP || h > 1)) return QFCA_ERR_UNSUPPORTED;
        g.fref = 1;
        g.stride = sample_stride(h, w, budget);
        g.nsx = (w + g.stride - 1) / g.stride;
        g.nsamp = ((h + g.stride - 1) / g.stride) * g.nsx;
        if (g.nsamp >= 65536) return QFCA_ERR_UNSUPPORTED;
        int r = 0;
        while ((1 << r) < t * t + 1) ++r;
        g.rounds = r;
    }
    size_t bytes = 0;
    for (int rc = 16; rc >= 2; rc /= 2) {
        g.RC = rc;
        switch (w) {
            case 32: bytes = s5_total<32>(g); break;
            case 64: bytes = s5_total<64>(g); break;
            default: bytes = s5_total<128>(g); break;
        }
        if (bytes <= (size_t)S5_SMEM_MAX) break;
    }
    if (bytes > (size_t)S5_SMEM_MAX) return QFCA_ERR_UNSUPPORTED;
    int groups = groups_hint;
    if (groups <= 0) groups = balanced_groups(images, C, 1, 1);
    groups = groups < 1 ? 1 : (groups > C ? C : groups);
    g.cpg = (C + groups - 1) / groups;
    g.groups = (C + g.cpg - 1) / g.cpg;
    *out = g;
    *smem_out = bytes;
    return QFCA_OK;
}

int score5_query(int h, int w, int n_bins, int t, int C, int64_t images, int groups_hint,
                 int pad, int budget, int want_fref, int* fref) {
    Score5Geom g;
    size_t smem;
    if (score5_plan(h, w, n_bins, t, C, images, groups_hint, pad, budget, want_fref == 0, &g,
                    &smem) != QFCA_OK)
        return -1;
    if (fref) *fref = g.fref;
    return g.groups;
}

int launch_score5(const void* bins, int bins_bytes, const float* lo, const float* hi,
                  const int32_t* V, int64_t images, int C, int h, int w, int n_bins, int t,
                  int pad, int budget, int groups, float* partial, cudaStream_t st) {
    if (bins_bytes != 1) return QFCA_ERR_UNSUPPORTED;
    Score5Geom g;
    size_t smem;
    int rc = score5_plan(h, w, n_bins, t, C, images, groups, pad, budget, V != nullptr, &g,
                         &smem);
    if (rc != QFCA_OK) return rc;
    if (groups > 0 && g.groups != groups) return QFCA_ERR_ARG;
    void (*kern)(const uint8_t*, const float*, const float*, const int32_t*, const Score5Geom,
                 float*) = w == 32 ? k_score5<32> : (w == 64 ? k_score5<64> : k_score5<128>);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return QFCA_ERR_CUDA;
    const int64_t grid = images * g.groups;
    kern<<<(unsigned)grid, 5 * w, smem, st>>>((const uint8_t*)bins, lo, hi, V, g, partial);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
