// tiles.cu -- gather of the row-band x column-strip tiles of wide bin planes
// (sharding.py _strip_partial, configs[4]: 1024^2 feature planes scored by the
// 128-column fused kernel).  out[t][c][y][x] = bins[c][r_t + y][a_t + x] with
// t = (row band, column strip); 4-byte words (tile starts are multiples of 4
// columns: strip step 128 - 4 (T/2), last strip w - 128).
#include "common.cuh"

namespace qfca {

__global__ void k_gather_tiles(const uint32_t* __restrict__ bins, int C, int h, int w,
                               const int* __restrict__ rst, int nr, const int* __restrict__ cst,
                               int ncs, int th, int tw, uint32_t* __restrict__ out) {
    const int tw4 = tw / 4, w4 = w / 4;
    const int64_t total = (int64_t)nr * ncs * C * th * tw4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t q = i;
        const int x4 = (int)(q % tw4);
        q /= tw4;
        const int y = (int)(q % th);
        q /= th;
        const int c = (int)(q % C);
        q /= C;
        const int s = (int)(q % ncs);
        const int r = (int)(q / ncs);
        out[i] = bins[((int64_t)c * h + rst[r] + y) * w4 + cst[s] / 4 + x4];
    }
}

int launch_gather_tiles(const void* bins, int C, int h, int w, const int* rst, int nr,
                        const int* cst, int ncs, int th, int tw, void* out, cudaStream_t st) {
    if (C <= 0 || h <= 0 || w <= 0 || nr <= 0 || ncs <= 0 || th <= 0 || tw <= 0)
        return QFCA_ERR_ARG;
    if (w % 4 || tw % 4 || (reinterpret_cast<uintptr_t>(bins) & 3) ||
        (reinterpret_cast<uintptr_t>(out) & 3))
        return QFCA_ERR_UNSUPPORTED;
    k_gather_tiles<<<148 * 16, 256, 0, st>>>((const uint32_t*)bins, C, h, w, rst, nr, cst, ncs,
                                             th, tw, (uint32_t*)out);
    return cudaGetLastError() == cudaSuccess ? QFCA_OK : QFCA_ERR_CUDA;
}

}  // namespace qfca
