// capi.cu -- extern "C" entry points declared in include/qfca_b200.h.
#include <math.h>

#include <vector>

#include "../../include/qfca_b200.h"
#include "common.cuh"

namespace qfca {
int launch_pool_interior(const void*, const void* const*, int32_t, const uint8_t*,
                         const uint8_t* const*, int32_t, int32_t, int32_t, int32_t, double*,
                         uint8_t*, float*, int32_t*, unsigned long long*, cudaStream_t);
int64_t rank_stats_workspace_bytes(int64_t, int32_t);
int launch_rank_stats(const void*, int32_t, const uint8_t*, int64_t, void*, int64_t, void*,
                      unsigned long long*, cudaStream_t);
int64_t components_workspace_bytes(int64_t);
int launch_components(const uint8_t*, int32_t, int32_t, int32_t, void*, int64_t, int32_t*, int32_t*,
                      int32_t*, cudaStream_t);
int launch_pro_histograms(const double*, const int32_t*, int64_t, const double*, int32_t, int32_t,
                          int32_t, int32_t*, unsigned long long*, cudaStream_t);
int launch_pro_accumulate(int32_t*, int32_t, int32_t, double*, cudaStream_t);
int launch_minmax(const float*, int64_t, int64_t, float*, float*, int*, cudaStream_t);
int launch_quantize_fused(const float*, int64_t, int64_t, int, float*, float*, int*, void*, int,
                          cudaStream_t);
int launch_bin(const float*, int64_t, int64_t, const float*, const float*, int, void*, int,
               cudaStream_t);
int launch_plane_mean(const float*, int64_t, int64_t, double*, cudaStream_t);
int sample_stride(int, int, int);
int launch_reference(const void*, int, const float*, const float*, int64_t, int, int, int, int,
                     int, int, int, int32_t*, cudaStream_t);
int launch_window_counts(const void*, int, int64_t, int, int, int, int, int, uint16_t*, void*, int,
                         cudaStream_t);
int launch_mismatch_pixels(const uint16_t*, int64_t, int64_t, int, const double*, const double*,
                           const uint8_t*, double*, cudaStream_t);
int launch_mismatch_rows(const double*, int64_t, int, const double*, const double*, double*,
                         cudaStream_t);
int launch_smooth_gather(const double*, const void*, int, int64_t, int, int, int, int, int,
                         const double*, double, double*, double*, cudaStream_t);
int launch_channel_sum(const double*, int64_t, int, int64_t, const uint8_t*, int, double*, int*,
                       cudaStream_t);
int launch_count_used(const float*, const float*, int64_t, int, int*, cudaStream_t);
int score_groups(int, int, int, int, int, int64_t, int);
int launch_score(const void*, int, const float*, const float*, const int32_t*, int64_t, int, int,
                 int, int, int, int, int, float*, cudaStream_t);
int launch_reduce_partials(const float*, int64_t, int, int64_t, const int*, double*,
                           cudaStream_t);
int launch_divide_used(const double*, int64_t, int64_t, const int*, double*, cudaStream_t);
int launch_sep_conv(const double*, int64_t, int, int, int, const double*, int, int, double*,
                    cudaStream_t);
int launch_image_score(const double*, int64_t, int, int, int, double*, cudaStream_t);
int launch_upsample(const double*, int64_t, int, int, int, int, float*, cudaStream_t);
int launch_pca_residual(const float*, int64_t, int, int64_t, const double*, const double*, int,
                        int, float*, cudaStream_t);
int launch_center(const float*, int64_t, int64_t, const double*, float*, cudaStream_t);
int launch_cholqr(double*, int64_t, int, int, cudaStream_t);
int64_t cov_i8_workspace(int64_t, int, int);
int launch_chol_rinv(const double*, int64_t, int, double*, cudaStream_t);
int launch_sym_eig(const double*, int64_t, int, double*, double*, cudaStream_t);
int launch_lanczos(const double*, int64_t, int, int, const double*, double*, double*, double*,
                   double*, int*, cudaStream_t);
int launch_ritz(const double*, int64_t, int, const double*, int, double*, double*, cudaStream_t);
int launch_pad_planes(const void*, int64_t, int, int, int, int, int, int, void*, cudaStream_t);
int launch_build_sat(const void*, int, int64_t, int, int, int, int, int, double*, cudaStream_t);
int launch_sat_box(const double*, int64_t, int, int, int, int, double, double*, cudaStream_t);
int launch_sat_rects(const double*, int, const int32_t*, int64_t, double*, cudaStream_t);
int launch_naive_box(const void*, int, int64_t, int, int, int, int, int, double*, cudaStream_t);
int launch_gather_tiles(const void*, int, int, int, const int*, int, const int*, int, int, int, void*,
                        cudaStream_t);
int launch_cov_i8(const float*, int64_t, int, int, const double*, double*, void*, int64_t,
                  double*, cudaStream_t);
int score2_query(int, int, int, int, int, int64_t, int, int, int, int, int*);
int launch_score2(const void*, int, const float*, const float*, const int32_t*, int64_t, int, int,
                  int, int, int, int, int, int, float*, cudaStream_t);

int score3_query(int, int, int, int, int, int64_t, int, int, int, int, int*);
int launch_score3(const void*, int, const float*, const float*, const int32_t*, int64_t, int, int,
                  int, int, int, int, int, int, float*, cudaStream_t);
int score4_query(int, int, int, int, int, int64_t, int, int, int, int, int*);
int score5_query(int, int, int, int, int, int64_t, int, int, int, int, int*);
int launch_score5(const void*, int, const float*, const float*, const int32_t*, int64_t, int, int,
                  int, int, int, int, int, int, float*, cudaStream_t);
int launch_score4(const void*, int, const float*, const float*, const int32_t*, int64_t, int, int,
                  int, int, int, int, int, int, float*, cudaStream_t);
int score6_query(int, int, int, int, int, int64_t, int, int, int, int, int*);
int64_t reference_weights_workspace_bytes(int64_t, int, int, int, int, int, int);
int launch_pca_residual_slice(const float*, int64_t, int, int64_t, const double*, const double*,
                              int, int, int, int, float*, cudaStream_t);
int launch_reference_weights(const float*, const void*, int, const float*, const float*, int64_t,
                             int, int, int, int, int, int, int, void*, int64_t, double*,
                             cudaStream_t);
int64_t score6_scratch_bytes(int);
int launch_score6(const void*, int, const float*, const float*, const int32_t*, int64_t, int, int,
                  int, int, int, int, int, int, void*, int64_t, float*, cudaStream_t);
int launch_score6_src(const void*, int, const float*, const float*, const int32_t*, int64_t, int,
                      int, int, int, int, int, int, int, void*, int64_t, float*, cudaStream_t,
                      const int*, const int*, int, int, int, int);
int score7_query(int, int, int, int, int, int64_t, int, int, int, int, int*);
int64_t score7_scratch_bytes(int);
int launch_score7(const void*, int, const float*, const float*, const int32_t*, int64_t, int, int,
                  int, int, int, int, int, int, void*, int64_t, float*, cudaStream_t);

// fused-kernel selection: 0 = auto (with a caller-supplied scratch v6, else v7;
// then v4, v3, v5, v2, v1 -- the first that applies), 1 .. 7 = force that version
static int g_score_kernel = 0;

struct ScoreChoice {
    int groups;  // channel groups (partial maps per image); <= 0: unsupported
    int ver;     // N: scoreN.cu (1: score.cu)
    int fref;    // 1: the reference is selected inside the kernel
};

// want_fref: the caller has no reference (V) and wants the kernel to select it
static ScoreChoice score_choose(int h, int w, int n_bins, int t, int C, int64_t images,
                                int groups_hint, int bins_bytes, int pad, int budget,
                                int want_fref, int allow_scratch = 0) {
    ScoreChoice ch{-1, 1, 0};
    if (allow_scratch && (g_score_kernel == 0 || g_score_kernel == 6) && bins_bytes == 1) {
        int fr = 0;
        const int gg = score6_query(h, w, n_bins, t, C, images, groups_hint, pad, budget,
                                    want_fref, &fr);
        // v6 either selects the reference itself or takes the caller's
        if (gg > 0 && fr == (want_fref ? 1 : 0)) return ScoreChoice{gg, 6, fr};
    }
    if (g_score_kernel == 6) return ch;
    if (allow_scratch && (g_score_kernel == 0 || g_score_kernel == 7) && bins_bytes == 1) {
        // large patches: v7 selects the reference itself when its sample store
        // fits, else takes the caller's (K3)
        int fr = 0;
        int gg = score7_query(h, w, n_bins, t, C, images, groups_hint, pad, budget, want_fref, &fr);
        if (gg <= 0 && want_fref)
            gg = score7_query(h, w, n_bins, t, C, images, groups_hint, pad, budget, 0, &fr);
        if (gg > 0) return ScoreChoice{gg, 7, fr};
    }
    if (g_score_kernel == 7) return ch;
    if ((g_score_kernel == 0 || g_score_kernel == 4) && bins_bytes == 1) {
        int fr = 0;
        const int gg = score4_query(h, w, n_bins, t, C, images, groups_hint, pad, budget,
                                    want_fref, &fr);
        // v4 either selects the reference itself or takes the caller's
        if (gg > 0 && fr == (want_fref ? 1 : 0)) return ScoreChoice{gg, 4, fr};
    }
    if (g_score_kernel == 4) return ch;
    if ((g_score_kernel == 0 || g_score_kernel == 3) && bins_bytes == 1) {
        int fr = 0;
        const int gg = score3_query(h, w, n_bins, t, C, images, groups_hint, pad, budget,
                                    want_fref, &fr);
        if (gg > 0) return ScoreChoice{gg, 3, fr};
    }
    if (g_score_kernel == 3) return ch;
    if ((g_score_kernel == 0 || g_score_kernel == 5) && bins_bytes == 1) {
        int fr = 0;
        const int gg = score5_query(h, w, n_bins, t, C, images, groups_hint, pad, budget,
                                    want_fref, &fr);
        if (gg > 0 && fr == (want_fref ? 1 : 0)) return ScoreChoice{gg, 5, fr};
    }
    if (g_score_kernel == 5) return ch;
    if ((g_score_kernel == 0 || g_score_kernel == 2) && bins_bytes == 1) {
        int fr = 0;
        const int gg = score2_query(h, w, n_bins, t, C, images, groups_hint, pad, budget,
                                    want_fref, &fr);
        if (gg > 0) return ScoreChoice{gg, 2, fr};
    }
    if (g_score_kernel == 2) return ch;
    ch.groups = score_groups(h, w, n_bins, t, C, images, groups_hint);
    return ch;
}

static int64_t choice_scratch_bytes(const ScoreChoice& ch, int h) {
    return ch.ver == 6 ? score6_scratch_bytes(h) : ch.ver == 7 ? score7_scratch_bytes(h) : 0;
}

static int launch_score_any(const ScoreChoice& ch, const void* bins, int bins_bytes,
                            const float* lo, const float* hi, const int32_t* V, int64_t images,
                            int C, int h, int w, int n_bins, int t, int pad, int budget,
                            float* partial, cudaStream_t st, void* scratch = nullptr,
                            int64_t scratch_bytes = 0) {
    if (ch.groups <= 0) return QFCA_ERR_UNSUPPORTED;
    if (ch.ver == 6)
        return launch_score6(bins, bins_bytes, lo, hi, ch.fref ? nullptr : V, images, C, h, w,
                             n_bins, t, pad, budget, ch.groups, scratch, scratch_bytes, partial,
                             st);
    if (ch.ver == 7)
        return launch_score7(bins, bins_bytes, lo, hi, ch.fref ? nullptr : V, images, C, h, w,
                             n_bins, t, pad, budget, ch.groups, scratch, scratch_bytes, partial,
                             st);
    if (ch.ver == 5)
        return launch_score5(bins, bins_bytes, lo, hi, ch.fref ? nullptr : V, images, C, h, w,
                             n_bins, t, pad, budget, ch.groups, partial, st);
    if (ch.ver == 4)
        return launch_score4(bins, bins_bytes, lo, hi, ch.fref ? nullptr : V, images, C, h, w,
                             n_bins, t, pad, budget, ch.groups, partial, st);
    if (ch.ver == 3)
        return launch_score3(bins, bins_bytes, lo, hi, ch.fref ? nullptr : V, images, C, h, w,
                             n_bins, t, pad, budget, ch.groups, partial, st);
    if (ch.ver == 2)
        return launch_score2(bins, bins_bytes, lo, hi, ch.fref ? nullptr : V, images, C, h, w,
                             n_bins, t, pad, budget, ch.groups, partial, st);
    if (!V) return QFCA_ERR_UNSUPPORTED;
    return launch_score(bins, bins_bytes, lo, hi, V, images, C, h, w, n_bins, t, pad, ch.groups,
                        partial, st);
}
}  // namespace qfca

using namespace qfca;

#include <atomic>
// launches of this library's kernels since load (evidence for the bench's
// gpu_launches claim); only successful launches are counted
static std::atomic<long long> g_launches{0};
static inline int counted(int status, int kernels) {
    if (status == QFCA_OK) g_launches.fetch_add(kernels, std::memory_order_relaxed);
    return status;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int qfca_abi_version(void) { return 1; }

int64_t qfca_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* qfca_status_str(int status) {
    switch (status) {
        case QFCA_OK: return "ok";
        case QFCA_ERR_ARG: return "invalid argument";
        case QFCA_ERR_CUDA: return "CUDA error";
        case QFCA_ERR_UNSUPPORTED: return "configuration not supported by this kernel";
        default: return "unknown status";
    }
}

int qfca_fit_quantizer(const float* x, int64_t planes, int64_t plane_len, float* lo, float* hi,
                       int32_t* nonfinite, void* stream) {
    return counted(launch_minmax(x, planes, plane_len, lo, hi, nonfinite, S(stream)), 1);
}

int qfca_bin_indices(const float* x, int64_t planes, int64_t plane_len, const float* lo,
                     const float* hi, int32_t n_bins, void* bins, int32_t bins_bytes,
                     void* stream) {
    return counted(launch_bin(x, planes, plane_len, lo, hi, n_bins, bins, bins_bytes, S(stream)), 1);
}

int qfca_quantize(const float* x, int64_t planes, int64_t plane_len, int32_t n_bins, float* lo,
                  float* hi, int32_t* nonfinite, void* bins, int32_t bins_bytes, void* stream) {
    int rc = launch_quantize_fused(x, planes, plane_len, n_bins, lo, hi, nonfinite, bins,
                                   bins_bytes, S(stream));
    if (rc != QFCA_ERR_UNSUPPORTED) return counted(rc, 1);
    if ((rc = counted(launch_minmax(x, planes, plane_len, lo, hi, nonfinite, S(stream)), 1)))
        return rc;
    return counted(launch_bin(x, planes, plane_len, lo, hi, n_bins, bins, bins_bytes, S(stream)), 1);
}

int qfca_sample_stride(int32_t h, int32_t w, int32_t sample_budget) {
    if (h <= 0 || w <= 0 || sample_budget < 1) return -1;
    return sample_stride(h, w, sample_budget);
}

int qfca_select_reference(const void* bins, int32_t bins_bytes, const float* lo, const float* hi,
                          int64_t planes, int32_t h, int32_t w, int32_t n_bins,
                          int32_t patch_size, int32_t pad, int32_t sample_budget, int32_t mode,
                          int32_t* stats, void* stream) {
    if (pad < 0 || pad > 2) return QFCA_ERR_ARG;
    return counted(launch_reference(bins, bins_bytes, lo, hi, planes, h, w, n_bins, patch_size, pad,
                            sample_budget, mode, stats, S(stream)), 1);
}

int qfca_window_counts(const void* bins, int32_t bins_bytes, int64_t planes, int32_t h,
                       int32_t w, int32_t n_bins, int32_t patch_size, int32_t pad,
                       uint16_t* scratch, void* counts, int32_t counts_kind, void* stream) {
    if (pad < 0 || pad > 2) return QFCA_ERR_ARG;
    return counted(launch_window_counts(bins, bins_bytes, planes, h, w, n_bins, patch_size, pad, scratch,
                                counts, counts_kind, S(stream)), 2);
}

int qfca_mismatch_pixels(const uint16_t* counts, int64_t planes, int64_t hw, int32_t n_bins,
                         const double* ref_weights, const double* centers, const uint8_t* skip,
                         double* err, void* stream) {
    return counted(launch_mismatch_pixels(counts, planes, hw, n_bins, ref_weights, centers, skip, err,
                                  S(stream)), 1);
}

int qfca_mismatch_rows(const double* Pb, int64_t rows, int32_t n_bins, const double* R,
                       const double* Q, double* out, void* stream) {
    return counted(launch_mismatch_rows(Pb, rows, n_bins, R, Q, out, S(stream)), 1);
}

int qfca_smooth_gather(const double* err, const void* bins, int32_t bins_bytes, int64_t planes,
                       int32_t h, int32_t w, int32_t n_bins, int32_t patch_size, int32_t pad,
                       const double* taps_host, double post_scale, double* scratch,
                       double* score, void* stream) {
    if (pad < 0 || pad > 2 || !taps_host) return QFCA_ERR_ARG;
    return counted(launch_smooth_gather(err, bins, bins_bytes, planes, h, w, n_bins, patch_size, pad,
                                taps_host, post_scale, scratch, score, S(stream)), 2);
}

int qfca_channel_sum(const double* score, int64_t images, int32_t channels, int64_t hw,
                     const uint8_t* skip, int32_t accumulate, double* acc, int32_t* used,
                     void* stream) {
    return counted(launch_channel_sum(score, images, channels, hw, skip, accumulate, acc, used,
                              S(stream)), 1);
}

int qfca_count_used(const float* lo, const float* hi, int64_t images, int32_t channels,
                    int32_t* used, void* stream) {
    return counted(launch_count_used(lo, hi, images, channels, used, S(stream)), 1);
}

int qfca_score_groups(int32_t h, int32_t w, int32_t n_bins, int32_t patch_size, int32_t channels,
                      int64_t images, int32_t groups_hint, int32_t pad, int32_t sample_budget,
                      int32_t with_reference) {
    const ScoreChoice ch = score_choose(h, w, n_bins, patch_size, channels, images, groups_hint,
                                        n_bins <= 256 ? 1 : 2, pad, sample_budget,
                                        with_reference ? 0 : 1);
    if (!with_reference && !ch.fref) return -1;
    return ch.groups;
}

int qfca_score_groups_ex(int32_t h, int32_t w, int32_t n_bins, int32_t patch_size,
                         int32_t channels, int64_t images, int32_t groups_hint, int32_t pad,
                         int32_t sample_budget, int32_t with_reference, int32_t with_scratch) {
    const ScoreChoice ch = score_choose(h, w, n_bins, patch_size, channels, images, groups_hint,
                                        n_bins <= 256 ? 1 : 2, pad, sample_budget,
                                        with_reference ? 0 : 1, with_scratch);
    if (!with_reference && !ch.fref) return -1;
    return ch.groups;
}

int64_t qfca_score_scratch_bytes(int32_t h, int32_t w, int32_t n_bins, int32_t patch_size,
                                 int32_t channels, int64_t images, int32_t groups_hint,
                                 int32_t pad, int32_t sample_budget, int32_t with_reference) {
    const ScoreChoice ch = score_choose(h, w, n_bins, patch_size, channels, images, groups_hint,
                                        n_bins <= 256 ? 1 : 2, pad, sample_budget,
                                        with_reference ? 0 : 1, 1);
    if (ch.groups <= 0 || (!with_reference && !ch.fref)) return -1;
    return choice_scratch_bytes(ch, h);
}

int qfca_score_version(int32_t h, int32_t w, int32_t n_bins, int32_t patch_size,
                       int32_t channels, int64_t images, int32_t pad, int32_t sample_budget,
                       int32_t with_reference) {
    // the choice qfca_detect makes (its workspace carries the v6 scratch)
    const ScoreChoice ch = score_choose(h, w, n_bins, patch_size, channels, images, 0,
                                        n_bins <= 256 ? 1 : 2, pad, sample_budget,
                                        with_reference ? 0 : 1, 1);
    if (ch.groups <= 0 || (!with_reference && !ch.fref)) return -1;
    return ch.ver;
}

int qfca_set_score_kernel(int32_t version) {
    if (version < 0 || version > 7) return QFCA_ERR_ARG;
    g_score_kernel = version;
    return QFCA_OK;
}

int qfca_score(const void* bins, int32_t bins_bytes, const float* lo, const float* hi,
               const int32_t* ref_cum, int64_t images, int32_t channels, int32_t h, int32_t w,
               int32_t n_bins, int32_t patch_size, int32_t pad, int32_t sample_budget,
               int32_t groups, float* partial, void* stream) {
    const ScoreChoice ch = score_choose(h, w, n_bins, patch_size, channels, images, groups,
                                        bins_bytes, pad, sample_budget, ref_cum ? 0 : 1);
    if (groups > 0 && ch.groups != groups) return QFCA_ERR_ARG;
    if (!ref_cum && !ch.fref) return QFCA_ERR_UNSUPPORTED;
    return counted(launch_score_any(ch, bins, bins_bytes, lo, hi, ref_cum, images, channels, h,
                                    w, n_bins, patch_size, pad, sample_budget, partial, S(stream)),
                   1);
}

int qfca_score_ex(const void* bins, int32_t bins_bytes, const float* lo, const float* hi,
                  const int32_t* ref_cum, int64_t images, int32_t channels, int32_t h, int32_t w,
                  int32_t n_bins, int32_t patch_size, int32_t pad, int32_t sample_budget,
                  int32_t groups, void* scratch, int64_t scratch_bytes, float* partial,
                  void* stream) {
    const ScoreChoice ch = score_choose(h, w, n_bins, patch_size, channels, images, groups,
                                        bins_bytes, pad, sample_budget, ref_cum ? 0 : 1,
                                        scratch != nullptr && scratch_bytes > 0);
    if (groups > 0 && ch.groups != groups) return QFCA_ERR_ARG;
    if (!ref_cum && !ch.fref) return QFCA_ERR_UNSUPPORTED;
    if (scratch_bytes < choice_scratch_bytes(ch, h)) return QFCA_ERR_ARG;
    return counted(launch_score_any(ch, bins, bins_bytes, lo, hi, ref_cum, images, channels, h,
                                    w, n_bins, patch_size, pad, sample_budget, partial, S(stream),
                                    scratch, scratch_bytes),
                   1);
}

int qfca_score_tiles(const void* bins, int32_t bins_bytes, const float* lo, const float* hi,
                     const int32_t* ref_cum, int32_t channels, int32_t hbig, int32_t wbig,
                     const int32_t* rst, int32_t nr, const int32_t* cst, int32_t ncs,
                     int32_t col_align, int32_t th, int32_t tw, int32_t n_bins,
                     int32_t patch_size, int32_t pad, int32_t sample_budget, int32_t groups,
                     void* scratch, int64_t scratch_bytes, float* partial, void* stream) {
    if (!bins || !ref_cum || !rst || !cst || nr < 1 || ncs < 1 || th < 1 || th > hbig ||
        tw > wbig)
        return QFCA_ERR_ARG;
    const int64_t images = (int64_t)nr * ncs;
    const ScoreChoice ch = score_choose(th, tw, n_bins, patch_size, channels, images, groups,
                                        bins_bytes, pad, sample_budget, 0,
                                        scratch != nullptr && scratch_bytes > 0);
    if (ch.ver != 6 || ch.fref) return QFCA_ERR_UNSUPPORTED;  // the in-place read is v6's
    if (groups > 0 && ch.groups != groups) return QFCA_ERR_ARG;
    if (scratch_bytes < choice_scratch_bytes(ch, th)) return QFCA_ERR_ARG;
    const int csz = col_align % 16 == 0 ? 16 : (col_align % 8 == 0 ? 8 : 4);
    if (col_align % 4) return QFCA_ERR_UNSUPPORTED;
    return counted(launch_score6_src(bins, bins_bytes, lo, hi, ref_cum, images, channels, th, tw,
                                     n_bins, patch_size, pad, sample_budget, ch.groups, scratch,
                                     scratch_bytes, partial, S(stream), rst, cst, ncs, hbig,
                                     wbig, csz),
                   1);
}

int qfca_reduce_partials(const float* partial, int64_t images, int32_t groups, int64_t hw,
                         const int32_t* used, double* agg, void* stream) {
    return counted(launch_reduce_partials(partial, images, groups, hw, used, agg, S(stream)), 1);
}

int qfca_divide_used(const double* acc, int64_t images, int64_t hw, const int32_t* used,
                     double* agg, void* stream) {
    return counted(launch_divide_used(acc, images, hw, used, agg, S(stream)), 1);
}

int qfca_sep_conv(const double* in, int64_t images, int32_t h, int32_t w, int32_t axis,
                  const double* taps_host, int32_t ntaps, int32_t pad, double* out, void* stream) {
    if (pad < 0 || pad > 2 || !taps_host || (axis != 0 && axis != 1)) return QFCA_ERR_ARG;
    return counted(launch_sep_conv(in, images, h, w, axis, taps_host, ntaps, pad, out, S(stream)), 1);
}

int qfca_image_score(const double* scores, int64_t images, int32_t h, int32_t w, int32_t border,
                     double* image_score, void* stream) {
    return counted(launch_image_score(scores, images, h, w, border, image_score, S(stream)), 1);
}

int qfca_upsample(const double* in, int64_t images, int32_t h, int32_t w, int32_t out_h,
                  int32_t out_w, float* out, void* stream) {
    return counted(launch_upsample(in, images, h, w, out_h, out_w, out, S(stream)), 1);
}

int qfca_plane_mean(const float* x, int64_t planes, int64_t plane_len, double* mean,
                    void* stream) {
    return counted(launch_plane_mean(x, planes, plane_len, mean, S(stream)), 1);
}

int qfca_center(const float* x, int64_t planes, int64_t plane_len, const double* mean, float* out,
                void* stream) {
    return counted(launch_center(x, planes, plane_len, mean, out, S(stream)), 1);
}

int qfca_pca_residual(const float* x, int64_t images, int32_t channels, int64_t hw,
                      const double* mean, const double* comps, int32_t k,
                      int32_t per_image_model, float* out, void* stream) {
    return counted(launch_pca_residual(x, images, channels, hw, mean, comps, k, per_image_model, out,
                               S(stream)), 1);
}

int qfca_cholqr(double* blocks, int64_t batch, int32_t rows, int32_t cols, void* stream) {
    return counted(launch_cholqr(blocks, batch, rows, cols, S(stream)), 1);
}

int qfca_chol_rinv(const double* gram, int64_t batch, int32_t p, double* rinv, void* stream) {
    return counted(launch_chol_rinv(gram, batch, p, rinv, S(stream)), 1);
}

int qfca_sym_eig(const double* h, int64_t batch, int32_t p, double* evals, double* evecs,
                 void* stream) {
    return counted(launch_sym_eig(h, batch, p, evals, evecs, S(stream)), 1);
}

int qfca_lanczos(const double* cov, int64_t batch, int32_t C, int32_t passes, const double* q0,
                 double* basis, double* h, double* twin_basis, double* exchange,
                 int32_t* flags, void* stream) {
    return counted(launch_lanczos(cov, batch, C, passes, q0, basis, h, twin_basis, exchange,
                                  flags, S(stream)), 1);
}

int qfca_ritz(const double* h, int64_t batch, int32_t n, const double* x0, int32_t iters,
              double* x, double* hm, void* stream) {
    return counted(launch_ritz(h, batch, n, x0, iters, x, hm, S(stream)), 1);
}

int qfca_pad_planes(const void* x, int64_t planes, int32_t h, int32_t w, int32_t margin,
                    int32_t mode_rows, int32_t mode_cols, int32_t elem_bytes, void* out,
                    void* stream) {
    return counted(launch_pad_planes(x, planes, h, w, margin, mode_rows, mode_cols, elem_bytes,
                                     out, S(stream)), 1);
}

int qfca_build_sat(const void* x, int32_t dtype, int64_t planes, int32_t h, int32_t w,
                   int32_t margin, int32_t mode_rows, int32_t mode_cols, double* cumsum,
                   void* stream) {
    return counted(launch_build_sat(x, dtype, planes, h, w, margin, mode_rows, mode_cols, cumsum,
                                    S(stream)), 2);
}

int qfca_sat_box(const double* cumsum, int64_t planes, int32_t h, int32_t w, int32_t k,
                 int32_t clamp, double divisor, double* out, void* stream) {
    return counted(launch_sat_box(cumsum, planes, h, w, k, clamp, divisor, out, S(stream)), 1);
}

int qfca_sat_rects(const double* cumsum, int32_t sat_w, const int32_t* rects, int64_t n,
                   double* out, void* stream) {
    return counted(launch_sat_rects(cumsum, sat_w, rects, n, out, S(stream)), 1);
}

int qfca_naive_box(const void* x, int32_t dtype, int64_t planes, int32_t h, int32_t w, int32_t k,
                   int32_t mode_rows, int32_t mode_cols, double* out, void* stream) {
    return counted(launch_naive_box(x, dtype, planes, h, w, k, mode_rows, mode_cols, out,
                                    S(stream)), 1);
}

int qfca_pca_residual_slice(const float* x, int64_t images, int32_t channels, int64_t hw,
                            const double* mean, const double* comps, int32_t k,
                            int32_t per_image_model, int32_t c_lo, int32_t c_hi, float* out,
                            void* stream) {
    return counted(launch_pca_residual_slice(x, images, channels, hw, mean, comps, k,
                                             per_image_model, c_lo, c_hi, out, S(stream)),
                   1);
}

int64_t qfca_reference_weights_workspace_bytes(int64_t planes, int32_t h, int32_t w,
                                               int32_t n_bins, int32_t patch_size,
                                               int32_t sample_budget, int32_t mode) {
    return reference_weights_workspace_bytes(planes, h, w, n_bins, patch_size, sample_budget,
                                             mode);
}

int qfca_reference_weights(const float* values, const void* bins, int32_t bins_bytes,
                           const float* lo, const float* hi, int64_t planes, int32_t h, int32_t w,
                           int32_t n_bins, int32_t patch_size, int32_t pad, int32_t sample_budget,
                           int32_t mode, void* workspace, int64_t workspace_bytes,
                           double* weights, void* stream) {
    return counted(launch_reference_weights(values, bins, bins_bytes, lo, hi, planes, h, w,
                                            n_bins, patch_size, pad, sample_budget, mode,
                                            workspace, workspace_bytes, weights, S(stream)),
                   mode == QFCA_REF_MEAN_QUAN ? 4 : 2);
}

int qfca_gather_tiles(const void* bins, int32_t channels, int32_t h, int32_t w,
                      const int32_t* row_starts, int32_t n_rows, const int32_t* col_starts,
                      int32_t n_cols, int32_t tile_h, int32_t tile_w, void* out, void* stream) {
    return counted(launch_gather_tiles(bins, channels, h, w, row_starts, n_rows, col_starts,
                                       n_cols, tile_h, tile_w, out, S(stream)), 1);
}

int64_t qfca_covariance_workspace_bytes(int64_t images, int32_t C, int32_t hw) {
    if (images <= 0 || C <= 0 || hw <= 0) return -1;
    return cov_i8_workspace(images, C, hw);
}

int qfca_covariance(const float* x, int64_t images, int32_t C, int32_t hw, const double* mean,
                    void* workspace, int64_t workspace_bytes, double* cov, void* stream) {
    if (!mean) return QFCA_ERR_ARG;
    return counted(launch_cov_i8(x, images, C, hw, mean, nullptr, workspace, workspace_bytes,
                                 cov, S(stream)),
                   2);
}

int qfca_mean_covariance(const float* x, int64_t images, int32_t C, int32_t hw, double* mean,
                         void* workspace, int64_t workspace_bytes, double* cov, void* stream) {
    if (!mean) return QFCA_ERR_ARG;
    return counted(launch_cov_i8(x, images, C, hw, nullptr, mean, workspace, workspace_bytes,
                                 cov, S(stream)),
                   2);
}

// ---------------------------------------------------------------- detect
struct DetectLayout {
    size_t lo, hi, bins, V, partial, used_scratch, agg, tmp, kscratch, kscratch_bytes, total;
    int groups, bins_bytes;
    ScoreChoice choice;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int detect_layout(int64_t images, int32_t C, int32_t h, int32_t w, const qfca_config* cfg,
                         DetectLayout* L) {
    if (!cfg || images <= 0 || C <= 0 || h <= 0 || w <= 0) return QFCA_ERR_ARG;
    if (cfg->n_bins < 1 || cfg->n_bins > 65536 || cfg->patch_size < 1 ||
        (cfg->patch_size & 1) == 0 || cfg->sample_budget < 1 || cfg->sigma_s < 0)
        return QFCA_ERR_ARG;
    if (cfg->pad != QFCA_PAD_REFLECT && cfg->pad != QFCA_PAD_WRAP) return QFCA_ERR_UNSUPPORTED;
    const int64_t planes = images * C, hw = (int64_t)h * w;
    L->bins_bytes = cfg->n_bins <= 256 ? 1 : 2;
    L->choice = score_choose(h, w, cfg->n_bins, cfg->patch_size, C, images, cfg->groups,
                             L->bins_bytes, cfg->pad, cfg->sample_budget, 1, 1);
    L->groups = L->choice.groups;
    if (L->groups <= 0) return QFCA_ERR_UNSUPPORTED;
    size_t off = 0;
    L->lo = off; off = align256(off + planes * 4);
    L->hi = off; off = align256(off + planes * 4);
    L->bins = off; off = align256(off + planes * hw * L->bins_bytes);
    L->V = off; off = align256(off + planes * (int64_t)cfg->n_bins * 4);
    L->partial = off; off = align256(off + images * (int64_t)L->groups * hw * 4);
    L->used_scratch = off; off = align256(off + images * 4);
    L->agg = off; off = align256(off + images * hw * 8);
    L->tmp = off; off = align256(off + images * hw * 8);
    L->kscratch_bytes = (size_t)choice_scratch_bytes(L->choice, h);
    L->kscratch = off; off = align256(off + L->kscratch_bytes);
    L->total = off;
    return QFCA_OK;
}

int64_t qfca_detect_workspace_bytes(int64_t images, int32_t channels, int32_t h, int32_t w,
                                    const qfca_config* cfg) {
    DetectLayout L;
    if (detect_layout(images, channels, h, w, cfg, &L) != QFCA_OK) return -1;
    return (int64_t)L.total;
}

static void gauss_taps(double sigma, std::vector<double>& k) {
    // features.py:49-53
    const int radius = (int)ceil(3 * sigma);
    k.resize(2 * radius + 1);
    double s = 0.0;
    for (int i = -radius; i <= radius; ++i) {
        const double x = (double)i / sigma;
        k[i + radius] = exp(-0.5 * (x * x));
        s += k[i + radius];
    }
    for (auto& v : k) v /= s;
}

int qfca_detect(const float* features, int64_t images, int32_t C, int32_t h, int32_t w,
                const qfca_config* cfg, void* workspace, int64_t workspace_bytes, double* scores,
                double* image_scores, int32_t* used, int32_t* nonfinite, void* stream) {
    return qfca_detect_ex(features, images, C, h, w, cfg, workspace, workspace_bytes, scores,
                          image_scores, used, nonfinite, nullptr, stream);
}

int qfca_detect_ex(const float* features, int64_t images, int32_t C, int32_t h, int32_t w,
                   const qfca_config* cfg, void* workspace, int64_t workspace_bytes,
                   double* scores, double* image_scores, int32_t* used, int32_t* nonfinite,
                   void* const* stage_events, void* stream) {
    DetectLayout L;
    int rc = detect_layout(images, C, h, w, cfg, &L);
    if (rc != QFCA_OK) return rc;
    if (!workspace || workspace_bytes < (int64_t)L.total || !scores || !image_scores || !used)
        return QFCA_ERR_ARG;
    cudaStream_t st = S(stream);
    uint8_t* ws = (uint8_t*)workspace;
    float* lo = (float*)(ws + L.lo);
    float* hi = (float*)(ws + L.hi);
    void* bins = ws + L.bins;
    int32_t* V = (int32_t*)(ws + L.V);
    float* partial = (float*)(ws + L.partial);
    double* agg = (double*)(ws + L.agg);
    double* tmp = (double*)(ws + L.tmp);
    const int64_t planes = images * C, hw = (int64_t)h * w;
    // K1 + K2 fused (one read of the features) when the planes fit in shared memory
    rc = launch_quantize_fused(features, planes, hw, cfg->n_bins, lo, hi, nonfinite, bins,
                               L.bins_bytes, st);
    if (rc == QFCA_OK) {
        counted(rc, 1);
    } else if (rc == QFCA_ERR_UNSUPPORTED) {
        if ((rc = counted(launch_minmax(features, planes, hw, lo, hi, nonfinite, st), 1))) return rc;
        if ((rc = counted(launch_bin(features, planes, hw, lo, hi, cfg->n_bins, bins, L.bins_bytes, st), 1)))
            return rc;
    } else {
        return rc;
    }
    if (!L.choice.fref &&  // else the scoring kernel selects the reference itself
        (rc = counted(launch_reference(bins, L.bins_bytes, lo, hi, planes, h, w, cfg->n_bins,
                                       cfg->patch_size, cfg->pad, cfg->sample_budget, 0, V, st),
                      1)))
        return rc;
    if ((rc = counted(launch_count_used(lo, hi, images, C, used, st), 1))) return rc;
    if (cudaMemsetAsync(partial, 0, images * (int64_t)L.groups * hw * 4, st) != cudaSuccess)
        return QFCA_ERR_CUDA;
    if (stage_events && stage_events[0] &&
        cudaEventRecord((cudaEvent_t)stage_events[0], st) != cudaSuccess)
        return QFCA_ERR_CUDA;
    if ((rc = counted(launch_score_any(L.choice, bins, L.bins_bytes, lo, hi, V, images, C, h, w,
                                       cfg->n_bins, cfg->patch_size, cfg->pad,
                                       cfg->sample_budget, partial, st, ws + L.kscratch,
                                       (int64_t)L.kscratch_bytes),
                      1)))
        return rc;
    if (stage_events && stage_events[1] &&
        cudaEventRecord((cudaEvent_t)stage_events[1], st) != cudaSuccess)
        return QFCA_ERR_CUDA;
    if ((rc = counted(launch_reduce_partials(partial, images, L.groups, hw, used, agg, st), 1)))
        return rc;
    double* final_map = agg;
    if (cfg->sigma_s > 0) {
        std::vector<double> k;
        gauss_taps(cfg->sigma_s, k);
        if ((int)k.size() > QFCA_MAX_TAPS) return QFCA_ERR_UNSUPPORTED;
        if ((rc = counted(launch_sep_conv(agg, images, h, w, 0, k.data(), (int)k.size(), cfg->pad, tmp,
                                  st), 1)))
            return rc;
        if ((rc = counted(launch_sep_conv(tmp, images, h, w, 1, k.data(), (int)k.size(), cfg->pad,
                                  scores, st), 1)))
            return rc;
        final_map = scores;
    } else {
        if (cudaMemcpyAsync(scores, agg, images * hw * 8, cudaMemcpyDeviceToDevice, st) !=
            cudaSuccess)
            return QFCA_ERR_CUDA;
        final_map = scores;
    }
    return counted(launch_image_score(final_map, images, h, w, cfg->border, image_scores, st), 1);
}

int qfca_pool_interior(const void* scores, int32_t scores_bytes, const uint8_t* mask,
                       int32_t images, int32_t H, int32_t W, int32_t border, double* out,
                       uint8_t* labels, float* out32, int32_t* inexact, uint64_t* image_max,
                       void* stream) {
    return counted(launch_pool_interior(scores, nullptr, scores_bytes, mask, nullptr, images, H,
                                        W, border, out, labels, out32, inexact,
                                        (unsigned long long*)image_max, S(stream)), 1);
}

int qfca_pool_interior_table(const void* const* score_images, int32_t scores_bytes,
                             const uint8_t* const* mask_images, int32_t images, int32_t H,
                             int32_t W, int32_t border, double* out, uint8_t* labels, float* out32,
                             int32_t* inexact, uint64_t* image_max, void* stream) {
    if (!score_images) return QFCA_ERR_ARG;
    return counted(launch_pool_interior(nullptr, score_images, scores_bytes, nullptr, mask_images,
                                        images, H, W, border, out, labels, out32, inexact,
                                        (unsigned long long*)image_max, S(stream)), 1);
}

int64_t qfca_rank_stats_workspace_bytes(int64_t n, int32_t key_bytes) {
    return rank_stats_workspace_bytes(n, key_bytes);
}

int qfca_rank_stats(const void* scores, int32_t key_bytes, const uint8_t* labels, int64_t n,
                    void* workspace, int64_t workspace_bytes, void* sorted_out, uint64_t* stats,
                    void* stream) {
    // radix sort (CUB onesweep passes) + 3 rank kernels
    return counted(launch_rank_stats(scores, key_bytes, labels, n, workspace, workspace_bytes,
                                     sorted_out, (unsigned long long*)stats, S(stream)), 3);
}

int64_t qfca_components_workspace_bytes(int64_t n) { return components_workspace_bytes(n); }

int qfca_components(const uint8_t* mask, int32_t images, int32_t h, int32_t w, void* workspace,
                    int64_t workspace_bytes, int32_t* labels, int32_t* comp, int32_t* n_comp,
                    void* stream) {
    return counted(launch_components(mask, images, h, w, workspace, workspace_bytes, labels, comp,
                                     n_comp, S(stream)), 4);
}

int qfca_pro_histograms(const double* scores, const int32_t* comp, int64_t n,
                        const double* thr_asc, int32_t m, int32_t comp_lo, int32_t comp_hi,
                        int32_t* comp_hist, uint64_t* normal_hist, void* stream) {
    return counted(launch_pro_histograms(scores, comp, n, thr_asc, m, comp_lo, comp_hi, comp_hist,
                                         (unsigned long long*)normal_hist, S(stream)), 1);
}

int qfca_pro_accumulate(int32_t* comp_hist, int32_t ncomp, int32_t m, double* pro, void* stream) {
    return counted(launch_pro_accumulate(comp_hist, ncomp, m, pro, S(stream)), ncomp > 0 ? 2 : 0);
}

}  // extern "C"
