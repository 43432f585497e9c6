// sf_common.cuh -- shared device helpers and internal launch interfaces.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/splatfield_b200.h"

#define SF_CUTOFF 9.0          // projection.py:33 CUTOFF_MAHAL_SQ
#define SF_LOWPASS 0.3         // projection.py:32 LOWPASS_FLOOR
#define SF_ALPHA_CLAMP 0.99    // projection.py:34 ALPHA_CLAMP
#define SF_EARLY_EXIT_T 1e-4   // rasterizer.py:45 EARLY_EXIT_T

namespace sf {

// numpy ufunc semantics (NaN-propagating) -- needed wherever the reference's
// np.minimum / np.maximum / np.clip feed an integer or membership decision.
__host__ __device__ __forceinline__ double np_minimum(double a, double b) {
    if (a != a) return a;
    if (b != b) return b;
    return (a <= b) ? a : b;
}
__host__ __device__ __forceinline__ double np_maximum(double a, double b) {
    if (a != a) return a;
    if (b != b) return b;
    return (a >= b) ? a : b;
}
__host__ __device__ __forceinline__ double np_clip(double x, double lo, double hi) {
    return np_minimum(np_maximum(x, lo), hi);
}
// numpy float64 -> int64 cast on x86-64: NaN / out of range -> INT64_MIN.
__host__ __device__ __forceinline__ int64_t np_to_i64(double v) {
    if (!(v >= -9223372036854775808.0 && v < 9223372036854775808.0)) return INT64_MIN;
    return (int64_t)v;
}
// numpy floor_divide(a, b) (npy_divmod) for the tile size.
__host__ __device__ __forceinline__ double np_floor_divide(double a, double b) {
    double mod = fmod(a, b);
    double div = (a - mod) / b;
    if (mod) {
        if ((b < 0) != (mod < 0)) {
            mod += b;
            div -= 1.0;
        }
    }
    double fl;
    if (div) {
        fl = floor(div);
        if (div - fl > 0.5) fl += 1.0;
    } else {
        fl = copysign(0.0, a / b);
    }
    return fl;
}

// min_mahalanobis_sq_to_rect, projection.py:191-226, one (mean, A, rect).
// Exact fp64 op order of the reference; callers compile with -fmad=false.
__host__ __device__ __forceinline__ double min_mahal_sq_to_rect(double mx, double my, double a,
                                                               double b, double c, double lx,
                                                               double ly, double hx, double hy) {
    double best = INFINITY;
    {
        double dx = lx - mx;
        double ys = np_clip(my - (b / c) * dx, ly, hy);
        double dy = ys - my;
        best = np_minimum(best, (a * dx) * dx + ((2.0 * b) * dx) * dy + (c * dy) * dy);
    }
    {
        double dx = hx - mx;
        double ys = np_clip(my - (b / c) * dx, ly, hy);
        double dy = ys - my;
        best = np_minimum(best, (a * dx) * dx + ((2.0 * b) * dx) * dy + (c * dy) * dy);
    }
    {
        double dy = ly - my;
        double xs = np_clip(mx - (b / a) * dy, lx, hx);
        double dx = xs - mx;
        best = np_minimum(best, (a * dx) * dx + ((2.0 * b) * dx) * dy + (c * dy) * dy);
    }
    {
        double dy = hy - my;
        double xs = np_clip(mx - (b / a) * dy, lx, hx);
        double dx = xs - mx;
        best = np_minimum(best, (a * dx) * dx + ((2.0 * b) * dx) * dy + (c * dy) * dy);
    }
    if ((mx >= lx) && (mx <= hx) && (my >= ly) && (my <= hy)) best = 0.0;
    return best;
}

// numpy floor_divide(a, 2^k) for the power-of-two tile size: a * 2^-k is
// exact (no rounding above the subnormal range), so npy_divmod's
// fmod/(a - mod)/b/floor sequence reduces to floor(a * 2^-k); a negative
// subnormal that underflows to -0 still floors to -1 as npy_divmod does.
__host__ __device__ __forceinline__ double np_floor_divide_pow2(double a, double inv_b) {
    const double q = a * inv_b;
    if (q == 0.0 && a < 0.0) return -1.0;
    return floor(q);
}

// min_mahal_sq_to_rect with the per-Gaussian quotients hoisted: the same
// IEEE operations in the same order (b / c, b / a and 2 b are computed once
// per Gaussian instead of once per rectangle), so the result is identical.
struct MahalPre {
    double mx, my, a, b, c, boc, boa, twob;
};
__host__ __device__ __forceinline__ MahalPre mahal_pre(double mx, double my, double a, double b, double c) {
    return MahalPre{mx, my, a, b, c, b / c, b / a, 2.0 * b};
}
__host__ __device__ __forceinline__ double min_mahal_sq_to_rect_pre(const MahalPre& p, double lx, double ly,
                                                                    double hx, double hy) {
    if ((p.mx >= lx) && (p.mx <= hx) && (p.my >= ly) && (p.my <= hy)) return 0.0;
    double best = INFINITY;
    {
        double dx = lx - p.mx;
        double ys = np_clip(p.my - p.boc * dx, ly, hy);
        double dy = ys - p.my;
        best = np_minimum(best, (p.a * dx) * dx + (p.twob * dx) * dy + (p.c * dy) * dy);
    }
    {
        double dx = hx - p.mx;
        double ys = np_clip(p.my - p.boc * dx, ly, hy);
        double dy = ys - p.my;
        best = np_minimum(best, (p.a * dx) * dx + (p.twob * dx) * dy + (p.c * dy) * dy);
    }
    {
        double dy = ly - p.my;
        double xs = np_clip(p.mx - p.boa * dy, lx, hx);
        double dx = xs - p.mx;
        best = np_minimum(best, (p.a * dx) * dx + (p.twob * dx) * dy + (p.c * dy) * dy);
    }
    {
        double dy = hy - p.my;
        double xs = np_clip(p.mx - p.boa * dy, lx, hx);
        double dx = xs - p.mx;
        best = np_minimum(best, (p.a * dx) * dx + (p.twob * dx) * dy + (p.c * dy) * dy);
    }
    return best;
}

// Projected record of one surviving Gaussian (fp64, the reference's values).
struct __align__(8) Proj64 {
    double mx, my;  // means2d
    double a, b, c; // inv_cov2d [[a, b], [b, c]]
};

// Per-Gaussian record in canonical (depth, id) rank order, 80 bytes:
// fp32 inputs of the blend's rejection test, then the reference's fp64
// values (means2d, inv_cov2d) used by binning and by the exact alpha.
struct __align__(16) GeomRec {
    float mx_hi, mx_lo, my_hi, my_lo;  // mean split so (px - hi) - lo is ~exact
    float a, k, d, opacity;            // q = a (dx + k dy)^2 + d dy^2, k = b/a, d = det/a
    double mx, my;                     // means2d (fp64, bitwise the reference's)
    double a64, b64;                   // inv_cov2d[0][0], inv_cov2d[0][1]
    double c64;                        // inv_cov2d[1][1]
    uint32_t row, pad;
};
// fp32 fields of a GeomRec from its fp64 ones (mean split hi + lo; the conic
// as a, k = b / a, d = det / a)
__host__ __device__ __forceinline__ void geom_fill_f32(GeomRec& q) {
    q.mx_hi = (float)q.mx;
    q.mx_lo = (float)(q.mx - (double)q.mx_hi);
    q.my_hi = (float)q.my;
    q.my_lo = (float)(q.my - (double)q.my_hi);
    q.a = (float)q.a64;
    q.k = (float)(q.b64 / q.a64);
    q.d = (float)((q.a64 * q.c64 - q.b64 * q.b64) / q.a64);
}
__host__ __device__ __forceinline__ Proj64 geom_proj(const GeomRec& g) {
    Proj64 p;
    p.mx = g.mx;
    p.my = g.my;
    p.a = g.a64;
    p.b = g.b64;
    p.c = g.c64;
    return p;
}
// Scatter plan of one Gaussian (sparse_splat.py:126-132): C u32 channel
// words = channel id (level block * L + index) x kChanWord -- the byte offset
// of the channel's row in the blend accumulator -- then, at a 16-byte
// boundary, C f32 values; both parts padded to 16 bytes (C = 12 -> 96 B).
constexpr uint32_t kChanWord = 129 * 4;  // blend accumulator pitch (floats) x 4 bytes
__host__ __device__ __forceinline__ int chan_val_offset(int C) { return (4 * C + 15) / 16 * 16; }
__host__ __device__ __forceinline__ int chan_rec_bytes(int C) { return 2 * chan_val_offset(C); }
__host__ __device__ __forceinline__ int chan_id(uint32_t word) { return (int)(word / kChanWord); }

// Workspace carving helper.
struct Carver {
    char* base;
    size_t off, cap;
    __host__ Carver(void* p, size_t c) : base((char*)p), off(0), cap(c) {}
    template <typename T>
    __host__ T* take(size_t n) {
        off = (off + 255) & ~(size_t)255;
        T* p = (T*)(base ? base + off : nullptr);
        off += n * sizeof(T);
        return p;
    }
    __host__ bool ok() const { return off <= cap; }
};

__host__ __device__ __forceinline__ int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Selected semantic levels, passed by value (no host->device copy).
constexpr int kMaxLevels = 8;
struct LevelSelDev {
    int n;
    int lv[kMaxLevels];
};

// sf_runtime.cu: per-(kernel, device) dynamic shared-memory limit (thread-safe),
// and the current device's SM count (persistent grids)
int ensure_smem_attr(const void* func, size_t bytes);
// message for sf_last_error (sf_capi.cu)
void set_error(const char* fmt, ...);
int device_sm_count();
// a side stream and fork / join events bound to (device, primary stream), for
// independent kernels of one launcher to run concurrently; nullptr -> serial
struct SideStream {
    cudaStream_t s;
    cudaEvent_t fork, join;
};
SideStream* side_stream(cudaStream_t primary);

// ---------------- internal launchers (one .cu each) ----------------

// sf_preprocess.cu
void launch_preprocess(const SfScene& s, const SfCamera& cam, GeomRec* geom, uint64_t* keys,
                       uint32_t* vals, int64_t* stats, cudaStream_t st);
void launch_project_compact(const SfScene& s, const GeomRec* geom, const uint64_t* keys,
                            const int64_t* orig_rows_or_null, int32_t* flags, int32_t* scan,
                            double* means2d, double* inv_covs, double* depths, double* opac,
                            int64_t* source_ids, int64_t* rows, int64_t* count, void* cub_tmp,
                            size_t cub_bytes, cudaStream_t st);
size_t project_compact_cub_bytes(int64_t G);

// sf_binning.cu
// sf_sort.cu: stable LSD radix sort of (u64 key, u32 value); the inputs are scratch
size_t depth_sort_tmp_bytes(int64_t n);
int depth_sort(uint64_t* keys_in, uint64_t* keys_out, uint32_t* vals_in, uint32_t* vals_out, int64_t n, void* tmp,
               size_t tmp_bytes, cudaStream_t st);
// per-row scatter plan (channel ids + values) of the selected levels
void launch_pack_channels(const SfScene& s, const LevelSelDev& levels, unsigned char* chan, cudaStream_t st);
// Frame-mode tile entries leave the emit pass as row | half-tile flags << 30
// (bit 30: the top 16x8 half may see the Gaussian, bit 31: the bottom half);
// the per-tile sort moves the flags to a byte array parallel to the entries,
// so every consumer of the sorted lists reads plain rows.
constexpr int kEntryFlagShift = 30;
constexpr uint32_t kEntryRowMask = (1u << kEntryFlagShift) - 1u;
// Binning over n_items geometry records.  row_keys == null (sf_bin): record
// i has canonical rank i (i < stats[VISIBLE]) and the lists hold ranks.
// row_keys != null (frame): record i is scene row i, culled iff row_keys[i]
// == ~0, and each list's rows are sorted by (row_keys[row], row).
// tile_counts holds 2 * n_tiles counters; aux one BinAux per item.
constexpr int kBinSlots = 8;
struct __align__(16) BinAux {
    unsigned long long mask;     // hits over the candidate rectangle, row-major (<= 64 tiles)
    uint16_t tx0, ty0, w, h;     // candidate rectangle
    uint32_t pos[kBinSlots];     // in-tile position of the first kBinSlots hits
};
void launch_binning(int64_t n_items, const int64_t* stats, const GeomRec* geom, const uint64_t* row_keys,
                    uint8_t* entry_flags, int W, int H, int64_t pair_capacity, uint32_t* tile_counts,
                    uint32_t* tile_offsets, uint32_t* tile_cursor, uint32_t* entries, uint32_t* sort_scratch,
                    BinAux* aux, uint32_t* cta_base, int tile_row0, int tile_row1, cudaStream_t st);
// per-(count CTA, tile) range bases of the aggregated count pass
size_t bin_cta_base_elems(int W, int H);

// sf_blend.cu
struct BlendArgs {
    int W, H, tiles_x, tiles_y;
    int tile0, n_band_tiles;  // tiles [tile0, tile0 + n_band_tiles) are blended (whole tile rows)
    int n_ch;          // n_levels * L
    int C;             // channels per Gaussian = n_levels * K
    int early_exit;
    const uint32_t* tile_offsets;
    const uint32_t* entries;
    const uint8_t* entry_flags;  // frame lists: half-tile flags per entry (launch_binning), or null
    const GeomRec* geom;
    const unsigned char* chan;
    const int64_t* stats;  // overflow flag gate
    uint32_t* fixup_list;  // (tile << 8 | pixel slot) of pixels whose early-exit decision is ambiguous
    uint32_t* fixup_count;
    uint32_t fixup_capacity;
    uint32_t* sched;       // [0]: next half tile to claim (tensor-core splat), zeroed per frame
    float* fixup_w;        // exact coefficients of the replayed pixels (fused decode), or null
    uint32_t fixup_w_capacity;
    float* coeff_map;      // (H,W,n_ch) or null
    float* final_t;        // (H,W) or null
    // fused projected-codebook relevancy (optional)
    const double* proj_cb; // (n_levels, L, 1 + n_canon) or null
    int n_levels, L, n_canon;
    double* relevancy_raw; // (n_levels, H, W)
    int64_t* fixups;
    // fused decode (optional): features (n_levels, H, W, D) from the blended tile
    float* features;
    int D;
    int64_t feat_level_stride;  // H * W * D
    const void* dec_b;          // k_dec_codebook_image output (blend_dec_image_bytes)
    const float* dec_scale;     // per-level output scale (inside that image)
    const float* codebooks;     // scene codebooks (levels, L, D): exact fp64 decode of fixup pixels
    LevelSelDev lv;
    uint64_t* timeline;         // development aid (SF_BLEND_TIMELINE), normally null
};
int launch_blend(const BlendArgs& a, cudaStream_t st);
// transpose of the splat (training backward): ghat (levels, G, K) += e * dW gathers
int launch_splat_transpose(const BlendArgs& a, const float* dW, float* ghat, int K, int64_t G, cudaStream_t st);
// fused decode: supported shape, and the bytes of its codebook image
bool blend_dec_supported(int n_levels, int L, int K, int D);
size_t blend_dec_image_bytes(int n_levels, int D);
void launch_dec_codebook_image(const float* codebooks, const LevelSelDev& lv, int L, int D, void* out,
                               cudaStream_t st);
// relevancy of every pixel/level from a coefficient map already in HBM
void launch_relevancy_from_cmap(int64_t P, int n_ch, const float* cmap, const double* proj_cb,
                                int n_levels, int L, int n_canon, double* out, int64_t out_level_stride,
                                cudaStream_t st);

// many prompts over one map: proj (n_levels, L, nq + n_canon) from
// launch_project_vectors; out (nq, n_levels, P) (prompt-major).  Returns
// nonzero when the shape is unsupported (n_canon > 8, L % 4, n_ch % 4).
int launch_relevancy_sweep(int64_t P, int n_ch, const float* cmap, const double* proj, int n_levels, int L,
                           int nq, int n_canon, double* out, int64_t out_prompt_stride, int64_t out_level_stride,
                           cudaStream_t st);

// sf_post.cu
void launch_project_codebook(const float* codebooks, const LevelSelDev& levels, int L, int D,
                             const double* q, const double* canon, int n_canon, double* out,
                             cudaStream_t st);
// columns q[0..nq) then canon[0..n_canon): out (levels, L, nq + n_canon)
void launch_project_vectors(const float* codebooks, const LevelSelDev& levels, int L, int D, const double* q,
                            int nq, const double* canon, int n_canon, double* out, cudaStream_t st);
size_t filter_select_batch_ws_bytes(int n_queries, int n_maps, int H, int W);
void launch_filter_select_batch(int n_queries, int n_maps, int H, int W, const double* raw, int window,
                                double* filtered, double threshold, uint8_t* masks, int64_t* stats_i64,
                                double* stats_f64, void* ws, cudaStream_t st, int y0 = 0, int y1 = 0);
void launch_relevancy_f32(int64_t P, int D, const float* f, const double* q, const double* c,
                          int nc, double* out, cudaStream_t st);
void launch_relevancy_f64(int64_t P, int D, const double* f, const double* q, const double* c,
                          int nc, double* out, cudaStream_t st);
// [y0, y1): output / reduced rows (band mode); y1 <= y0 = all rows
void launch_mean_filter(int n_maps, int H, int W, const double* in, int window, double* tmp,
                        double* out, cudaStream_t st, int y0 = 0, int y1 = 0);
size_t select_segment_ws_bytes(int n_maps, int H, int W);
void launch_select_segment(int n_maps, int H, int W, const double* maps, int fixed_level,
                           double threshold, uint8_t* mask, int64_t* stats_i64,
                           double* stats_f64, void* ws, cudaStream_t st, int y0 = 0, int y1 = 0);
// fused mean filter + selection statistics + mask (window / 2 <= 8)
bool filter_select_fusable(int window);
void launch_filter_select(int n_maps, int H, int W, const double* raw, int window, double* filtered,
                          int fixed_level, double threshold, uint8_t* mask, int64_t* stats_i64,
                          double* stats_f64, void* ws, cudaStream_t st, int y0 = 0, int y1 = 0);
void launch_mask_rows(int H, int W, const double* maps, int level, double lo, double hi, double threshold,
                      int y0, int y1, uint8_t* mask, cudaStream_t st);

// sf_io.cu
void launch_lsv2_unpack(const uint8_t* rec, int64_t G, int levels, int K, int L, float* pos, float* rot,
                        float* scl, float* opa, float* col, uint16_t* cidx, float* cval, uint32_t* flags,
                        cudaStream_t st);

// sf_decode.cu (SIMT cross-check) / sf_decode_tc.cu (tcgen05 3xTF32)
int launch_decode_simt(int64_t P, int L, int D, const float* w, int64_t w_stride, const float* cb,
                       float* out, cudaStream_t st);
size_t decode_ws_bytes(int L, int D);
int launch_decode(int64_t P, int L, int D, const float* w, int64_t w_stride, const float* cb,
                  float* out, void* ws, cudaStream_t st);

}  // namespace sf
