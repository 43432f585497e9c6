// sf_post.cu -- K8-K10: relevancy, mean filter, level selection, argmax, mask.
//
// Reference: relevancy_map (query.py:65-84, raw dot products, two-branch
// sigmoid), mean_filter (query.py:87-108, edge-clamped box filter),
// select_level (:111-118, first argmax of maxima), localize (:121-126, first
// row-major argmax), segment (:136-145, min-max normalised > threshold).
// All fp64: the outputs feed discontinuous decisions (level, point, mask).
#include <cub/cub.cuh>

#include "sf_common.cuh"

namespace sf {

// two-branch logistic (query.py:65-84), evaluated branch-free: both branches
// take exp(-|x|), so a warp with mixed signs runs one exp instead of two
__device__ __forceinline__ double sigmoid2p(double x) {
    const double e = exp(-fabs(x));
    return (x >= 0 ? 1.0 : e) / (1.0 + e);
}

// P[b][l][j] = atoms_{lv_b}[l] . v_j, v_j = q[j] for j < nq, else canonical
// j - nq (fp64).  One warp per (b, l, j) dot product of length D, shuffle-reduced.
__global__ void __launch_bounds__(256) k_project_codebook(const float* __restrict__ cb, LevelSelDev lv, int L, int D,
                                                          const double* __restrict__ q, int nq,
                                                          const double* __restrict__ canon, int n_canon,
                                                          double* __restrict__ out) {
    const int nv = nq + n_canon;
    const int lane = threadIdx.x & 31;
    const int idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int total = lv.n * L * nv;
    if (idx >= total) return;
    const int j = idx % nv;
    const int l = (idx / nv) % L;
    const int b = idx / (nv * L);
    const float* a = cb + ((size_t)lv.lv[b] * L + l) * D;
    const double* v = (j < nq) ? q + (size_t)j * D : canon + (size_t)(j - nq) * D;
    double s = 0.0;
    for (int d = lane; d < D; d += 32) s = fma((double)a[d], v[d], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[idx] = s;
}

void launch_project_codebook(const float* codebooks, const LevelSelDev& lv, int L, int D,
                             const double* q, const double* canon, int n_canon, double* out,
                             cudaStream_t st) {
    launch_project_vectors(codebooks, lv, L, D, q, 1, canon, n_canon, out, st);
}

void launch_project_vectors(const float* codebooks, const LevelSelDev& lv, int L, int D, const double* q, int nq,
                            const double* canon, int n_canon, double* out, cudaStream_t st) {
    int total = lv.n * L * (nq + n_canon);
    k_project_codebook<<<ceil_div((int64_t)total * 32, 256), 256, 0, st>>>(codebooks, lv, L, D, q, nq, canon,
                                                                          n_canon, out);
}

template <typename T>
__global__ void k_relevancy(int64_t P, int D, const T* __restrict__ f, const double* __restrict__ q,
                            const double* __restrict__ c, int nc, double* __restrict__ out) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const T* fp = f + (size_t)p * D;
    double lq = 0.0;
    for (int d = 0; d < D; ++d) lq = fma((double)fp[d], q[d], lq);
    double best = INFINITY;
    for (int j = 0; j < nc; ++j) {
        double lc = 0.0;
        const double* cj = c + (size_t)j * D;
        for (int d = 0; d < D; ++d) lc = fma((double)fp[d], cj[d], lc);
        best = np_minimum(best, sigmoid2p(lq - lc));
    }
    out[p] = best;
}

void launch_relevancy_f32(int64_t P, int D, const float* f, const double* q, const double* c,
                          int nc, double* out, cudaStream_t st) {
    if (P) k_relevancy<float><<<ceil_div(P, 128), 128, 0, st>>>(P, D, f, q, c, nc, out);
}
void launch_relevancy_f64(int64_t P, int D, const double* f, const double* q, const double* c,
                          int nc, double* out, cudaStream_t st) {
    if (P) k_relevancy<double><<<ceil_div(P, 128), 128, 0, st>>>(P, D, f, q, c, nc, out);
}

// Separable edge-clamped box filter.  Pass 1 sums rows, pass 2 columns.
// Output rows [y0, y1) (band mode); pass 1 covers the rows pass 2 reads.
__global__ void k_box_rows(int n_maps, int H, int W, const double* __restrict__ in, int r,
                           double* __restrict__ out, int ry0, int nrows) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)n_maps * nrows * W;
    if (i >= total) return;
    const int64_t per = (int64_t)nrows * W;
    const int64_t m = i / per;
    i = m * (int64_t)H * W + (int64_t)ry0 * W + (i - m * per);  // index in the (n_maps, H, W) arrays
    int x = (int)(i % W);
    const double* row = in + (i - x);
    double s = 0.0;
    for (int d = -r; d <= r; ++d) {
        int xx = min(max(x + d, 0), W - 1);
        s += row[xx];
    }
    out[i] = s;
}
__global__ void k_box_cols(int n_maps, int H, int W, const double* __restrict__ in, int r,
                           double inv_area, double* __restrict__ out, int y0, int nrows) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)n_maps * nrows * W;
    if (i >= total) return;
    const int64_t per = (int64_t)nrows * W;
    const int64_t mm = i / per;
    i = mm * (int64_t)H * W + (int64_t)y0 * W + (i - mm * per);
    int64_t hw = (int64_t)H * W;
    int64_t m = i / hw;
    int64_t rem = i - m * hw;
    int y = (int)(rem / W), x = (int)(rem % W);
    const double* base = in + m * hw;
    double s = 0.0;
    for (int d = -r; d <= r; ++d) {
        int yy = min(max(y + d, 0), H - 1);
        s += base[(int64_t)yy * W + x];
    }
    out[i] = s / inv_area;
}

void launch_mean_filter(int n_maps, int H, int W, const double* in, int window, double* tmp,
                        double* out, cudaStream_t st, int y0, int y1) {
    if (y1 <= y0) y0 = 0, y1 = H;
    int64_t total = (int64_t)n_maps * (y1 - y0) * W;
    if (total == 0) return;
    if (window == 1) {
        for (int m = 0; m < n_maps; ++m)
            cudaMemcpyAsync(out + ((size_t)m * H + y0) * W, in + ((size_t)m * H + y0) * W,
                            (size_t)(y1 - y0) * W * sizeof(double), cudaMemcpyDeviceToDevice, st);
        return;
    }
    int r = window / 2;
    const int ry0 = max(0, y0 - r), ry1 = min(H, y1 + r);
    const int64_t total_rows = (int64_t)n_maps * (ry1 - ry0) * W;
    k_box_rows<<<ceil_div(total_rows, 256), 256, 0, st>>>(n_maps, H, W, in, r, tmp, ry0, ry1 - ry0);
    k_box_cols<<<ceil_div(total, 256), 256, 0, st>>>(n_maps, H, W, tmp, r, (double)window * (double)window, out,
                                                     y0, y1 - y0);
}

// ---- select_level / localize / segment ----

struct MaxMin {
    double mx;
    int64_t idx;  // first index of the maximum
    double mn;
};

__device__ __forceinline__ MaxMin mm_combine(MaxMin a, MaxMin b) {
    MaxMin r;
    if (b.mx > a.mx || (b.mx == a.mx && b.idx < a.idx)) {
        r.mx = b.mx;
        r.idx = b.idx;
    } else {
        r.mx = a.mx;
        r.idx = a.idx;
    }
    r.mn = fmin(a.mn, b.mn);
    return r;
}

constexpr int kRedBlocks = 296;  // 2 x 148 SMs

__global__ void __launch_bounds__(256) k_reduce_maps(int64_t hw, const double* __restrict__ maps,
                                                     MaxMin* __restrict__ partial, int64_t i0, int64_t i1) {
    int m = blockIdx.y;
    const double* p = maps + (size_t)m * hw;
    MaxMin acc{-INFINITY, INT64_MAX, INFINITY};
    for (int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < i1;
         i += (int64_t)gridDim.x * blockDim.x) {
        double v = p[i];
        MaxMin x{v, i, v};
        acc = mm_combine(acc, x);
    }
    typedef cub::BlockReduce<MaxMin, 256> Red;
    __shared__ typename Red::TempStorage tmp;
    struct Op {
        __device__ MaxMin operator()(const MaxMin& a, const MaxMin& b) const { return mm_combine(a, b); }
    };
    MaxMin r = Red(tmp).Reduce(acc, Op());
    if (threadIdx.x == 0) partial[(size_t)m * gridDim.x + blockIdx.x] = r;
}

// One warp per map reduces the per-block partials; thread 0 then selects.
__global__ void k_finalize_select(int n_maps, int nblk, int W, const MaxMin* __restrict__ partial,
                                  int fixed_level, int64_t* stats_i64, double* stats_f64) {
    __shared__ MaxMin per_map[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < n_maps) {
        MaxMin acc{-INFINITY, INT64_MAX, INFINITY};
        for (int b = lane; b < nblk; b += 32) acc = mm_combine(acc, partial[(size_t)warp * nblk + b]);
        for (int o = 16; o > 0; o >>= 1) {
            MaxMin other;
            other.mx = __shfl_xor_sync(0xffffffffu, acc.mx, o);
            other.idx = __shfl_xor_sync(0xffffffffu, acc.idx, o);
            other.mn = __shfl_xor_sync(0xffffffffu, acc.mn, o);
            acc = mm_combine(acc, other);
        }
        if (lane == 0) per_map[warp] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int lvl = fixed_level;
        if (lvl < 0) {
            lvl = 0;
            for (int m = 1; m < n_maps; ++m)
                if (per_map[m].mx > per_map[lvl].mx) lvl = m;  // ties -> lowest level
        }
        MaxMin c = per_map[lvl];
        stats_i64[SF_STAT_LEVEL] = lvl;
        stats_i64[SF_STAT_ROW] = c.idx / W;
        stats_i64[SF_STAT_COL] = c.idx % W;
        stats_i64[SF_STAT_DEGENERATE] = (c.mx <= c.mn) ? 1 : 0;
        stats_f64[SF_STATF_MIN] = c.mn;
        stats_f64[SF_STATF_MAX] = c.mx;
        for (int m = 0; m < n_maps; ++m) {
            stats_f64[SF_STATF_LEVEL_MAX + m] = per_map[m].mx;
            stats_f64[SF_STATF_LEVEL_MAX + n_maps + m] = per_map[m].mn;
            stats_i64[SF_STAT_LEVEL_ARGMAX + m] = per_map[m].idx;
        }
    }
}

// blockIdx.y: query of a batch (maps / statistics / mask of query y at
// y * (n_maps hw, 16, 8 + 2 n_maps, hw)).
// V pixels per thread (V = 4: two 16-byte map loads, one 4-byte mask store;
// the launcher uses it when hw, i0 and i1 are multiples of 4).
template <int V>
__global__ void k_mask(int64_t hw, const double* __restrict__ maps, const int64_t* __restrict__ stats_i64,
                       const double* __restrict__ stats_f64, double threshold, uint8_t* __restrict__ mask,
                       int64_t i0, int64_t i1, int n_maps = 0) {
    const int64_t i = i0 + V * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= i1) return;
    maps += (size_t)blockIdx.y * n_maps * hw;
    stats_i64 += (size_t)blockIdx.y * 16;
    stats_f64 += (size_t)blockIdx.y * (8 + 2 * n_maps);
    mask += (size_t)blockIdx.y * hw;
    const int lvl = (int)stats_i64[SF_STAT_LEVEL];
    const double lo = stats_f64[SF_STATF_MIN], hi = stats_f64[SF_STATF_MAX];
    const double* m = maps + (size_t)lvl * hw + i;
    if (V == 4) {
        const double2 a = reinterpret_cast<const double2*>(m)[0], b = reinterpret_cast<const double2*>(m)[1];
        const double x[4] = {a.x, a.y, b.x, b.y};
        uint32_t packed = 0;
        if (!(hi <= lo)) {
#pragma unroll
            for (int k = 0; k < 4; ++k) packed |= (uint32_t)(((x[k] - lo) / (hi - lo)) > threshold) << (8 * k);
        }
        *reinterpret_cast<uint32_t*>(mask + i) = packed;
    } else {
        uint8_t v = 0;
        if (!(hi <= lo)) v = ((m[0] - lo) / (hi - lo)) > threshold;
        mask[i] = v;
    }
}

static void launch_mask(int64_t hw, const double* maps, const int64_t* stats_i64, const double* stats_f64,
                        double threshold, uint8_t* mask, int64_t i0, int64_t i1, int n_queries, int n_maps,
                        cudaStream_t st) {
    const bool vec = hw % 4 == 0 && i0 % 4 == 0 && i1 % 4 == 0 && ((uintptr_t)maps & 15) == 0 &&
                     ((uintptr_t)mask & 3) == 0;
    if (vec)
        k_mask<4><<<dim3(ceil_div((i1 - i0) / 4, 256), n_queries), 256, 0, st>>>(hw, maps, stats_i64, stats_f64,
                                                                                  threshold, mask, i0, i1, n_maps);
    else
        k_mask<1><<<dim3(ceil_div(i1 - i0, 256), n_queries), 256, 0, st>>>(hw, maps, stats_i64, stats_f64, threshold,
                                                                           mask, i0, i1, n_maps);
}

__global__ void k_mask_rows(int64_t hw, const double* __restrict__ maps, int level, double lo, double hi,
                            double threshold, uint8_t* __restrict__ mask, int64_t i0, int64_t i1) {
    int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= i1) return;
    uint8_t v = 0;
    if (!(hi <= lo)) v = ((maps[(size_t)level * hw + i] - lo) / (hi - lo)) > threshold;
    mask[i] = v;
}

void launch_mask_rows(int H, int W, const double* maps, int level, double lo, double hi, double threshold,
                      int y0, int y1, uint8_t* mask, cudaStream_t st) {
    const int64_t hw = (int64_t)H * W, i0 = (int64_t)y0 * W, i1 = (int64_t)y1 * W;
    if (i1 > i0) k_mask_rows<<<ceil_div(i1 - i0, 256), 256, 0, st>>>(hw, maps, level, lo, hi, threshold, mask, i0, i1);
}

// Fused mean filter + selection statistics: one CTA per 64 x 16 output tile
// of one map.  The edge-clamped input tile (+ r halo) is staged in shared
// memory; row sums then column sums are taken in exactly k_box_rows /
// k_box_cols's order (bitwise the same filtered values), and the CTA's
// max / first argmax / min over its owned pixels go to the partials that
// k_finalize_select reduces -- the filtered maps are written once, never
// re-read for the statistics.
// k_finalize_select for many partials: the whole CTA reduces one map at a time
__global__ void __launch_bounds__(1024) k_finalize_select_wide(int n_maps, int nblk, int W,
                                                               const MaxMin* __restrict__ partial, int fixed_level,
                                                               int64_t* stats_i64, double* stats_f64) {
    typedef cub::BlockReduce<MaxMin, 1024> Red;
    __shared__ typename Red::TempStorage tmp;
    __shared__ MaxMin per_map[kMaxLevels];
    // blockIdx.x: query of a batch
    partial += (size_t)blockIdx.x * n_maps * nblk;
    stats_i64 += (size_t)blockIdx.x * 16;
    stats_f64 += (size_t)blockIdx.x * (8 + 2 * n_maps);
    struct Op {
        __device__ MaxMin operator()(const MaxMin& a, const MaxMin& b) const { return mm_combine(a, b); }
    };
    for (int m = 0; m < n_maps; ++m) {
        MaxMin acc{-INFINITY, INT64_MAX, INFINITY};
        for (int b = threadIdx.x; b < nblk; b += blockDim.x) acc = mm_combine(acc, partial[(size_t)m * nblk + b]);
        const MaxMin r = Red(tmp).Reduce(acc, Op());
        if (threadIdx.x == 0) per_map[m] = r;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        int lvl = fixed_level;
        if (lvl < 0) {
            lvl = 0;
            for (int m = 1; m < n_maps; ++m)
                if (per_map[m].mx > per_map[lvl].mx) lvl = m;  // ties -> lowest level
        }
        const MaxMin c = per_map[lvl];
        stats_i64[SF_STAT_LEVEL] = lvl;
        stats_i64[SF_STAT_ROW] = c.idx / W;
        stats_i64[SF_STAT_COL] = c.idx % W;
        stats_i64[SF_STAT_DEGENERATE] = (c.mx <= c.mn) ? 1 : 0;
        stats_f64[SF_STATF_MIN] = c.mn;
        stats_f64[SF_STATF_MAX] = c.mx;
        for (int m = 0; m < n_maps; ++m) {
            stats_f64[SF_STATF_LEVEL_MAX + m] = per_map[m].mx;
            stats_f64[SF_STATF_LEVEL_MAX + n_maps + m] = per_map[m].mn;
            stats_i64[SF_STAT_LEVEL_ARGMAX + m] = per_map[m].idx;
        }
    }
}

constexpr int kBoxTX = 64, kBoxTY = 16, kBoxRMax = 8;
// RC > 0: the radius as a compile-time constant (unrolled sums, constant
// divisors); RC = 0 takes it from r.  Same summation order either way.
template <int RC>
__global__ void __launch_bounds__(256) k_box2d_stats(int H, int W, const double* __restrict__ in, int r_rt,
                                                     double area, double* __restrict__ out,
                                                     MaxMin* __restrict__ partial, int y0, int y1) {
    // a fixed radius sizes the halo exactly, which leaves room for 32-row tiles
    constexpr int TY = RC > 0 ? 2 * kBoxTY : kBoxTY, RR = RC > 0 ? RC : kBoxRMax;
    __shared__ double tin[TY + 2 * RR][kBoxTX + 2 * RR];
    __shared__ double trs[TY + 2 * RR][kBoxTX];
    const int r = RC > 0 ? RC : r_rt;
    const int m = blockIdx.z;
    const int x0 = blockIdx.x * kBoxTX, ty0 = y0 + blockIdx.y * TY;
    const int64_t hw = (int64_t)H * W;
    const double* src = in + (size_t)m * hw;
    const int nr = TY + 2 * r, nc = kBoxTX + 2 * r;
    for (int i = threadIdx.x; i < nr * nc; i += blockDim.x) {
        const int rr = i / nc, cc = i - rr * nc;
        const int yy = min(max(ty0 - r + rr, 0), H - 1), xx = min(max(x0 - r + cc, 0), W - 1);
        tin[rr][cc] = src[(int64_t)yy * W + xx];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * kBoxTX; i += blockDim.x) {
        const int rr = i / kBoxTX, x = i - rr * kBoxTX;
        double acc = 0.0;
        if (RC > 0) {
#pragma unroll
            for (int d = -RC; d <= RC; ++d) acc += tin[rr][x + RC + d];
        } else {
            for (int d = -r; d <= r; ++d) acc += tin[rr][x + r + d];
        }
        trs[rr][x] = acc;
    }
    __syncthreads();
    MaxMin best{-INFINITY, INT64_MAX, INFINITY};
    for (int i = threadIdx.x; i < TY * kBoxTX; i += blockDim.x) {
        const int yl = i / kBoxTX, x = i - yl * kBoxTX;
        const int y = ty0 + yl, gx = x0 + x;
        if (y >= y1 || gx >= W) continue;
        double acc = 0.0;
        if (RC > 0) {
#pragma unroll
            for (int d = -RC; d <= RC; ++d) acc += trs[yl + RC + d][x];
        } else {
            for (int d = -r; d <= r; ++d) acc += trs[yl + r + d][x];
        }
        const double v = acc / area;
        const int64_t idx = (int64_t)y * W + gx;
        out[(size_t)m * hw + idx] = v;
        best = mm_combine(best, MaxMin{v, idx, v});
    }
    typedef cub::BlockReduce<MaxMin, 256> Red;
    __shared__ typename Red::TempStorage tmp;
    struct Op {
        __device__ MaxMin operator()(const MaxMin& a, const MaxMin& b) const { return mm_combine(a, b); }
    };
    const MaxMin rsum = Red(tmp).Reduce(best, Op());
    if (threadIdx.x == 0)
        partial[(size_t)m * gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = rsum;
}

// returns the number of partials per map (the grid's x * y)
static int launch_box2d_stats(int n_maps, int H, int W, const double* in, int r, double* out, MaxMin* partial,
                              int y0, int y1, cudaStream_t st) {
    const double area = (double)(2 * r + 1) * (double)(2 * r + 1);
    const int ty = r == 5 ? 2 * kBoxTY : kBoxTY;
    dim3 grid(ceil_div(W, kBoxTX), ceil_div(y1 - y0, ty), n_maps);
    if (r == 5)
        k_box2d_stats<5><<<grid, 256, 0, st>>>(H, W, in, r, area, out, partial, y0, y1);
    else
        k_box2d_stats<0><<<grid, 256, 0, st>>>(H, W, in, r, area, out, partial, y0, y1);
    return (int)(grid.x * grid.y);
}

static int box_tiles(int H, int W) { return ceil_div(W, kBoxTX) * ceil_div(H, kBoxTY); }

size_t select_segment_ws_bytes(int n_maps, int H, int W) {
    const size_t nblk = (size_t)(box_tiles(H, W) > kRedBlocks ? box_tiles(H, W) : kRedBlocks);
    return sizeof(MaxMin) * nblk * (size_t)n_maps + 256;
}

bool filter_select_fusable(int window) { return window > 1 && window / 2 <= kBoxRMax; }

void launch_filter_select(int n_maps, int H, int W, const double* raw, int window, double* filtered,
                          int fixed_level, double threshold, uint8_t* mask, int64_t* stats_i64,
                          double* stats_f64, void* ws, cudaStream_t st, int y0, int y1) {
    if (y1 <= y0) y0 = 0, y1 = H;
    if (y1 <= y0 || W == 0) return;
    const int r = window / 2;
    MaxMin* partial = (MaxMin*)ws;
    const int nblk = launch_box2d_stats(n_maps, H, W, raw, r, filtered, partial, y0, y1, st);
    k_finalize_select_wide<<<1, 1024, 0, st>>>(n_maps, nblk, W, partial, fixed_level, stats_i64, stats_f64);
    const int64_t hw = (int64_t)H * W, i0 = (int64_t)y0 * W, i1 = (int64_t)y1 * W;
    if (mask && i1 > i0)
        launch_mask(hw, filtered, stats_i64, stats_f64, threshold, mask, i0, i1, 1, 0, st);
}

// n_queries filter + select + mask passes in three launches: raw / filtered
// (n_queries, n_maps, H, W), masks (n_queries, H, W), statistics
// (n_queries, 16) / (n_queries, 8 + 2 n_maps); ws holds
// filter_select_batch_ws_bytes.  Whole images, automatic level.
size_t filter_select_batch_ws_bytes(int n_queries, int n_maps, int H, int W) {
    return sizeof(MaxMin) * (size_t)box_tiles(H, W) * n_maps * n_queries + 256;
}

void launch_filter_select_batch(int n_queries, int n_maps, int H, int W, const double* raw, int window,
                                double* filtered, double threshold, uint8_t* masks, int64_t* stats_i64,
                                double* stats_f64, void* ws, cudaStream_t st, int y0, int y1) {
    if (y1 <= y0) y0 = 0, y1 = H;
    if (n_queries == 0 || W == 0 || y1 <= y0) return;
    const int r = window / 2;
    MaxMin* partial = (MaxMin*)ws;
    const int nblk = launch_box2d_stats(n_maps * n_queries, H, W, raw, r, filtered, partial, y0, y1, st);
    k_finalize_select_wide<<<n_queries, 1024, 0, st>>>(n_maps, nblk, W, partial, -1, stats_i64, stats_f64);
    const int64_t hw = (int64_t)H * W;
    if (masks)
        launch_mask(hw, filtered, stats_i64, stats_f64, threshold, masks, (int64_t)y0 * W, (int64_t)y1 * W, n_queries,
                    n_maps, st);
}

void launch_select_segment(int n_maps, int H, int W, const double* maps, int fixed_level,
                           double threshold, uint8_t* mask, int64_t* stats_i64, double* stats_f64,
                           void* ws, cudaStream_t st, int y0, int y1) {
    int64_t hw = (int64_t)H * W;
    if (y1 <= y0) y0 = 0, y1 = H;
    const int64_t i0 = (int64_t)y0 * W, i1 = (int64_t)y1 * W;
    MaxMin* partial = (MaxMin*)ws;
    k_reduce_maps<<<dim3(kRedBlocks, n_maps), 256, 0, st>>>(hw, maps, partial, i0, i1);
    k_finalize_select<<<1, 32 * n_maps, 0, st>>>(n_maps, kRedBlocks, W, partial, fixed_level, stats_i64,
                                                  stats_f64);
    if (mask && i1 > i0)
        launch_mask(hw, maps, stats_i64, stats_f64, threshold, mask, i0, i1, 1, 0, st);
}

}  // namespace sf
