/*
 * splat_oracle.c -- CPU restatement of the splatfield hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the sm_100a
 * product path and the "port" CPU baseline timed by bench.py.  Nothing under
 * paper_2507_07136_b200/ links, loads or calls it; only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline leg / --impl reference)
 * may.
 *
 * Every function restates one function of the reference package
 * (/root/reference/pkg/src/splatfield, cited file:line) with the same
 * floating-point operation order.  Where the reference multiplies small
 * matrices through numpy -> OpenBLAS dgemm/dsyrk, the BLAS kernel evaluates a
 * K=3 dot product as the FMA chain fma(a2,b2, fma(a1,b1, a0*b0)); those sites
 * use fma() explicitly and nothing else may contract (compile with
 * -ffp-contract=off).  The restatement is pinned bitwise against the imported
 * reference by oracle/gen_golden.py + tests/test_oracle_golden.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_LOWPASS 0.3      /* projection.py:32 */
#define OR_CUTOFF 9.0       /* projection.py:33 */
#define OR_ALPHA_CLAMP 0.99 /* projection.py:34 */
#define OR_EARLY_EXIT 1e-4  /* rasterizer.py:45 */

typedef struct {
    double R[9]; /* world->camera rotation, row-major */
    double t[3];
    double fx, fy, cx, cy, near_;
    int64_t width, height;
} OrCamera;

/* numpy's NaN-propagating minimum / maximum / clip (ufunc semantics). */
static inline double np_minimum(double a, double b) {
    if (a != a) return a;
    if (b != b) return b;
    return (a <= b) ? a : b;
}
static inline double np_maximum(double a, double b) {
    if (a != a) return a;
    if (b != b) return b;
    return (a >= b) ? a : b;
}
static inline double np_clip(double x, double lo, double hi) {
    return np_minimum(np_maximum(x, lo), hi);
}

/* float64 -> int64 as numpy's astype does on x86-64 (cvttsd2si): NaN and
 * out-of-range values become INT64_MIN. */
static inline int64_t np_to_i64(double v) {
    if (!(v >= -9223372036854775808.0 && v < 9223372036854775808.0)) return INT64_MIN;
    return (int64_t)v;
}

/* npy_floor_divide(a, b) for b = tile size (a power of two in practice);
 * restated from numpy's npy_divmod so NaN/inf behave the same. */
static inline double np_floor_divide(double a, double b) {
    double mod = fmod(a, b);
    double div = (a - mod) / b;
    if (mod) {
        if ((b < 0) != (mod < 0)) {
            mod += b;
            div -= 1.0;
        }
    }
    double floordiv;
    if (div) {
        floordiv = floor(div);
        if (div - floordiv > 0.5) floordiv += 1.0;
    } else {
        floordiv = copysign(0.0, a / b);
    }
    return floordiv;
}

/* min_mahalanobis_sq_to_rect, projection.py:191-226 (one row). */
static inline double min_mahal_sq_to_rect(double mx, double my, double a, double b, double c,
                                          double lx, double ly, double hx, double hy) {
#define QUAD(dx, dy) ((a * (dx)) * (dx) + ((2.0 * b) * (dx)) * (dy) + (c * (dy)) * (dy))
    double best = INFINITY;
    double ex[2] = {lx, hx};
    for (int i = 0; i < 2; ++i) {
        double dx = ex[i] - mx;
        double ys = np_clip(my - (b / c) * dx, ly, hy);
        double dy = ys - my;
        best = np_minimum(best, QUAD(dx, dy));
    }
    double ey[2] = {ly, hy};
    for (int i = 0; i < 2; ++i) {
        double dy = ey[i] - my;
        double xs = np_clip(mx - (b / a) * dy, lx, hx);
        double dx = xs - mx;
        best = np_minimum(best, QUAD(dx, dy));
    }
    if ((mx >= lx) && (mx <= hx) && (my >= ly) && (my <= hy)) best = 0.0;
    return best;
#undef QUAD
}

/*
 * project_arrays, projection.py:240-308, with batch_covariances core.py:193-209.
 * Outputs are written compacted (row order preserved); returns N.
 * inv_covs is (N, 4) = [[i00, i01], [i10, i11]].
 */
int64_t or_project(int64_t G, const float* positions, const float* rotations, const float* scales,
                   const float* opacities, const int64_t* ids, const OrCamera* cam,
                   double* means2d, double* inv_covs, double* depths, double* opac_out,
                   int64_t* source_ids, int64_t* rows_out) {
    const double* R = cam->R;
    int64_t n = 0;
    for (int64_t g = 0; g < G; ++g) {
        double p0 = positions[3 * g], p1 = positions[3 * g + 1], p2 = positions[3 * g + 2];
        double cp[3];
        for (int r = 0; r < 3; ++r)  /* pos @ R.T (dgemm) + t */
            cp[r] = fma(p2, R[3 * r + 2], fma(p1, R[3 * r + 1], p0 * R[3 * r])) + cam->t[r];
        double x = cp[0], y = cp[1], z = cp[2];
        if (!(z > cam->near_)) continue;
        double m0 = (cam->fx * x) / z + cam->cx;
        double m1 = (cam->fy * y) / z + cam->cy;

        /* batch_covariances */
        double w = rotations[4 * g], qx = rotations[4 * g + 1], qy = rotations[4 * g + 2],
               qz = rotations[4 * g + 3];
        double rot[9];
        rot[0] = 1 - 2 * (qy * qy + qz * qz);
        rot[1] = 2 * (qx * qy - w * qz);
        rot[2] = 2 * (qx * qz + w * qy);
        rot[3] = 2 * (qx * qy + w * qz);
        rot[4] = 1 - 2 * (qx * qx + qz * qz);
        rot[5] = 2 * (qy * qz - w * qx);
        rot[6] = 2 * (qx * qz - w * qy);
        rot[7] = 2 * (qy * qz + w * qx);
        rot[8] = 1 - 2 * (qx * qx + qy * qy);
        double s[3] = {scales[3 * g], scales[3 * g + 1], scales[3 * g + 2]};
        double m[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) m[3 * r + c] = rot[3 * r + c] * s[c];
        double cov[9];
        for (int r = 0; r < 3; ++r)  /* m @ m^T (dsyrk) */
            for (int c = 0; c < 3; ++c)
                cov[3 * r + c] = fma(m[3 * r + 2], m[3 * c + 2],
                                     fma(m[3 * r + 1], m[3 * c + 1], m[3 * r] * m[3 * c]));
        double cs[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) cs[3 * r + c] = (cov[3 * r + c] + cov[3 * c + r]) * 0.5;

        /* J @ W rows, projection.py:265-271 */
        double jw[6];
        double fxz = cam->fx / z, fyz = cam->fy / z;
        double gx = (cam->fx * x) / (z * z), gy = (cam->fy * y) / (z * z);
        for (int k = 0; k < 3; ++k) {
            jw[k] = fxz * R[k] - gx * R[6 + k];
            jw[3 + k] = fyz * R[3 + k] - gy * R[6 + k];
        }
        /* (jw @ cov3d) @ jw.T (two dgemms) */
        double tmp[6];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                tmp[3 * r + c] = fma(jw[3 * r + 2], cs[6 + c],
                                     fma(jw[3 * r + 1], cs[3 + c], jw[3 * r] * cs[c]));
        double c2[4];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c)
                c2[2 * r + c] = fma(tmp[3 * r + 2], jw[3 * c + 2],
                                    fma(tmp[3 * r + 1], jw[3 * c + 1], tmp[3 * r] * jw[3 * c]));
        c2[0] += OR_LOWPASS;
        c2[3] += OR_LOWPASS;
        double det = c2[0] * c2[3] - c2[1] * c2[2];
        int ok = isfinite(det) && (det > 0) && isfinite(m0) && isfinite(m1);
        if (!ok) continue;
        double i00 = c2[3] / det, i11 = c2[0] / det, off = -c2[1] / det;
        double qmin = min_mahal_sq_to_rect(m0, m1, i00, off, i11, 0.0, 0.0,
                                           (double)(cam->width - 1), (double)(cam->height - 1));
        if (!(qmin <= OR_CUTOFF)) continue;
        means2d[2 * n] = m0;
        means2d[2 * n + 1] = m1;
        inv_covs[4 * n] = i00;
        inv_covs[4 * n + 1] = off;
        inv_covs[4 * n + 2] = off;
        inv_covs[4 * n + 3] = i11;
        depths[n] = z;
        opac_out[n] = (double)opacities[g];
        source_ids[n] = ids[g];
        rows_out[n] = g;
        ++n;
    }
    return n;
}

/* ---------------- binning, projection.py:379-450 ---------------- */

static const double* g_sort_depth;
static const int64_t* g_sort_ids;
static int cmp_depth_id(const void* pa, const void* pb) {
    int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    double da = g_sort_depth[a], db = g_sort_depth[b];
    if (da < db) return -1;
    if (da > db) return 1;
    if (g_sort_ids[a] < g_sort_ids[b]) return -1;
    if (g_sort_ids[a] > g_sort_ids[b]) return 1;
    return (a < b) ? -1 : (a > b);
}

/* canonical order = lexsort((source_ids, depths)), projection.py:396 */
void or_canonical_order(int64_t n, const double* depths, const int64_t* source_ids, int64_t* order) {
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    g_sort_depth = depths;
    g_sort_ids = source_ids;
    qsort(order, (size_t)n, sizeof(int64_t), cmp_depth_id);
}

/* candidate tile rectangle, projection.py:406-418 (one canonical Gaussian) */
static inline void cand_rect(double mx, double my, const double* inv, int64_t ts, int64_t tiles_x,
                             int64_t tiles_y, int64_t* tx0, int64_t* tx1, int64_t* ty0,
                             int64_t* ty1) {
    double den = inv[0] * inv[3] - inv[1] * inv[1];
    double cov_xx = inv[3] / den;
    double cov_yy = inv[0] / den;
    double rx = 3.0 * sqrt(np_maximum(cov_xx, 0.0));
    double ry = 3.0 * sqrt(np_maximum(cov_yy, 0.0));
    double tsd = (double)ts;
    int64_t v;
#define CLIPI(v, hi) ((v) < 0 ? 0 : ((v) > (hi) ? (hi) : (v)))
    v = np_to_i64(np_floor_divide(mx - rx, tsd)); *tx0 = CLIPI(v, tiles_x - 1);
    v = np_to_i64(np_floor_divide(mx + rx, tsd)); *tx1 = CLIPI(v, tiles_x - 1);
    v = np_to_i64(np_floor_divide(my - ry, tsd)); *ty0 = CLIPI(v, tiles_y - 1);
    v = np_to_i64(np_floor_divide(my + ry, tsd)); *ty1 = CLIPI(v, tiles_y - 1);
#undef CLIPI
}

static inline int tile_hit(double mx, double my, const double* inv, int64_t tx, int64_t ty,
                           int64_t ts, int64_t W, int64_t H) {
    double lx = (double)(tx * ts), ly = (double)(ty * ts);
    double hx = np_minimum(lx + (double)ts, (double)W) - 1;
    double hy = np_minimum(ly + (double)ts, (double)H) - 1;
    double q = min_mahal_sq_to_rect(mx, my, inv[0], inv[1], inv[3], lx, ly, hx, hy);
    return q <= OR_CUTOFF;
}

/*
 * Per-tile lists.  Inputs are the projected arrays in canonical order
 * (caller applied or_canonical_order).  tile_offsets has n_tiles+1 entries;
 * tile_lists receives canonical indices; capacity = size of tile_lists.
 * Returns total pairs (may exceed capacity: call again with more room).
 */
int64_t or_bin(int64_t n, const double* means2d, const double* inv_covs, int64_t ts, int64_t W,
               int64_t H, int64_t* tile_offsets, int64_t* tile_lists, int64_t capacity) {
    int64_t tiles_x = (W + ts - 1) / ts, tiles_y = (H + ts - 1) / ts;
    int64_t n_tiles = tiles_x * tiles_y;
    int64_t* counts = (int64_t*)calloc((size_t)n_tiles, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        int64_t tx0, tx1, ty0, ty1;
        const double* inv = inv_covs + 4 * i;
        cand_rect(means2d[2 * i], means2d[2 * i + 1], inv, ts, tiles_x, tiles_y, &tx0, &tx1, &ty0, &ty1);
        for (int64_t ty = ty0; ty <= ty1; ++ty)
            for (int64_t tx = tx0; tx <= tx1; ++tx)
                if (tile_hit(means2d[2 * i], means2d[2 * i + 1], inv, tx, ty, ts, W, H))
                    counts[ty * tiles_x + tx]++;
    }
    tile_offsets[0] = 0;
    for (int64_t t = 0; t < n_tiles; ++t) tile_offsets[t + 1] = tile_offsets[t] + counts[t];
    int64_t total = tile_offsets[n_tiles];
    if (total <= capacity) {
        memset(counts, 0, (size_t)n_tiles * sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i) {
            int64_t tx0, tx1, ty0, ty1;
            const double* inv = inv_covs + 4 * i;
            cand_rect(means2d[2 * i], means2d[2 * i + 1], inv, ts, tiles_x, tiles_y, &tx0, &tx1, &ty0, &ty1);
            for (int64_t ty = ty0; ty <= ty1; ++ty)
                for (int64_t tx = tx0; tx <= tx1; ++tx)
                    if (tile_hit(means2d[2 * i], means2d[2 * i + 1], inv, tx, ty, ts, W, H)) {
                        int64_t t = ty * tiles_x + tx;
                        tile_lists[tile_offsets[t] + counts[t]++] = i;
                    }
        }
    }
    free(counts);
    return total;
}

/*
 * Fused multi-level sparse splat: tile_blend_weights rasterizer.py:133-181 +
 * the scatter loop of _splat_levels sparse_splat.py:138-150.  Projected
 * arrays are in canonical order; rows[] maps to scene rows.
 *   cat_idx (G, C) int64 channel indices, cat_vals (G, C) float32 values
 *   out (H, W, nch) float64 zero-initialised by the caller, final_t (H, W).
 * Tiles are independent; OpenMP parallelises over them (worker-count
 * invariant like the reference's thread pool).
 */
void or_splat(int64_t n_tiles_x, int64_t n_tiles_y, int64_t ts, int64_t W, int64_t H,
              const int64_t* tile_offsets, const int64_t* tile_lists, const double* means2d,
              const double* inv_covs, const double* opac, const int64_t* rows, int64_t C,
              const int64_t* cat_idx, const float* cat_vals, int64_t nch, int early_exit,
              double* out, double* final_t, int64_t tile_begin, int64_t tile_end) {
    int64_t n_tiles = n_tiles_x * n_tiles_y;
    if (tile_end > n_tiles) tile_end = n_tiles;
#pragma omp parallel
    {
        int64_t cap = 0;
        double* alpha = NULL;
        double* T = NULL;
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = tile_begin; t < tile_end; ++t) {
            int64_t ty = t / n_tiles_x, tx = t % n_tiles_x;
            int64_t x0 = tx * ts, y0 = ty * ts;
            int64_t x1 = (x0 + ts < W) ? x0 + ts : W, y1 = (y0 + ts < H) ? y0 + ts : H;
            int64_t beg = tile_offsets[t], n = tile_offsets[t + 1] - beg;
            int64_t npx = (x1 - x0) * (y1 - y0);
            if (npx > cap) {
                cap = npx;
                alpha = (double*)realloc(alpha, sizeof(double) * (size_t)cap);
                T = (double*)realloc(T, sizeof(double) * (size_t)cap);
            }
            for (int64_t p = 0; p < npx; ++p) T[p] = 1.0;
            for (int64_t k = 0; k < n; ++k) {
                int64_t i = tile_lists[beg + k];
                double mx = means2d[2 * i], my = means2d[2 * i + 1];
                double a = inv_covs[4 * i], b = inv_covs[4 * i + 1], c = inv_covs[4 * i + 3];
                double o = opac[i];
                int live = 0;
                for (int64_t p = 0; p < npx; ++p) {
                    double px = (double)(x0 + p % (x1 - x0)), py = (double)(y0 + p / (x1 - x0));
                    double dx = px - mx, dy = py - my;
                    double q = (a * dx) * dx + ((2.0 * b) * dx) * dy + (c * dy) * dy;
                    double al = o * exp(-0.5 * q);
                    al = np_minimum(al, OR_ALPHA_CLAMP);
                    if (q > OR_CUTOFF) al = 0.0;
                    double tb = T[p];
                    double e = (!early_exit || tb >= OR_EARLY_EXIT) ? al * tb : 0.0;
                    alpha[p] = e;
                    if (e > 0.0) live = 1;
                    /* cumprod keeps multiplying past the cut; counted is a prefix */
                    if (!early_exit || tb >= OR_EARLY_EXIT) T[p] = tb * (1.0 - al);
                    else T[p] = tb;  /* frozen at the last counted value */
                }
                if (!live) continue;
                int64_t row = rows[i];
                for (int64_t cc = 0; cc < C; ++cc) {
                    int64_t ch = cat_idx[row * C + cc];
                    double v = (double)cat_vals[row * C + cc];
                    for (int64_t p = 0; p < npx; ++p) {
                        int64_t xx = x0 + p % (x1 - x0), yy = y0 + p / (x1 - x0);
                        out[(yy * W + xx) * nch + ch] += alpha[p] * v;
                    }
                }
            }
            for (int64_t p = 0; p < npx; ++p) {
                int64_t xx = x0 + p % (x1 - x0), yy = y0 + p / (x1 - x0);
                final_t[yy * W + xx] = T[p];
            }
        }
        free(alpha);
        free(T);
    }
}

/* decode, sparse_splat.py:183-199: one level, (HW, L) @ (L, D) in float64. */
void or_decode(int64_t hw, int64_t L, int64_t D, const double* w, int64_t w_stride,
               const float* atoms, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < hw; ++p) {
        double* o = out + p * D;
        for (int64_t d = 0; d < D; ++d) o[d] = 0.0;
        for (int64_t l = 0; l < L; ++l) {
            double wl = w[p * w_stride + l];
            if (wl == 0.0) continue;
            const float* arow = atoms + l * D;
            for (int64_t d = 0; d < D; ++d) o[d] += wl * (double)arow[d];
        }
    }
}

/* two-branch stable sigmoid, query.py:55-62 */
static inline double sigmoid2(double x) {
    if (x >= 0) return 1.0 / (1.0 + exp(-x));
    double ex = exp(x);
    return ex / (1.0 + ex);
}

/* relevancy_map, query.py:65-84: min over canonicals of sigma(f.q - f.c). */
void or_relevancy(int64_t hw, int64_t D, const double* feats, const double* q, int64_t nc,
                  const double* canon, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < hw; ++p) {
        const double* f = feats + p * D;
        double ql = 0.0;
        for (int64_t d = 0; d < D; ++d) ql += f[d] * q[d];
        double best = INFINITY;
        for (int64_t j = 0; j < nc; ++j) {
            double cl = 0.0;
            for (int64_t d = 0; d < D; ++d) cl += f[d] * canon[j * D + d];
            double s = sigmoid2(ql - cl);
            best = np_minimum(best, s);
        }
        out[p] = best;
    }
}

/* mean_filter, query.py:87-108: edge padding + integral image. */
void or_mean_filter(int64_t h, int64_t w, const double* in, int64_t window, double* out) {
    int64_t r = window / 2;
    int64_t ph = h + 2 * r, pw = w + 2 * r;
    double* integ = (double*)calloc((size_t)((ph + 1) * (pw + 1)), sizeof(double));
    /* cumsum over axis 0 of the padded map, then over axis 1 */
    for (int64_t y = 0; y < ph; ++y) {
        int64_t sy = y - r; sy = sy < 0 ? 0 : (sy >= h ? h - 1 : sy);
        for (int64_t x = 0; x < pw; ++x) {
            int64_t sx = x - r; sx = sx < 0 ? 0 : (sx >= w ? w - 1 : sx);
            double v = in[sy * w + sx];
            double above = (y > 0) ? integ[y * (pw + 1) + (x + 1)] : 0.0;
            integ[(y + 1) * (pw + 1) + (x + 1)] = (y > 0) ? above + v : v;
        }
    }
    for (int64_t y = 0; y < ph; ++y) {
        double* row = integ + (y + 1) * (pw + 1) + 1;
        for (int64_t x = 1; x < pw; ++x) row[x] = row[x - 1] + row[x];
    }
#define I(yy, xx) integ[(yy) * (pw + 1) + (xx)]
    double inv = (double)(window * window);
    for (int64_t y = 0; y < h; ++y)
        for (int64_t x = 0; x < w; ++x) {
            double s = I(y + window, x + window) - I(y, x + window) - I(y + window, x) + I(y, x);
            out[y * w + x] = s / inv;
        }
#undef I
    free(integ);
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
