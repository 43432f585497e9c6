// sf_train.cu -- the training step of the sparse coefficient field on the
// device (reference splatfield/train.py).
//
// Geometry is frozen, so the rendered coefficient map W is linear in the
// per-Gaussian coefficients and the blend weights are constants of a step
// (train.py:1-18).  One step here:
//
//   k_train_plan      softmax -> top-K -> renormalise per (Gaussian, level)
//                     (normalize_batch, train.py:131-139) written straight
//                     into the blend's scatter-plan record; the blend kernel
//                     then renders W (sf_render_frame).
//   k_train_residual  per 32-pixel block and level: F = W atoms, r = (F - T)
//                     mask, the block's loss partial, dF = 2 s r (+ the
//                     cosine term), dW = dF atoms^T (forward_loss
//                     train.py:201-279 and the first half of backward
//                     train.py:303-329), all fp64; F itself never goes to HBM.
//   k_train_cbgrad    dL/datoms = W^T dF (train.py:321) as a split-K product
//                     with per-split partials, k_train_sum_splits adds them
//                     in split order (deterministic).
//   k_splat_transpose (sf_blend.cu) ghat = e^T dW over the same tile lists.
//   k_train_logits    the top-K softmax backward (train.py:331-340), then,
//                     in a training step, the Adam update of the logits
//                     (OptimState.step, train.py:79-107); squared-gradient
//                     partials for the gradient norm.
//   k_train_adam      Adam on the codebooks.
//   k_train_reduce    fixed-order sums of the loss / norm partials.
//
// Every reduction runs in a fixed order: the loss and the gradients do not
// depend on scheduling (the transpose splat's per-Gaussian sums excepted,
// which use fp32 atomics across tiles).
#include <stdint.h>

#include "sf_common.cuh"

namespace sf {
namespace train {

constexpr int kPx = 32;       // pixels per residual block
constexpr int kCols = 64;     // feature columns per chunk
constexpr int kThreads = 256;
constexpr int kApitch = kCols + 1;  // padded atom chunk rows (conflict-free column walks)

// ---------------------------------------------------------------------------
// softmax -> top-K -> renormalise, one warp per (device row, level): lane
// holds logits l = lane and lane + 32 (L <= 64).  Ties in p go to the lower
// index (the stable argsort of -p, train.py:125-128); the kept indices are
// emitted in ascending order.

struct RowSoftmax {
    double p0, p1;      // p at l = lane, lane + 32 (0 beyond L)
    int idx[16];        // kept indices, ascending (K <= 16)
    double kept_sum;
};

__device__ __forceinline__ RowSoftmax row_softmax(const double* __restrict__ lg, int L, int K, int lane) {
    RowSoftmax r;
    const bool v0 = lane < L, v1 = lane + 32 < L;
    const double x0 = v0 ? lg[lane] : -INFINITY, x1 = v1 ? lg[lane + 32] : -INFINITY;
    double m = fmax(x0, x1);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const double e0 = v0 ? exp(x0 - m) : 0.0, e1 = v1 ? exp(x1 - m) : 0.0;
    double s = e0 + e1;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    r.p0 = e0 / s;
    r.p1 = e1 / s;
    // K rounds of (max p, lowest index)
    bool t0 = !v0, t1 = !v1;  // taken (or invalid)
    uint32_t sel_lo = 0u, sel_hi = 0u;  // selected indices as a 64-bit set
    for (int k = 0; k < K; ++k) {
        double bp = -1.0;
        int bi = 0x7fffffff;
        if (!t0) bp = r.p0, bi = lane;
        if (!t1 && (r.p1 > bp)) bp = r.p1, bi = lane + 32;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double op = __shfl_xor_sync(0xffffffffu, bp, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (op > bp || (op == bp && oi < bi)) bp = op, bi = oi;
        }
        if (bi == lane) t0 = true;
        if (bi == lane + 32) t1 = true;
        if (bi < 32) sel_lo |= 1u << bi;
        else sel_hi |= 1u << (bi - 32);
    }
    // ascending order of the selected set; the kept sum in that order
    int k = 0;
    double ks = 0.0;
    for (uint32_t m2 = sel_lo; m2; m2 &= m2 - 1) r.idx[k++] = __ffs(m2) - 1;
    for (uint32_t m2 = sel_hi; m2; m2 &= m2 - 1) r.idx[k++] = 32 + __ffs(m2) - 1;
    for (int j = 0; j < K; ++j) {
        const int i = r.idx[j];
        const double pi = __shfl_sync(0xffffffffu, i < 32 ? r.p0 : r.p1, i & 31);
        ks += pi;
    }
    r.kept_sum = ks;
    return r;
}

__device__ __forceinline__ double p_at(const RowSoftmax& r, int i) {
    return __shfl_sync(0xffffffffu, i < 32 ? r.p0 : r.p1, i & 31);
}

// plan record of device row g (layout of launch_pack_channels: C channel
// words, then C fp32 values at chan_val_offset(C))
__global__ void __launch_bounds__(kThreads) k_train_plan(int64_t G, int levels, int L, int K,
                                                         const double* __restrict__ logits,
                                                         unsigned char* __restrict__ plan) {
    const int64_t g = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= G) return;
    const int C = levels * K;
    const int cs = chan_rec_bytes(C), voff = chan_val_offset(C);
    unsigned char* rec = plan + (size_t)g * cs;
    for (int b = 0; b < levels; ++b) {
        const RowSoftmax r = row_softmax(logits + ((size_t)b * G + g) * L, L, K, lane);
        for (int j = 0; j < K; ++j) {
            const int i = r.idx[j];
            const double pi = p_at(r, i);
            if (lane == 0) {
                reinterpret_cast<uint32_t*>(rec)[b * K + j] = (uint32_t)(i + b * L) * kChanWord;
                reinterpret_cast<float*>(rec + voff)[b * K + j] = (float)(pi / r.kept_sum);
            }
        }
    }
    if (lane == 0)
        for (int c = C; c < voff / 4; ++c) {
            reinterpret_cast<uint32_t*>(rec)[c] = 0u;
            reinterpret_cast<float*>(rec + voff)[c] = 0.f;
        }
}

// ---------------------------------------------------------------------------
// residual block: 32 pixels x one level; 8 chunks of 64 feature columns.
// MODE 0: per-pixel cosine statistics only (F.T, |F|^2, |T|^2).
// MODE 1: loss partial, dF (fp64, to HBM for the codebook gradient), dW.

struct ResArgs {
    int64_t HW;
    int levels, L, D;
    const float* wmap;       // (HW, levels * L) coefficient map
    const double* atoms;     // (levels, L, D)
    const double* targets;   // (levels, HW, D)
    const double* mask;      // (HW) 0 / 1, or null
    double scale;            // 1 / (levels * n_valid)
    double cos_w;            // cosine weight
    double* pix_stats;       // (levels, HW, 3) [MODE 0 out / MODE 1 in when cos_w]
    double* dF;              // (levels, HW, D)
    float* dW;               // (HW, levels * L)
    double* loss_part;       // (levels, n_blocks, 2): squared residual, cosine term
};

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_train_residual(ResArgs A) {
    extern __shared__ __align__(16) double tr_smem[];
    double* Wt = tr_smem;                       // [32][64]
    double* Ac = Wt + kPx * 64;                 // [64][kApitch]
    double* dFc = Ac + 64 * kApitch;            // [32][64]
    __shared__ double red[kThreads / 32][3];
    const int lv = blockIdx.y, L = A.L, D = A.D;
    const int64_t p0 = (int64_t)blockIdx.x * kPx;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nch = A.levels * L;
    for (int i = tid; i < kPx * 64; i += kThreads) {
        const int px = i / 64, l = i % 64;
        const int64_t p = p0 + px;
        Wt[i] = (p < A.HW && l < L) ? (double)A.wmap[p * nch + (size_t)lv * L + l] : 0.0;
    }
    const int px = tid >> 3, cq = tid & 7;  // pixel of the thread, column phase
    const int64_t p = p0 + px;
    const bool inside = p < A.HW;
    const double mk = (A.mask && inside) ? A.mask[p] : 1.0;
    double sq = 0.0, ft = 0.0, ff = 0.0, tt = 0.0;
    double cosv = 0.0, fn = 0.0, tn = 0.0, denom = 1.0, fnn = 1.0;
    if (MODE == 1 && A.cos_w != 0.0 && inside) {
        const double* ps = A.pix_stats + ((size_t)lv * A.HW + p) * 3;
        fn = sqrt(ps[1]);
        tn = sqrt(ps[2]);
        denom = fmax(fn * tn, 1e-12);
        cosv = ps[0] / denom;
        fnn = fmax(fn * fn, 1e-12);
    }
    double dw[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) dw[j] = 0.0;
    const double* arow = A.atoms + (size_t)lv * L * D;
    const double* trow = A.targets + ((size_t)lv * A.HW + (inside ? p : 0)) * D;
    for (int c0 = 0; c0 < D; c0 += kCols) {
        __syncthreads();
        for (int i = tid; i < 64 * kCols; i += kThreads) {
            const int l = i / kCols, c = i % kCols;
            Ac[l * kApitch + c] = (l < L && c0 + c < D) ? arow[(size_t)l * D + c0 + c] : 0.0;
        }
        __syncthreads();
        // F[px][c] for c = cq + 8 j
        double f[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = 0.0;
        for (int l = 0; l < L; ++l) {
            const double w = Wt[px * 64 + l];
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = fma(w, Ac[l * kApitch + cq + 8 * j], f[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = cq + 8 * j;
            const bool col = c0 + c < D;
            const double t = (inside && col) ? trow[c0 + c] : 0.0;
            if (MODE == 0) {
                ft = fma(f[j], t, ft);
                ff = fma(f[j], f[j], ff);
                tt = fma(t, t, tt);
            } else {
                double r = (f[j] - t) * mk;
                if (!inside || !col) r = 0.0;
                sq = fma(r, r, sq);
                double g = 2.0 * A.scale * r;
                if (A.cos_w != 0.0) {
                    const double cg = -(t / denom - cosv * f[j] / fnn) * mk;
                    g += A.cos_w * A.scale * ((inside && col) ? cg : 0.0);
                }
                dFc[px * 64 + c] = g;
                if (inside && col) A.dF[((size_t)lv * A.HW + p) * D + c0 + c] = g;
            }
        }
        if (MODE == 1) {
            __syncthreads();
            // dW[px][l] for l = cq + 8 j: sum over this chunk's columns
            for (int c = 0; c < kCols; ++c) {
                const double g = dFc[px * 64 + c];
#pragma unroll
                for (int j = 0; j < 8; ++j) dw[j] = fma(g, Ac[(cq + 8 * j) * kApitch + c], dw[j]);
            }
        }
    }
    if (MODE == 0) {
        // per-pixel sums over the 8 threads of the pixel (lanes 8k .. 8k+7), fixed order
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            ft += __shfl_xor_sync(0xffffffffu, ft, o);
            ff += __shfl_xor_sync(0xffffffffu, ff, o);
            tt += __shfl_xor_sync(0xffffffffu, tt, o);
        }
        if (cq == 0 && inside) {
            double* ps = A.pix_stats + ((size_t)lv * A.HW + p) * 3;
            ps[0] = ft;
            ps[1] = ff;
            ps[2] = tt;
        }
        return;
    }
    if (inside) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int l = cq + 8 * j;
            if (l < L) A.dW[p * nch + (size_t)lv * L + l] = (float)dw[j];
        }
    }
    // loss partials: squared residual, and the cosine term once per pixel
    double ct = (A.cos_w != 0.0 && inside && cq == 0) ? (1.0 - cosv) * mk : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        ct += __shfl_xor_sync(0xffffffffu, ct, o);
    }
    if (lane == 0) {
        red[wid][0] = sq;
        red[wid][1] = ct;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) a += red[w][0], b += red[w][1];
        double* lp = A.loss_part + ((size_t)lv * gridDim.x + blockIdx.x) * 2;
        lp[0] = a;
        lp[1] = b;
    }
}

// ---------------------------------------------------------------------------
// dL/datoms = W^T dF: block = (64-column slice n0, level, pixel split s);
// thread = 4 x 4 outputs (l = lg + 16 i, n = ng + 16 j).
__global__ void __launch_bounds__(kThreads) k_train_cbgrad(int64_t HW, int levels, int L, int D, int splits,
                                                           const float* __restrict__ wmap,
                                                           const double* __restrict__ dF,
                                                           double* __restrict__ part) {
    __shared__ double Ws[kPx][64 + 1];
    __shared__ double Gs[kPx][64 + 1];
    const int n0 = blockIdx.x * 64, lv = blockIdx.y, s = blockIdx.z;
    const int tid = threadIdx.x, ng = tid & 15, lg = tid >> 4;
    const int nch = levels * L;
    const int64_t per = (HW + splits - 1) / splits;
    const int64_t pa = (int64_t)s * per, pb = min(HW, pa + per);
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int64_t q0 = pa; q0 < pb; q0 += kPx) {
        __syncthreads();
        for (int i = tid; i < kPx * 64; i += kThreads) {
            const int pp = i / 64, c = i % 64;
            const int64_t q = q0 + pp;
            const bool ok = q < pb;
            Ws[pp][c] = (ok && c < L) ? (double)wmap[q * nch + (size_t)lv * L + c] : 0.0;
            Gs[pp][c] = (ok && n0 + c < D) ? dF[((size_t)lv * HW + q) * D + n0 + c] : 0.0;
        }
        __syncthreads();
        for (int pp = 0; pp < kPx; ++pp) {
            double w[4], g[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) w[i] = Ws[pp][lg + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) g[j] = Gs[pp][ng + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(w[i], g[j], acc[i][j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int l = lg + 16 * i, n = n0 + ng + 16 * j;
            if (l < L && n < D) part[(((size_t)s * levels + lv) * L + l) * D + n] = acc[i][j];
        }
}

__global__ void k_train_sum_splits(int64_t n, int splits, const double* __restrict__ part, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double a = 0.0;
    for (int s = 0; s < splits; ++s) a += part[(size_t)s * n + i];
    out[i] = a;
}

// ---------------------------------------------------------------------------
// top-K softmax backward (train.py:331-340) and, optionally, Adam on the
// logits.  ghat: (levels, G, K) fp32 from the transpose splat (plan slot
// order = ascending kept index).
struct AdamArgs {
    double lr, beta1, beta2, eps, bc1, bc2;  // bc = 1 - beta^t
};

__global__ void __launch_bounds__(kThreads) k_train_logits(int64_t G, int levels, int L, int K,
                                                           double* __restrict__ logits,
                                                           const float* __restrict__ ghat,
                                                           double* __restrict__ grad_out,
                                                           double* __restrict__ m, double* __restrict__ v,
                                                           AdamArgs ad, int adam, double* __restrict__ norm_part) {
    __shared__ double red[kThreads / 32];
    const int64_t row = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;  // (level, g) pair
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double sq = 0.0;
    if (row < (int64_t)levels * G) {
        const int b = (int)(row / G);
        const int64_t g = row - (int64_t)b * G;
        double* lg = logits + ((size_t)b * G + g) * L;
        const RowSoftmax r = row_softmax(lg, L, K, lane);
        // d_y = (ghat - sum(ghat w)) / s over the kept slots; u scattered at idx
        double gw = 0.0;
        for (int j = 0; j < K; ++j) {
            const double w = p_at(r, r.idx[j]) / r.kept_sum;
            gw += (double)ghat[((size_t)b * G + g) * K + j] * w;
        }
        double u0 = 0.0, u1 = 0.0;
        for (int j = 0; j < K; ++j) {
            const int i = r.idx[j];
            const double dy = ((double)ghat[((size_t)b * G + g) * K + j] - gw) / r.kept_sum;
            if (i == lane) u0 = dy;
            if (i == lane + 32) u1 = dy;
        }
        double dot = u0 * r.p0 + u1 * r.p1;
#pragma unroll
        for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        const double g0 = r.p0 * (u0 - dot), g1 = r.p1 * (u1 - dot);
        const bool v0 = lane < L, v1 = lane + 32 < L;
        sq = (v0 ? g0 * g0 : 0.0) + (v1 ? g1 * g1 : 0.0);
        if (grad_out) {
            double* go = grad_out + ((size_t)b * G + g) * L;
            if (v0) go[lane] = g0;
            if (v1) go[lane + 32] = g1;
        }
        if (adam) {
            double* mm = m + ((size_t)b * G + g) * L;
            double* vv = v + ((size_t)b * G + g) * L;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int l = lane + 32 * h;
                if (l >= L) continue;
                const double gr = h ? g1 : g0;
                double mi = mm[l], vi = vv[l];
                mi += (1.0 - ad.beta1) * (gr - mi);
                vi += (1.0 - ad.beta2) * (gr * gr - vi);
                mm[l] = mi;
                vv[l] = vi;
                lg[l] -= ad.lr * (mi / ad.bc1) / (sqrt(vi / ad.bc2) + ad.eps);
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) red[wid] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) a += red[w];
        norm_part[blockIdx.x] = a;
    }
}

// Adam on the codebooks (elementwise) + squared-gradient partials
__global__ void __launch_bounds__(kThreads) k_train_adam(int64_t n, double* __restrict__ param,
                                                         const double* __restrict__ grad, double* __restrict__ m,
                                                         double* __restrict__ v, AdamArgs ad, int adam,
                                                         double* __restrict__ norm_part) {
    __shared__ double red[kThreads / 32];
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    double sq = 0.0;
    if (i < n) {
        const double gr = grad[i];
        sq = gr * gr;
        if (adam) {
            double mi = m[i], vi = v[i];
            mi += (1.0 - ad.beta1) * (gr - mi);
            vi += (1.0 - ad.beta2) * (gr * gr - vi);
            m[i] = mi;
            v[i] = vi;
            param[i] -= ad.lr * (mi / ad.bc1) / (sqrt(vi / ad.bc2) + ad.eps);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) a += red[w];
        norm_part[blockIdx.x] = a;
    }
}

// out[j] = sum over i of part[i * stride + j], i in order (one thread per j)
__global__ void k_train_reduce(int64_t n, int stride, int width, const double* __restrict__ part,
                               double* __restrict__ out) {
    const int j = threadIdx.x;
    if (j >= width) return;
    double a = 0.0;
    for (int64_t i = 0; i < n; ++i) a += part[i * stride + j];
    out[j] = a;
}

}  // namespace train
}  // namespace sf

using namespace sf;
using namespace sf::train;

static int tcheck(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return SF_ERR_CUDA;
    }
    return SF_OK;
}

extern "C" int sf_train_plan(int64_t G, int32_t levels, int32_t L, int32_t K, const double* logits, void* plan,
                             void* stream) {
    if (L < 1 || L > 64 || K < 1 || K > 16 || K > L || levels < 1 || levels * K > 16) {
        set_error("sf_train_plan: unsupported shape (levels %d, L %d, K %d)", levels, L, K);
        return SF_ERR_VALIDATION;
    }
    if (G > 0)
        k_train_plan<<<(unsigned)ceil_div(G * 32, kThreads), kThreads, 0, (cudaStream_t)stream>>>(
            G, levels, L, K, logits, (unsigned char*)plan);
    return tcheck("sf_train_plan");
}

extern "C" int64_t sf_train_loss_blocks(int64_t HW) { return ceil_div(HW, kPx); }
extern "C" int32_t sf_train_cb_splits(void) { return 12; }

extern "C" int sf_train_residual(int64_t HW, int32_t levels, int32_t L, int32_t D, const float* wmap,
                                 const double* atoms, const double* targets, const double* mask, double scale,
                                 double cos_w, double* pix_stats, double* dF, float* dW, double* loss_part,
                                 void* stream) {
    if (L < 1 || L > 64 || D < 1 || levels < 1) {
        set_error("sf_train_residual: unsupported shape (L %d, D %d)", L, D);
        return SF_ERR_VALIDATION;
    }
    if (cos_w != 0.0 && !pix_stats) {
        set_error("sf_train_residual: the cosine term needs the per-pixel statistics buffer");
        return SF_ERR_VALIDATION;
    }
    ResArgs a{HW, levels, L, D, wmap, atoms, targets, mask, scale, cos_w, pix_stats, dF, dW, loss_part};
    const size_t smem = sizeof(double) * (kPx * 64 + 64 * kApitch + kPx * 64);
    const dim3 grid((unsigned)ceil_div(HW, kPx), (unsigned)levels);
    cudaStream_t st = (cudaStream_t)stream;
    ensure_smem_attr((const void*)k_train_residual<0>, smem);
    ensure_smem_attr((const void*)k_train_residual<1>, smem);
    if (HW > 0) {
        if (cos_w != 0.0) k_train_residual<0><<<grid, kThreads, smem, st>>>(a);
        k_train_residual<1><<<grid, kThreads, smem, st>>>(a);
    }
    return tcheck("sf_train_residual");
}

extern "C" int sf_train_cbgrad(int64_t HW, int32_t levels, int32_t L, int32_t D, const float* wmap,
                               const double* dF, double* part, double* grad_cb, void* stream) {
    const int splits = sf_train_cb_splits();
    cudaStream_t st = (cudaStream_t)stream;
    if (L < 1 || L > 64 || D < 1) {
        set_error("sf_train_cbgrad: unsupported shape");
        return SF_ERR_VALIDATION;
    }
    k_train_cbgrad<<<dim3((unsigned)ceil_div(D, 64), (unsigned)levels, (unsigned)splits), kThreads, 0, st>>>(
        HW, levels, L, D, splits, wmap, dF, part);
    const int64_t n = (int64_t)levels * L * D;
    k_train_sum_splits<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, splits, part, grad_cb);
    return tcheck("sf_train_cbgrad");
}

extern "C" int64_t sf_train_logit_blocks(int64_t G, int32_t levels) { return ceil_div((int64_t)levels * G * 32, kThreads); }
extern "C" int64_t sf_train_adam_blocks(int64_t n) { return ceil_div(n, kThreads); }

extern "C" int sf_train_logits(int64_t G, int32_t levels, int32_t L, int32_t K, double* logits, const float* ghat,
                               double* grad_out, double* m, double* v, double lr, double beta1, double beta2,
                               double eps, int64_t t, double* norm_part, void* stream) {
    if (L < 1 || L > 64 || K < 1 || K > 16) {
        set_error("sf_train_logits: unsupported shape");
        return SF_ERR_VALIDATION;
    }
    const int adam = t > 0 && m && v;
    AdamArgs ad{lr, beta1, beta2, eps, adam ? 1.0 - pow(beta1, (double)t) : 1.0, adam ? 1.0 - pow(beta2, (double)t) : 1.0};
    const int64_t nb = sf_train_logit_blocks(G, levels);
    if (nb > 0)
        k_train_logits<<<(unsigned)nb, kThreads, 0, (cudaStream_t)stream>>>(G, levels, L, K, logits, ghat, grad_out,
                                                                            m, v, ad, adam, norm_part);
    return tcheck("sf_train_logits");
}

extern "C" int sf_train_adam(int64_t n, double* param, const double* grad, double* m, double* v, double lr,
                             double beta1, double beta2, double eps, int64_t t, double* norm_part, void* stream) {
    const int adam = t > 0 && m && v;
    AdamArgs ad{lr, beta1, beta2, eps, adam ? 1.0 - pow(beta1, (double)t) : 1.0, adam ? 1.0 - pow(beta2, (double)t) : 1.0};
    const int64_t nb = sf_train_adam_blocks(n);
    if (nb > 0)
        k_train_adam<<<(unsigned)nb, kThreads, 0, (cudaStream_t)stream>>>(n, param, grad, m, v, ad, adam, norm_part);
    return tcheck("sf_train_adam");
}

extern "C" int sf_train_reduce(int64_t n, int32_t stride, int32_t width, const double* part, double* out,
                               void* stream) {
    if (width < 1 || width > 1024) {
        set_error("sf_train_reduce: width %d", width);
        return SF_ERR_VALIDATION;
    }
    k_train_reduce<<<1, 32 * ((width + 31) / 32), 0, (cudaStream_t)stream>>>(n, stride, width, part, out);
    return tcheck("sf_train_reduce");
}
