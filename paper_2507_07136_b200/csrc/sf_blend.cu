// sf_blend.cu -- K5/K6: per-tile front-to-back blending with top-K sparse scatter.
//
// Reference: tile_blend_weights (rasterizer.py:133-181) and the scatter loop
// of _splat_levels (sparse_splat.py:138-150):
//     alpha_i = min(o_i * exp(-q_i / 2), 0.99), alpha_i = 0 if q_i > 9
//     e_i = alpha_i * T_i  counted iff T_i >= 1e-4,  T_{i+1} = T_i (1 - alpha_i)
//     W[p, cat_idx[i]] += e_i[p] * cat_vals[i]
//
// B200 mapping.  One CTA per 16x16 tile (x channel block), one pixel per
// thread; each warp owns an 8x4 pixel patch so the set of Gaussians live in
// a warp stays small.  The tile's depth-ordered list is streamed through
// shared memory in batches of 32 Gaussians.  Per (pixel, Gaussian) the
// rejection test q > 9 runs in fp32 with a conservative guard band (|q32 -
// q64| <= 1.5e-6 S, guard 1e-4 (1 + S), S = a dx^2 + c dy^2); survivors are
// re-evaluated in fp64 with the reference's exact op order, so the q <= 9
// membership decision is bit-exact and alpha / T carry fp64 accuracy (the
// T >= 1e-4 early-exit decision therefore matches the fp64 reference).  The
// coefficient accumulator is fp32 in shared memory, laid out
// acc[channel][pixel-slot] with a 257-float row pitch: the K channel
// indices of a Gaussian are warp-uniform, so every scatter is one
// conflict-free wavefront; the pitch also makes the transposed read for the
// channel-contiguous HBM write conflict-free.  A warp skips a Gaussian's
// scatter unless some lane has e > 0 (__any_sync vote), and the CTA stops
// streaming when every pixel is saturated (__syncthreads_and vote).
//
// Optional fused epilogue: per pixel and level, logits against the query and
// the canonical phrases via the projected codebook P = atoms @ [q; c]^T
// (fp64), then relevancy = min_j sigmoid(l_q - l_j) (query.py:65-84) -- the
// coefficient tile never has to be re-read from HBM for the query.
#include "sf_common.cuh"

namespace sf {

constexpr int kBlendThreads = 256;
constexpr int kBatch = 32;
constexpr int kAccPitch = 257;
constexpr int kMaxC = 16;            // channels per Gaussian (levels*K) supported in one pass
constexpr int kChBlock = 192;        // accumulator channels per CTA (smem bound)
constexpr uint32_t kInvalidOff = 0xffffffffu;

struct BlendSmem {
    Blend32 g32[kBatch];
    Proj64 g64[kBatch];
    uint32_t off[kBatch][kMaxC];
    float val[kBatch][kMaxC];
};

__device__ __forceinline__ double sigmoid2(double x) {
    if (x >= 0) return 1.0 / (1.0 + exp(-x));
    double ex = exp(x);
    return ex / (1.0 + ex);
}

__global__ void __launch_bounds__(kBlendThreads, 1) k_blend(BlendArgs A, int ch_block) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BlendSmem& S = *reinterpret_cast<BlendSmem*>(smem_raw);
    float* acc = reinterpret_cast<float*>(smem_raw + sizeof(BlendSmem));
    __shared__ int s_done_all;

    if (A.stats[SF_STAT_OVERFLOW]) return;
    const int tile = blockIdx.x;
    const int ch0 = blockIdx.y * ch_block;
    const int nchb = min(ch_block, A.n_ch - ch0);
    const int tx = tile % A.tiles_x, ty = tile / A.tiles_x;
    const int x0 = tx * SF_TILE, y0 = ty * SF_TILE;
    const int slot = threadIdx.x;
    const int warp = slot >> 5, lane = slot & 31;
    const int lx = (warp & 1) * 8 + (lane & 7);
    const int ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = x0 + lx, py = y0 + ly;
    const bool inside = (px < A.W) && (py < A.H);

    for (int i = threadIdx.x; i < nchb * kAccPitch; i += kBlendThreads) acc[i] = 0.f;

    const uint32_t beg = A.tile_offsets[tile], end = A.tile_offsets[tile + 1];
    const float pxf = (float)px, pyf = (float)py;
    const double pxd = (double)px, pyd = (double)py;
    double T = 1.0;
    bool done = !inside;
    const int C = A.C;

    for (uint32_t base = beg; base < end; base += kBatch) {
        const int nb = (int)min((uint32_t)kBatch, end - base);
        __syncthreads();  // previous batch fully consumed
        if (threadIdx.x < nb) {
            uint32_t r = A.entries[base + threadIdx.x];
            S.g32[threadIdx.x] = A.b32[r];
            S.g64[threadIdx.x] = A.p64[r];
        }
        for (int idx = threadIdx.x; idx < nb * C; idx += kBlendThreads) {
            int j = idx / C, k = idx - j * C;
            uint32_t r = A.entries[base + j];
            int ch = (int)A.ch_idx[(size_t)r * C + k] - ch0;
            S.off[j][k] = (ch >= 0 && ch < nchb) ? (uint32_t)(ch * kAccPitch) : kInvalidOff;
            S.val[j][k] = A.ch_val[(size_t)r * C + k];
        }
        __syncthreads();

        for (int j = 0; j < nb; ++j) {
            float ef = 0.f;
            if (!done) {
                const Blend32 g = S.g32[j];
                float dx = (pxf - g.mx_hi) - g.mx_lo;
                float dy = (pyf - g.my_hi) - g.my_lo;
                float adx = g.a * dx, cdy = g.c * dy;
                float q32 = adx * dx + g.b2 * dx * dy + cdy * dy;
                float s32 = adx * dx + cdy * dy;
                if (q32 <= 9.0f + 1e-4f * (1.0f + s32)) {
                    // exact reference evaluation (rasterizer.py:161-168)
                    const Proj64 p = S.g64[j];
                    double ddx = __dadd_rn(pxd, -p.mx), ddy = __dadd_rn(pyd, -p.my);
                    double t1 = __dmul_rn(__dmul_rn(p.a, ddx), ddx);
                    double t2 = __dmul_rn(__dmul_rn(__dmul_rn(2.0, p.b), ddx), ddy);
                    double t3 = __dmul_rn(__dmul_rn(p.c, ddy), ddy);
                    double q = __dadd_rn(__dadd_rn(t1, t2), t3);
                    if (q <= SF_CUTOFF) {
                        double al = __dmul_rn((double)g.opacity, exp(__dmul_rn(-0.5, q)));
                        al = np_minimum(al, SF_ALPHA_CLAMP);
                        double e = __dmul_rn(al, T);
                        T = __dmul_rn(T, __dadd_rn(1.0, -al));
                        ef = (float)e;
                        if (A.early_exit && T < SF_EARLY_EXIT_T) done = true;
                    }
                }
            }
            if (__any_sync(0xffffffffu, ef > 0.f)) {
#pragma unroll 4
                for (int k = 0; k < C; ++k) {
                    uint32_t off = S.off[j][k];
                    if (off != kInvalidOff) acc[off + slot] += ef * S.val[j][k];
                }
            }
        }
        if (__syncthreads_and(done)) break;
    }
    __syncthreads();

    // ---- outputs ----
    if (blockIdx.y == 0 && A.final_t && inside) A.final_t[(size_t)py * A.W + px] = (float)T;
    if (A.coeff_map) {
        const int tw = min(SF_TILE, A.W - x0), th = min(SF_TILE, A.H - y0);
        for (int r = 0; r < th; ++r) {
            float* row = A.coeff_map + ((size_t)(y0 + r) * A.W + x0) * A.n_ch + ch0;
            const int wr = (r >> 2) * 2, lr = (r & 3) * 8;
            for (int idx = threadIdx.x; idx < tw * nchb; idx += kBlendThreads) {
                int x = idx / nchb, ch = idx - x * nchb;
                int sl = (wr + (x >> 3)) * 32 + lr + (x & 7);
                row[(size_t)x * A.n_ch + ch] = acc[ch * kAccPitch + sl];
            }
        }
    }
    if (A.proj_cb && inside && nchb == A.n_ch) {
        // fused relevancy: logits_j = sum_l W[l] * P[b][l][j]  (fp64)
        const int nv = 1 + A.n_canon;
        for (int b = 0; b < A.n_levels; ++b) {
            const double* P = A.proj_cb + (size_t)b * A.L * nv;
            double lq = 0.0;
            double best = INFINITY;
            // query logit
            for (int l = 0; l < A.L; ++l) lq = fma((double)acc[(b * A.L + l) * kAccPitch + slot], P[l * nv], lq);
            for (int j = 1; j < nv; ++j) {
                double lc = 0.0;
                for (int l = 0; l < A.L; ++l)
                    lc = fma((double)acc[(b * A.L + l) * kAccPitch + slot], P[l * nv + j], lc);
                best = np_minimum(best, sigmoid2(lq - lc));
            }
            A.relevancy_raw[(size_t)b * A.W * A.H + (size_t)py * A.W + px] = best;
        }
    }
}

// Relevancy from a coefficient map in HBM (used when the channel count does
// not fit one blend CTA).  One thread per pixel.
__global__ void k_relevancy_from_cmap(int64_t P, int n_ch, const float* __restrict__ cmap,
                                      const double* __restrict__ proj_cb, int n_levels, int L,
                                      int n_canon, double* __restrict__ out) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int nv = 1 + n_canon;
    const float* w = cmap + (size_t)p * n_ch;
    for (int b = 0; b < n_levels; ++b) {
        const double* Pm = proj_cb + (size_t)b * L * nv;
        double lq = 0.0;
        for (int l = 0; l < L; ++l) lq = fma((double)w[b * L + l], Pm[l * nv], lq);
        double best = INFINITY;
        for (int j = 1; j < nv; ++j) {
            double lc = 0.0;
            for (int l = 0; l < L; ++l) lc = fma((double)w[b * L + l], Pm[l * nv + j], lc);
            best = np_minimum(best, sigmoid2(lq - lc));
        }
        out[(size_t)b * P + p] = best;
    }
}

int launch_blend(const BlendArgs& a, cudaStream_t st) {
    if (a.C > kMaxC) return -2;
    int n_tiles = a.tiles_x * a.tiles_y;
    int ch_block = a.n_ch < kChBlock ? a.n_ch : kChBlock;
    int nblk = (a.n_ch + ch_block - 1) / ch_block;
    size_t smem = sizeof(BlendSmem) + (size_t)ch_block * kAccPitch * sizeof(float);
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(k_blend, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    if (n_tiles > 0) k_blend<<<dim3(n_tiles, nblk), kBlendThreads, smem, st>>>(a, ch_block);
    if (a.proj_cb && nblk > 1) {
        int64_t P = (int64_t)a.W * a.H;
        k_relevancy_from_cmap<<<ceil_div(P, 256), 256, 0, st>>>(P, a.n_ch, a.coeff_map, a.proj_cb,
                                                               a.n_levels, a.L, a.n_canon,
                                                               a.relevancy_raw);
    }
    return 0;
}

}  // namespace sf
