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
// a warp stays small.  The tile's depth-ordered list streams through shared
// memory in batches of 32 Gaussian records (80 B geometry + scatter plan),
// double-buffered with cp.async so the next batch's L2/HBM gathers overlap
// the current batch's math.  Per batch:
//   phase A  every thread runs the q > 9 rejection in fp32 for all 32
//            Gaussians (independent work, high ILP) with a conservative
//            guard band (|q32 - q64| <= 1.5e-6 S, guard 1e-4 (1 + S),
//            S = a dx^2 + c dy^2) -> a 32-bit candidate mask;
//   phase B  the warp walks the union of its candidate masks in depth order;
//            candidates are re-evaluated in fp64 with the reference's exact
//            op order (bit-exact q <= 9 membership), alpha = o exp(-q/2) via
//            a 1/128-step table times a degree-5 polynomial (~1e-16 rel.),
//            and T / e carried in fp64, so the T >= 1e-4 early-exit decision
//            matches the fp64 reference.
// The coefficient accumulator is fp32 in shared memory, acc[channel][slot]
// with a 257-float pitch: the K channel ids of a Gaussian are warp-uniform,
// so every scatter is one conflict-free wavefront, and the transposed read
// for the channel-contiguous HBM write is conflict-free too.  A warp skips
// a Gaussian's scatter unless some lane has e > 0 (__any_sync), skips whole
// batches once all its pixels saturated, and the CTA stops streaming when
// every pixel is saturated (__syncthreads_and).
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
constexpr int kMaxC = 16;            // channels per Gaussian (levels*K) supported
constexpr int kMaxChanRec = 96;      // chan_rec_bytes(16)
constexpr int kChBlock = 192;        // accumulator channels per CTA (smem bound)
constexpr int kExpSteps = 128;       // exp table resolution in y = q / 2
constexpr int kExpTable = 577;       // y in [0, 4.5]

__constant__ double c_exp_table[kExpTable];

struct __align__(16) BlendStage {
    GeomRec g[kBatch];
    unsigned char chan[kBatch * kMaxChanRec];
    uint32_t off[kBatch][kMaxC];
};

struct __align__(16) BlendSmem {
    BlendStage st[2];
    double exp_tab[kExpTable + 1];
};

__device__ __forceinline__ double sigmoid2(double x) {
    if (x >= 0) return 1.0 / (1.0 + exp(-x));
    double ex = exp(x);
    return ex / (1.0 + ex);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// exp(-y) for y in [0, 4.5]: table at k/128 times a degree-5 Taylor
// polynomial on f in [0, 1/128) (truncation < 3.2e-16 relative).
__device__ __forceinline__ double exp_neg(double y, const double* tab) {
    int k = (int)(y * (double)kExpSteps);  // exact scaling, truncation = floor (y >= 0)
    double f = fma(-(double)k, 1.0 / kExpSteps, y);  // exact: y - k/128
    double p = fma(f, -1.0 / 120.0, 1.0 / 24.0);
    p = fma(p, f, -1.0 / 6.0);
    p = fma(p, f, 0.5);
    p = fma(p, f, -1.0);
    p = fma(p, f, 1.0);
    return tab[k] * p;
}

// Issue the cp.async copies of one batch (nb records) into stage buffer S.
__device__ __forceinline__ void stage_batch(BlendStage& S, const BlendArgs& A, uint32_t base, int nb, int cs) {
    const int gchunks = (int)(sizeof(GeomRec) / 16);  // 5
    const int cchunks = cs / 16;
    const int per = gchunks + cchunks;
    for (int idx = threadIdx.x; idx < nb * per; idx += kBlendThreads) {
        int j = idx / per, c = idx - j * per;
        uint32_t r = __ldg(A.entries + base + j);
        if (c < gchunks) {
            cp_async16(reinterpret_cast<char*>(&S.g[j]) + 16 * c,
                       reinterpret_cast<const char*>(A.geom + r) + 16 * c);
        } else {
            c -= gchunks;
            cp_async16(S.chan + j * kMaxChanRec + 16 * c, A.chan + (size_t)r * cs + 16 * c);
        }
    }
}

// CT: channels per Gaussian (0 = runtime), SINGLE: one channel block,
// NV: fused relevancy vectors (0 = none, -1 = runtime count).
template <int CT, bool SINGLE, int NV>
__global__ void __launch_bounds__(kBlendThreads, 1) k_blend(BlendArgs A, int ch_block) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BlendSmem& S = *reinterpret_cast<BlendSmem*>(smem_raw);
    float* acc = reinterpret_cast<float*>(smem_raw + sizeof(BlendSmem));

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
    const int C = CT > 0 ? CT : A.C;
    const int cs = chan_rec_bytes(C);
    const int voff = chan_val_offset(C);

    const uint32_t beg = A.tile_offsets[tile], end = A.tile_offsets[tile + 1];
    if (beg < end) stage_batch(S.st[0], A, beg, (int)min((uint32_t)kBatch, end - beg), cs);
    cp_async_commit();
    for (int i = threadIdx.x; i < kExpTable; i += kBlendThreads) S.exp_tab[i] = c_exp_table[i];
    for (int i = threadIdx.x; i < nchb * kAccPitch; i += kBlendThreads) acc[i] = 0.f;

    const float pxf = (float)px, pyf = (float)py;
    const double pxd = (double)px, pyd = (double)py;
    double T = 1.0;
    bool done = !inside;

    int bi = 0;
    for (uint32_t base = beg; base < end; base += kBatch, ++bi) {
        const int nb = (int)min((uint32_t)kBatch, end - base);
        BlendStage& B = S.st[bi & 1];
        // prefetch the next batch into the other buffer (freed by the previous iteration's barrier)
        const uint32_t nbase = base + kBatch;
        if (nbase < end) stage_batch(S.st[(bi + 1) & 1], A, nbase, (int)min((uint32_t)kBatch, end - nbase), cs);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        // channel ids -> accumulator offsets for this CTA's channel block
        for (int idx = threadIdx.x; idx < nb * C; idx += kBlendThreads) {
            int j = idx / C, k = idx - j * C;
            int ch = (int)reinterpret_cast<const uint16_t*>(B.chan + j * kMaxChanRec)[k] - ch0;
            B.off[j][k] = ((unsigned)ch < (unsigned)nchb) ? (uint32_t)(ch * kAccPitch * 4) : 0xffffffffu;
        }
        __syncthreads();

        if (!__all_sync(0xffffffffu, done)) {
            // ---- phase A: fp32 rejection, candidate mask ----
            uint32_t cand = 0;
            if (!done) {
#pragma unroll 4
                for (int j = 0; j < nb; ++j) {
                    const float4 m4 = *reinterpret_cast<const float4*>(&B.g[j].mx_hi);
                    const float4 c4 = *reinterpret_cast<const float4*>(&B.g[j].a);
                    float dx = (pxf - m4.x) - m4.y;
                    float dy = (pyf - m4.z) - m4.w;
                    float adx = c4.x * dx, cdy = c4.z * dy;
                    float q32 = fmaf(adx, dx, fmaf(c4.y * dx, dy, cdy * dy));
                    float s32 = fmaf(adx, dx, cdy * dy);
                    if (q32 <= fmaf(1e-4f, s32, 9.0001f)) cand |= 1u << j;
                }
            }
            // ---- phase B: exact evaluation + scatter, depth order ----
            uint32_t wmask = __reduce_or_sync(0xffffffffu, cand);
            while (wmask) {
                const int j = __ffs(wmask) - 1;
                wmask &= wmask - 1;
                float ef = 0.f;
                if (((cand >> j) & 1u) && !done) {
                    const GeomRec& g = B.g[j];
                    double ddx = __dadd_rn(pxd, -g.mx), ddy = __dadd_rn(pyd, -g.my);
                    double t1 = __dmul_rn(__dmul_rn(g.a64, ddx), ddx);
                    double t2 = __dmul_rn(__dmul_rn(__dmul_rn(2.0, g.b64), ddx), ddy);
                    double t3 = __dmul_rn(__dmul_rn(g.c64, ddy), ddy);
                    double q = __dadd_rn(__dadd_rn(t1, t2), t3);
                    if (q <= SF_CUTOFF) {
                        double al = __dmul_rn((double)g.opacity, exp_neg(__dmul_rn(0.5, q), S.exp_tab));
                        al = np_minimum(al, SF_ALPHA_CLAMP);
                        double e = __dmul_rn(al, T);
                        T = __dmul_rn(T, __dadd_rn(1.0, -al));
                        ef = (float)e;
                        if (A.early_exit && T < SF_EARLY_EXIT_T) done = true;
                    }
                }
                if (__any_sync(0xffffffffu, ef > 0.f)) {
                    const float* val = reinterpret_cast<const float*>(B.chan + j * kMaxChanRec + voff);
                    char* accs = reinterpret_cast<char*>(acc + slot);
                    if (CT > 0 && CT % 4 == 0) {
                        const uint4* o4 = reinterpret_cast<const uint4*>(B.off[j]);
                        const float4* v4 = reinterpret_cast<const float4*>(val);
#pragma unroll
                        for (int q = 0; q < (CT > 0 ? CT : 4) / 4; ++q) {
                            const uint4 o = o4[q];
                            const float4 v = v4[q];
                            const uint32_t oo[4] = {o.x, o.y, o.z, o.w};
                            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                if (SINGLE || oo[e] != 0xffffffffu) {
                                    float* a = reinterpret_cast<float*>(accs + oo[e]);
                                    *a = fmaf(ef, vv[e], *a);
                                }
                            }
                        }
                    } else {
                        for (int k = 0; k < C; ++k) {
                            const uint32_t off = B.off[j][k];
                            if (off != 0xffffffffu) {
                                float* a = reinterpret_cast<float*>(accs + off);
                                *a = fmaf(ef, val[k], *a);
                            }
                        }
                    }
                }
            }
        }
        if (__syncthreads_and(done)) break;
    }
    cp_async_wait<0>();
    __syncthreads();

    // ---- outputs ----
    if (blockIdx.y == 0 && A.final_t && inside) A.final_t[(size_t)py * A.W + px] = (float)T;
    if (A.coeff_map) {
        // warp w writes pixels x = w, w + 8 of every tile row; lanes stride the
        // pixel's channels (contiguous in HBM), the smem read is conflict-free
        const int tw = min(SF_TILE, A.W - x0), th = min(SF_TILE, A.H - y0);
        for (int r = 0; r < th; ++r) {
            const int wr = (r >> 2) * 2, lr = (r & 3) * 8;
            for (int x = warp; x < tw; x += kBlendThreads / 32) {
                const int sl = (wr + (x >> 3)) * 32 + lr + (x & 7);
                float* dst = A.coeff_map + ((size_t)(y0 + r) * A.W + x0 + x) * A.n_ch + ch0;
                for (int ch = lane; ch < nchb; ch += 32) __stcs(dst + ch, acc[ch * kAccPitch + sl]);
            }
        }
    }
    if (NV != 0 && A.proj_cb && nchb == A.n_ch) {
        // fused relevancy: logits_j = sum_l W[l] * P[b][l][j] in fp64; the
        // projected codebook is staged in the idle batch buffers
        const int nv = NV > 0 ? NV : 1 + A.n_canon;
        const int np = A.n_levels * A.L * nv;
        double* Ps = reinterpret_cast<double*>(&S.st[0]);
        const bool fits = np * (int)sizeof(double) <= (int)sizeof(S.st);
        if (fits) {
            for (int i = threadIdx.x; i < np; i += kBlendThreads) Ps[i] = A.proj_cb[i];
            __syncthreads();
        }
        if (inside) {
            for (int b = 0; b < A.n_levels; ++b) {
                double best = INFINITY;
                if (NV > 0 && fits) {
                    const double* P = Ps + (size_t)b * A.L * nv;
                    double lg[NV > 0 ? NV : 1];
#pragma unroll
                    for (int t = 0; t < (NV > 0 ? NV : 1); ++t) lg[t] = 0.0;
                    for (int l = 0; l < A.L; ++l) {
                        const double w = (double)acc[(b * A.L + l) * kAccPitch + slot];
#pragma unroll
                        for (int t = 0; t < (NV > 0 ? NV : 1); ++t) lg[t] = fma(w, P[l * (NV > 0 ? NV : 1) + t], lg[t]);
                    }
#pragma unroll
                    for (int t = 1; t < (NV > 0 ? NV : 1); ++t) best = np_minimum(best, sigmoid2(lg[0] - lg[t]));
                } else {
                    const double* P = (fits ? Ps : A.proj_cb) + (size_t)b * A.L * nv;
                    double lq = 0.0;
                    for (int l = 0; l < A.L; ++l) lq = fma((double)acc[(b * A.L + l) * kAccPitch + slot], P[l * nv], lq);
                    for (int j = 1; j < nv; ++j) {
                        double lc = 0.0;
                        for (int l = 0; l < A.L; ++l)
                            lc = fma((double)acc[(b * A.L + l) * kAccPitch + slot], P[l * nv + j], lc);
                        best = np_minimum(best, sigmoid2(lq - lc));
                    }
                }
                A.relevancy_raw[(size_t)b * A.W * A.H + (size_t)py * A.W + px] = best;
            }
        }
    }
}

// Relevancy from a coefficient map in HBM (the map is written anyway when the
// features are decoded, or the channel count exceeds one blend CTA).  One
// thread per pixel; the projected codebook sits in shared memory.
template <int NV>
__global__ void __launch_bounds__(256) k_relevancy_from_cmap(int64_t P, int n_ch, const float* __restrict__ cmap,
                                                             const double* __restrict__ proj_cb, int n_levels,
                                                             int L, int n_canon, double* __restrict__ out) {
    extern __shared__ double Ps[];
    const int nv = NV > 0 ? NV : 1 + n_canon;
    for (int i = threadIdx.x; i < n_levels * L * nv; i += blockDim.x) Ps[i] = proj_cb[i];
    __syncthreads();
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const float* w = cmap + (size_t)p * n_ch;
    for (int b = 0; b < n_levels; ++b) {
        const double* Pm = Ps + (size_t)b * L * nv;
        double best = INFINITY;
        if (NV > 0) {
            double lg[NV > 0 ? NV : 1];
#pragma unroll
            for (int t = 0; t < (NV > 0 ? NV : 1); ++t) lg[t] = 0.0;
            for (int l0 = 0; l0 < L; l0 += 4) {
                const float4 w4 = __ldcs(reinterpret_cast<const float4*>(w + b * L + l0));
                const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const double wd = (double)wv[e];
#pragma unroll
                    for (int t = 0; t < (NV > 0 ? NV : 1); ++t) lg[t] = fma(wd, Pm[(l0 + e) * (NV > 0 ? NV : 1) + t], lg[t]);
                }
            }
#pragma unroll
            for (int t = 1; t < (NV > 0 ? NV : 1); ++t) best = np_minimum(best, sigmoid2(lg[0] - lg[t]));
        } else {
            double lq = 0.0;
            for (int l = 0; l < L; ++l) lq = fma((double)w[b * L + l], Pm[l * nv], lq);
            for (int j = 1; j < nv; ++j) {
                double lc = 0.0;
                for (int l = 0; l < L; ++l) lc = fma((double)w[b * L + l], Pm[l * nv + j], lc);
                best = np_minimum(best, sigmoid2(lq - lc));
            }
        }
        out[(size_t)b * P + p] = best;
    }
}

void launch_relevancy_from_cmap(int64_t P, int n_ch, const float* cmap, const double* proj_cb, int n_levels,
                                int L, int n_canon, double* out, cudaStream_t st) {
    if (P == 0) return;
    const size_t smem = sizeof(double) * (size_t)n_levels * L * (1 + n_canon);
    const bool vec = (L % 4 == 0) && (n_ch % 4 == 0) && ((uintptr_t)cmap % 16 == 0);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_relevancy_from_cmap<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_relevancy_from_cmap<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = true;
    }
    if (vec && n_canon == 4)
        k_relevancy_from_cmap<5><<<ceil_div(P, 256), 256, smem, st>>>(P, n_ch, cmap, proj_cb, n_levels, L, n_canon, out);
    else
        k_relevancy_from_cmap<0><<<ceil_div(P, 256), 256, smem, st>>>(P, n_ch, cmap, proj_cb, n_levels, L, n_canon, out);
}

static bool init_exp_table() {
    static bool done = false;
    if (done) return true;
    double h[kExpTable];
    for (int k = 0; k < kExpTable; ++k) h[k] = exp(-(double)k / kExpSteps);
    if (cudaMemcpyToSymbol(c_exp_table, h, sizeof(h)) != cudaSuccess) return false;
    done = true;
    return true;
}

int launch_blend(const BlendArgs& a, cudaStream_t st) {
    if (a.C > kMaxC) return -2;
    if (!init_exp_table()) return -3;
    int n_tiles = a.tiles_x * a.tiles_y;
    int ch_block = a.n_ch < kChBlock ? a.n_ch : kChBlock;
    int nblk = (a.n_ch + ch_block - 1) / ch_block;
    size_t smem = sizeof(BlendSmem) + (size_t)ch_block * kAccPitch * sizeof(float);
    const bool fast = (a.C == 12 && nblk == 1);
    const int nv = a.proj_cb ? 1 + a.n_canon : 0;
    void (*kern)(BlendArgs, int);
    int ki;
    if (fast && nv == 0) { kern = k_blend<12, true, 0>; ki = 0; }
    else if (fast && nv == 5) { kern = k_blend<12, true, 5>; ki = 1; }
    else if (fast) { kern = k_blend<12, true, -1>; ki = 2; }
    else { kern = k_blend<0, false, -1>; ki = 3; }
    static size_t configured[4] = {0, 0, 0, 0};
    if (smem > configured[ki]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured[ki] = smem;
    }
    if (n_tiles > 0) kern<<<dim3(n_tiles, nblk), kBlendThreads, smem, st>>>(a, ch_block);
    if (a.proj_cb && nblk > 1)
        launch_relevancy_from_cmap((int64_t)a.W * a.H, a.n_ch, a.coeff_map, a.proj_cb, a.n_levels, a.L,
                                   a.n_canon, a.relevancy_raw, st);
    return 0;
}

}  // namespace sf
