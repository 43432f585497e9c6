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
#include <algorithm>

#include "sf_common.cuh"

namespace sf {

// One CTA per half tile (16x8 pixels = 4 warp patches of 8x4): ~110 KB of
// shared memory, so two CTAs share an SM and one's list start-up and
// epilogue overlap the other's blending.
constexpr int kBlendThreads = 128;  // consumer threads: one per pixel
constexpr int kConsumerWarps = kBlendThreads / 32;
constexpr int kCTAThreads = kBlendThreads + 32;  // + one producer warp
constexpr int kTilePixels = 128;    // pixels per CTA (half a 16x16 tile)
constexpr int kStages = 2;          // batch ring between the producer and the consumer warps
constexpr int kBatch = 32;
constexpr int kAccPitch = 129;
constexpr int kMaxC = 16;            // channels per Gaussian (levels*K) supported
constexpr int kMaxChanRec = 96;      // chan_rec_bytes(16)
constexpr int kChBlock = 192;        // accumulator channels per CTA (smem bound)

struct __align__(16) BlendStage {
    GeomRec g[kBatch];
    unsigned char chan[kBatch * kMaxChanRec];
    uint32_t off[kBatch][kMaxC];
};

struct __align__(16) BlendSmem {
    BlendStage st[kStages];
    uint64_t full[kStages];   // producer -> consumers: batch staged (count 1)
    uint64_t empty[kStages];  // consumers -> producer: batch consumed (one arrival per consumer warp)
    int nb[kStages];          // batch size; 0 = end of the tile's stream
    int n_done_warps;         // consumer warps whose pixels all saturated
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

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

// Issue the cp.async copies of one batch (nb records) into stage buffer S
// (called by the 32 lanes of the producer warp).
__device__ __forceinline__ void stage_batch(BlendStage& S, const BlendArgs& A, uint32_t base, int nb, int cs) {
    const int gchunks = (int)(sizeof(GeomRec) / 16);  // 5
    const int cchunks = cs / 16;
    const int per = gchunks + cchunks;
    for (int idx = (int)(threadIdx.x & 31); idx < nb * per; idx += 32) {
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

// alpha = min(o exp(-q/2), 0.99) with q <= 9 membership (0 if outside).
// q is evaluated in fp32 as a (dx + k dy)^2 + d dy^2 (no cancellation); inside
// the guard band around 9 the reference's fp64 q decides (rasterizer.py:161-168).
__device__ __forceinline__ float blend_alpha(const GeomRec& g, float pxf, float pyf, double pxd, double pyd) {
    constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // -0.5 / ln 2
    const float dx = (pxf - g.mx_hi) - g.mx_lo;
    const float dy = (pyf - g.my_hi) - g.my_lo;
    const float u = fmaf(g.k, dy, dx);
    const float ddy = g.d * dy * dy;
    float q32 = fmaf(g.a * u, u, ddy);
    const float su = fabsf(dx) + fabsf(g.k * dy);
    const float guard = fmaf(1e-5f, fmaf(g.a * su, su, ddy), 1e-5f);
    if (q32 > 9.f + guard) return 0.f;
    if (q32 > 9.f - guard) {
        double ddx = __dadd_rn(pxd, -g.mx), ddyd = __dadd_rn(pyd, -g.my);
        double t1 = __dmul_rn(__dmul_rn(g.a64, ddx), ddx);
        double t2 = __dmul_rn(__dmul_rn(__dmul_rn(2.0, g.b64), ddx), ddyd);
        double t3 = __dmul_rn(__dmul_rn(g.c64, ddyd), ddyd);
        double q = __dadd_rn(__dadd_rn(t1, t2), t3);
        if (!(q <= SF_CUTOFF)) return 0.f;
        q32 = (float)q;
    }
    return fminf(g.opacity * exp2f(kNegHalfLog2e * q32), 0.99f);
}

// Conservative patch culling: may any pixel of the 8x4 patch with corner
// (x0, y0) have q <= 9?  q = a (dx + k dy)^2 + d dy^2 is convex, so its
// minimum over the pixel-centre rectangle is 0 when the mean lies inside,
// else on one of the four edges (1-D minimisation with clamping).  fp32 with
// the same relative guard as blend_alpha; false positives only cost work,
// blend_alpha still decides every pixel (exactly, inside the guard band).
__device__ __forceinline__ bool patch_may_hit(const GeomRec& g, float x0, float y0) {
    const float dx0 = (x0 - g.mx_hi) - g.mx_lo, dx1 = dx0 + 7.f;
    const float dy0 = (y0 - g.my_hi) - g.my_lo, dy1 = dy0 + 3.f;
    if (dx0 <= 0.f && dx1 >= 0.f && dy0 <= 0.f && dy1 >= 0.f) return true;
    const float a = g.a, k = g.k, d = g.d;
    const float c = fmaf(a * k, k, d);
    const float s = -(a * k) / c;  // dy* = s * dx on an x edge
    float best = INFINITY, bs = 0.f;
    auto eval = [&](float dx, float dy) {
        const float u = fmaf(k, dy, dx);
        const float q = fmaf(a * u, u, d * dy * dy);
        if (q < best) {
            best = q;
            const float su = fabsf(dx) + fabsf(k * dy);
            bs = fmaf(a * su, su, d * dy * dy);
        }
    };
    eval(dx0, fminf(fmaxf(s * dx0, dy0), dy1));
    eval(dx1, fminf(fmaxf(s * dx1, dy0), dy1));
    eval(fminf(fmaxf(-k * dy0, dx0), dx1), dy0);
    eval(fminf(fmaxf(-k * dy1, dx0), dx1), dy1);
    return best <= 9.f + fmaf(1e-4f, bs, 1e-4f);
}

// CT: channels per Gaussian (0 = runtime), SINGLE: one channel block,
// NC: canonical phrases of the fused relevancy (0 = none, -1 = runtime count).
template <int CT, bool SINGLE, int NC>
__global__ void __launch_bounds__(kCTAThreads, 2) k_blend(BlendArgs A, int ch_block) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BlendSmem& S = *reinterpret_cast<BlendSmem*>(smem_raw);
    float* acc = reinterpret_cast<float*>(smem_raw + sizeof(BlendSmem));

    if (A.stats[SF_STAT_OVERFLOW]) return;
    const int tile = A.tile0 + (blockIdx.x >> 1), half = blockIdx.x & 1;
    const int ch0 = blockIdx.y * ch_block;
    const int nchb = min(ch_block, A.n_ch - ch0);
    const int tx = tile % A.tiles_x, ty = tile / A.tiles_x;
    const int x0 = tx * SF_TILE, y0 = ty * SF_TILE;
    const int slot = threadIdx.x & (kTilePixels - 1);  // pixel slot within the CTA
    const int lane = slot & 31;
    const int cw = threadIdx.x >> 5;                  // warp index within the CTA
    const int warp = half * kConsumerWarps + (slot >> 5);  // patch index within the tile (0..7)
    const int lx = (warp & 1) * 8 + (lane & 7);
    const int ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = x0 + lx, py = y0 + ly;
    const bool inside = (threadIdx.x < kBlendThreads) && (px < A.W) && (py < A.H);
    const int C = CT > 0 ? CT : A.C;
    const int cs = chan_rec_bytes(C);
    const int voff = chan_val_offset(C);

    const uint32_t beg = A.tile_offsets[tile], end = A.tile_offsets[tile + 1];
    const bool consumer = threadIdx.x < kBlendThreads;
    if (threadIdx.x == 0) {
        for (int st = 0; st < kStages; ++st) {
            bar_init(&S.full[st], 1);
            bar_init(&S.empty[st], kConsumerWarps);
        }
        S.n_done_warps = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < nchb * kAccPitch; i += kCTAThreads) acc[i] = 0.f;
    __syncthreads();

    const float pxf = (float)px, pyf = (float)py;
    const float pdx0 = (float)(x0 + (warp & 1) * 8), pdy0 = (float)(y0 + (warp >> 1) * 4);  // patch corner
    const double pxd = (double)px, pyd = (double)py;
    float T = 1.f;        // transmittance (fp32: |dT|/T <= eb * 3e-6 + n * 1.2e-7, see header)
    float eb = 0.f;       // sum of alpha / (1 - alpha) over contributions (error-bound driver)
    float Tprev = 1.f;    // T before the last contribution
    int ncontrib = 0;
    bool done = !inside;

    if (!consumer) {
        // ---------------- producer warp: stream the tile's list through the ring ----------------
        const int pl = threadIdx.x & 31;
        for (int bi = 0;; ++bi) {
            const int st = bi % kStages;
            if (bi >= kStages) bar_wait(&S.empty[st], ((bi / kStages) - 1) & 1);
            const uint32_t base = beg + (uint32_t)bi * kBatch;
            const bool all_done = *reinterpret_cast<volatile int*>(&S.n_done_warps) == kConsumerWarps;
            const int nb = (base < end && !all_done) ? (int)min((uint32_t)kBatch, end - base) : 0;
            BlendStage& B = S.st[st];
            if (nb) {
                stage_batch(B, A, base, nb, cs);
                cp_async_commit();
                cp_async_wait<0>();
                __syncwarp();
                // channel ids -> accumulator byte offsets for this CTA's channel block
                for (int idx = pl; idx < nb * C; idx += 32) {
                    int j = idx / C, k = idx - j * C;
                    int ch = (int)reinterpret_cast<const uint16_t*>(B.chan + j * kMaxChanRec)[k] - ch0;
                    B.off[j][k] = ((unsigned)ch < (unsigned)nchb) ? (uint32_t)(ch * kAccPitch * 4) : 0xffffffffu;
                }
                __syncwarp();
            }
            if (pl == 0) {
                S.nb[st] = nb;
                bar_arrive(&S.full[st]);
            }
            if (nb == 0) break;
        }
    } else {
        // ---------------- consumer warps: progress independently through the ring ----------------
        bool warp_done = __all_sync(0xffffffffu, done);
        if (warp_done && lane == 0) atomicAdd(&S.n_done_warps, 1);
        for (int bi = 0;; ++bi) {
            const int st = bi % kStages;
            bar_wait(&S.full[st], (bi / kStages) & 1);
            const int nb = *reinterpret_cast<volatile int*>(&S.nb[st]);
            if (nb == 0) break;
            BlendStage& B = S.st[st];
            if (!warp_done) {
            // ---- phase A: lane j tests record j against the warp's 8x4 patch ----
            // (conservative fp32 minimum of q over the patch rectangle, see patch_may_hit)
            const uint32_t wcand = __ballot_sync(0xffffffffu, lane < nb && patch_may_hit(B.g[lane], pdx0, pdy0));
            // ---- phase B: alpha, transmittance, scatter -- depth order ----
            // alpha of the next candidate is computed before the current scatter
            // (it depends only on geometry), so its latency hides under the
            // scatter's shared-memory traffic.
            uint32_t wmask = wcand;
            int j = wmask ? __ffs(wmask) - 1 : -1;
            if (j >= 0) wmask &= wmask - 1;
            float al = (j >= 0 && !done) ? blend_alpha(B.g[j], pxf, pyf, pxd, pyd) : 0.f;
            while (j >= 0) {
                float ef = 0.f;
                if (al > 0.f && !done) {
                    ef = al * T;
                    Tprev = T;
                    T = fmaf(-al, T, T);
                    eb = fmaf(al, rcp_approx(1.f - al), eb);  // 1 - al in [0.01, 1]: no denormals
                    ++ncontrib;
                    if (A.early_exit && T < (float)SF_EARLY_EXIT_T) done = true;
                }
                const int jn = wmask ? __ffs(wmask) - 1 : -1;
                if (jn >= 0) wmask &= wmask - 1;
                const float aln = (jn >= 0 && !done) ? blend_alpha(B.g[jn], pxf, pyf, pxd, pyd) : 0.f;
                if (__any_sync(0xffffffffu, ef > 0.f)) {
                    const float* val = reinterpret_cast<const float*>(B.chan + j * kMaxChanRec + voff);
                    char* accs = reinterpret_cast<char*>(acc + slot);
                    if (CT > 0 && CT % 4 == 0 && SINGLE) {
                        // a Gaussian's channel ids are distinct: all loads, then FMAs, then stores
                        constexpr int NH = CT > 0 ? CT : 4;
                        const uint4* oh = reinterpret_cast<const uint4*>(B.off[j]);
                        const float4* vh = reinterpret_cast<const float4*>(val);
                        uint32_t oo[NH];
                        float vv[NH], av[NH];
#pragma unroll
                        for (int e = 0; e < NH / 4; ++e) {
                            const uint4 o4 = oh[e];
                            const float4 v4 = vh[e];
                            oo[4 * e] = o4.x, oo[4 * e + 1] = o4.y, oo[4 * e + 2] = o4.z, oo[4 * e + 3] = o4.w;
                            vv[4 * e] = v4.x, vv[4 * e + 1] = v4.y, vv[4 * e + 2] = v4.z, vv[4 * e + 3] = v4.w;
                        }
#pragma unroll
                        for (int e = 0; e < NH; ++e) av[e] = *reinterpret_cast<const float*>(accs + oo[e]);
#pragma unroll
                        for (int e = 0; e < NH; ++e) av[e] = fmaf(ef, vv[e], av[e]);
#pragma unroll
                        for (int e = 0; e < NH; ++e) *reinterpret_cast<float*>(accs + oo[e]) = av[e];
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
                j = jn;
                al = aln;
            }
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&S.empty[st]);
            if (!warp_done && __all_sync(0xffffffffu, done)) {
                warp_done = true;
                if (lane == 0) atomicAdd(&S.n_done_warps, 1);
            }
        }
    }
    __syncthreads();

    // Early-exit decisions (counted iff T >= 1e-4) that fp32 T cannot certify
    // are replayed exactly in fp64 by k_blend_fixup.
    if (inside && A.early_exit && A.fixup_list && blockIdx.y == 0) {
        const float tol = fmaf(4e-6f, eb, fmaf(3e-7f, (float)ncontrib, 2e-6f));
        const float thr = (float)SF_EARLY_EXIT_T;
        const bool amb = done ? (Tprev < thr * (1.f + tol) || T > thr * (1.f - tol)) : (T < thr * (1.f + tol));
        if (amb) {
            uint32_t k = atomicAdd(A.fixup_count, 1u);
            if (k < A.fixup_capacity) A.fixup_list[k] = ((uint32_t)tile << 8) | (uint32_t)(half * kTilePixels + slot);
        }
    }
    // ---- outputs ----
    if (blockIdx.y == 0 && A.final_t && inside) A.final_t[(size_t)py * A.W + px] = T;
    if (A.coeff_map) {
        // Each warp instruction writes 4 pixels x 32 channels as float4:
        // lane = (pixel p = lane / 8, channel quad q = lane % 8); the four
        // scalar smem reads hit bank (4q + e + slot) mod 32 -- conflict-free
        // with the 129-word pitch -- and the 16-byte stores of a pixel form
        // one 128-byte line.  Slots past the image edge are skipped.
        const int q = lane & 7, pl = lane >> 3;
        const bool vec = (nchb % 32 == 0) && (A.n_ch % 4 == 0) && (ch0 % 4 == 0) &&
                         ((reinterpret_cast<uintptr_t>(A.coeff_map) & 15) == 0);
        for (int sg = cw * 4; sg < kTilePixels; sg += 4 * kConsumerWarps) {
            const int sl = sg + pl;                      // this lane's pixel slot
            const int w8 = half * kConsumerWarps + (sl >> 5), l8 = sl & 31;
            const int gx = x0 + (w8 & 1) * 8 + (l8 & 7), gy = y0 + (w8 >> 1) * 4 + (l8 >> 3);
            const bool ok = gx < A.W && gy < A.H;
            float* dst = A.coeff_map + ((size_t)gy * A.W + gx) * A.n_ch + ch0;
            if (vec) {
                for (int c0 = 0; c0 < nchb; c0 += 32) {
                    const int c = c0 + 4 * q;
                    const float* src = acc + c * kAccPitch + sl;
                    const float4 v = make_float4(src[0], src[kAccPitch], src[2 * kAccPitch], src[3 * kAccPitch]);
                    if (ok) __stcs(reinterpret_cast<float4*>(dst + c), v);
                }
            } else if (ok) {
                for (int c = q; c < nchb; c += 8) __stcs(dst + c, acc[c * kAccPitch + sl]);
            }
        }
    }
    if (NC != 0 && A.proj_cb && nchb == A.n_ch) {
        // fused relevancy (query.py:65-84): l_q - l_j = W . Pd_j with the
        // logit-difference vectors Pd_j = P_q - P_cj of the projected codebook
        // P = atoms @ [q; c]^T, fp64, staged in the idle batch buffers
        const int nc = NC > 0 ? NC : A.n_canon;
        const int nv = 1 + A.n_canon;
        const int np = A.n_levels * A.L * nc;
        double* Pd = reinterpret_cast<double*>(&S.st[0]);
        const bool fits = np * (int)sizeof(double) <= (int)sizeof(S.st);
        if (fits) {
            for (int i = threadIdx.x; i < np; i += kCTAThreads) {
                const int j = i % nc, bl = i / nc;
                Pd[i] = A.proj_cb[(size_t)bl * nv] - A.proj_cb[(size_t)bl * nv + 1 + j];
            }
            __syncthreads();
        }
        if (inside) {
            for (int b = 0; b < A.n_levels; ++b) {
                double best = INFINITY;
                const float* wb = acc + (b * A.L) * kAccPitch + slot;
                if (NC == 4 && fits) {
                    const double* Pb = Pd + (size_t)b * A.L * 4;
                    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll 4
                    for (int l = 0; l < A.L; ++l) {
                        const double w = (double)wb[l * kAccPitch];
                        const double2 p01 = *reinterpret_cast<const double2*>(Pb + 4 * l);
                        const double2 p23 = *reinterpret_cast<const double2*>(Pb + 4 * l + 2);
                        d0 = fma(w, p01.x, d0);
                        d1 = fma(w, p01.y, d1);
                        d2 = fma(w, p23.x, d2);
                        d3 = fma(w, p23.y, d3);
                    }
                    // sigmoid is monotone: min_j sigmoid(d_j) = sigmoid(min_j d_j)
                    best = sigmoid2(np_minimum(np_minimum(d0, d1), np_minimum(d2, d3)));
                } else {
                    for (int j = 0; j < nc; ++j) {
                        double dj = 0.0;
                        for (int l = 0; l < A.L; ++l) {
                            const double pd = fits ? Pd[((size_t)b * A.L + l) * nc + j]
                                                   : A.proj_cb[((size_t)b * A.L + l) * nv] -
                                                         A.proj_cb[((size_t)b * A.L + l) * nv + 1 + j];
                            dj = fma((double)wb[l * kAccPitch], pd, dj);
                        }
                        best = np_minimum(best, sigmoid2(dj));
                    }
                }
                A.relevancy_raw[(size_t)b * A.W * A.H + (size_t)py * A.W + px] = best;
            }
        }
    }
}

// Relevancy from a coefficient map in HBM (the map is written anyway when the
// features are decoded, or the channel count exceeds one blend CTA).  One
// thread per pixel; shared memory holds the logit-difference vectors
// Pd_j = P_q - P_cj (so l_q - l_j = W . Pd_j: nc dot products instead of
// nc + 1), read as 16-byte broadcasts.
template <int NC>
__global__ void __launch_bounds__(256) k_relevancy_from_cmap(int64_t P, int n_ch, const float* __restrict__ cmap,
                                                             const double* __restrict__ proj_cb, int n_levels,
                                                             int L, int n_canon, double* __restrict__ out,
                                                             int64_t out_stride) {
    extern __shared__ __align__(16) double Pd[];
    const int nc = NC > 0 ? NC : n_canon;
    const int nv = 1 + n_canon;
    for (int i = threadIdx.x; i < n_levels * L * nc; i += blockDim.x) {
        const int j = i % nc, bl = i / nc;  // bl = b * L + l
        Pd[i] = proj_cb[(size_t)bl * nv] - proj_cb[(size_t)bl * nv + 1 + j];
    }
    __syncthreads();
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
        const float* w = cmap + (size_t)p * n_ch;
        for (int b = 0; b < n_levels; ++b) {
            const double* Pb = Pd + (size_t)b * L * nc;
            double best = INFINITY;
            if (NC > 0) {
                double d[NC > 0 ? NC : 1];
#pragma unroll
                for (int j = 0; j < (NC > 0 ? NC : 1); ++j) d[j] = 0.0;
                for (int l0 = 0; l0 < L; l0 += 4) {
                    const float4 w4 = __ldcs(reinterpret_cast<const float4*>(w + b * L + l0));
                    const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const double wd = (double)wv[e];
                        const double* Pl = Pb + (l0 + e) * (NC > 0 ? NC : 1);
#pragma unroll
                        for (int j = 0; j < (NC > 0 ? NC : 1); ++j) d[j] = fma(wd, Pl[j], d[j]);
                    }
                }
#pragma unroll
                for (int j = 0; j < (NC > 0 ? NC : 1); ++j) best = np_minimum(best, sigmoid2(d[j]));
            } else {
                for (int j = 0; j < nc; ++j) {
                    double dj = 0.0;
                    for (int l = 0; l < L; ++l) dj = fma((double)w[b * L + l], Pb[l * nc + j], dj);
                    best = np_minimum(best, sigmoid2(dj));
                }
            }
            out[(size_t)b * out_stride + p] = best;
        }
    }
}

void launch_relevancy_from_cmap(int64_t P, int n_ch, const float* cmap, const double* proj_cb, int n_levels,
                                int L, int n_canon, double* out, int64_t out_stride, cudaStream_t st) {
    if (P == 0) return;
    const size_t smem = sizeof(double) * (size_t)n_levels * L * n_canon;
    const bool vec = (L % 4 == 0) && (n_ch % 4 == 0) && ((uintptr_t)cmap % 16 == 0);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_relevancy_from_cmap<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_relevancy_from_cmap<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = true;
    }
    const int blocks = (int)std::min<int64_t>(ceil_div(P, 256), 148 * 8);
    if (vec && n_canon == 4)
        k_relevancy_from_cmap<4><<<blocks, 256, smem, st>>>(P, n_ch, cmap, proj_cb, n_levels, L, n_canon, out,
                                                            out_stride);
    else
        k_relevancy_from_cmap<0><<<blocks, 256, smem, st>>>(P, n_ch, cmap, proj_cb, n_levels, L, n_canon, out,
                                                            out_stride);
}

// Exact fp64 replay (rasterizer.py:161-177) of the pixels whose early-exit
// decision the fp32 transmittance could not certify.  One warp per pixel:
// lanes evaluate 32 list entries at once in fp64 (reference op order), a
// warp prefix product gives T before each entry, counted iff T >= 1e-4.
// W accumulates in fp64 in shared memory.
constexpr int kFixWarps = 4;
__global__ void __launch_bounds__(32 * kFixWarps) k_blend_fixup(BlendArgs A) {
    __shared__ double wsm[kFixWarps][kChBlock];
    const uint32_t count = min(*A.fixup_count, A.fixup_capacity);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        const_cast<int64_t*>(A.stats)[SF_STAT_FIXUPS] = (int64_t)*A.fixup_count;
    const int C = A.C;
    const int cs = chan_rec_bytes(C);
    const int voff = chan_val_offset(C);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* wl = wsm[wid];
    const bool local = A.n_ch <= kChBlock;
    for (uint32_t idx = blockIdx.x * kFixWarps + wid; idx < count; idx += gridDim.x * kFixWarps) {
        const uint32_t code = A.fixup_list[idx];
        const int tile = (int)(code >> 8), slot = (int)(code & 255u);
        const int w8 = slot >> 5, l8 = slot & 31;
        const int px = (tile % A.tiles_x) * SF_TILE + (w8 & 1) * 8 + (l8 & 7);
        const int py = (tile / A.tiles_x) * SF_TILE + (w8 >> 1) * 4 + (l8 >> 3);
        const size_t pix = (size_t)py * A.W + px;
        float* row = A.coeff_map ? A.coeff_map + pix * A.n_ch : nullptr;
        for (int c = lane; c < A.n_ch; c += 32) {
            if (local) wl[c] = 0.0;
            else row[c] = 0.f;
        }
        __syncwarp();
        double T = 1.0;  // transmittance before the current chunk
        const double pxd = (double)px, pyd = (double)py;
        const uint32_t beg = A.tile_offsets[tile], end = A.tile_offsets[tile + 1];
        for (uint32_t i0 = beg; i0 < end && T >= SF_EARLY_EXIT_T; i0 += 32) {
            const uint32_t i = i0 + lane;
            double al = 0.0;
            uint32_t r = 0;
            if (i < end) {
                r = A.entries[i];
                const GeomRec g = A.geom[r];
                double ddx = __dadd_rn(pxd, -g.mx), ddy = __dadd_rn(pyd, -g.my);
                double t1 = __dmul_rn(__dmul_rn(g.a64, ddx), ddx);
                double t2 = __dmul_rn(__dmul_rn(__dmul_rn(2.0, g.b64), ddx), ddy);
                double t3 = __dmul_rn(__dmul_rn(g.c64, ddy), ddy);
                double q = __dadd_rn(__dadd_rn(t1, t2), t3);
                if (q <= SF_CUTOFF)
                    al = np_minimum(__dmul_rn((double)g.opacity, exp(__dmul_rn(-0.5, q))), SF_ALPHA_CLAMP);
            }
            // inclusive prefix product of (1 - alpha) -> T before each lane's entry
            double f = __dadd_rn(1.0, -al);
            double incl = f;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                double v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl = __dmul_rn(v, incl);
            }
            double excl = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane == 0) excl = 1.0;
            const double Tb = __dmul_rn(T, excl);
            const bool counted = (i < end) && (Tb >= SF_EARLY_EXIT_T) && (al > 0.0);
            if (counted) {
                const double e = __dmul_rn(al, Tb);
                const unsigned char* rec = A.chan + (size_t)r * cs;
                const uint16_t* ch = reinterpret_cast<const uint16_t*>(rec);
                const float* val = reinterpret_cast<const float*>(rec + voff);
                for (int k = 0; k < C; ++k) {
                    if (local) atomicAdd(&wl[ch[k]], e * (double)val[k]);
                    else atomicAdd(&row[ch[k]], (float)(e * (double)val[k]));
                }
            }
            T = __dmul_rn(T, __shfl_sync(0xffffffffu, incl, 31));
            // stop at the first uncounted entry: T before later entries only shrinks
            if (__any_sync(0xffffffffu, (i < end) && !(Tb >= SF_EARLY_EXIT_T))) T = 0.0;
            const unsigned last_counted = __ballot_sync(0xffffffffu, (i < end) && (Tb >= SF_EARLY_EXIT_T));
            if (T == 0.0) {
                // final T = T after the last counted entry
                const int lc = 31 - __clz(last_counted);
                double Tl = __shfl_sync(0xffffffffu, __dmul_rn(Tb, f), lc < 0 ? 0 : lc);
                T = (lc < 0) ? 0.0 : Tl;
                break;
            }
        }
        __syncwarp();
        if (local && row)
            for (int c = lane; c < A.n_ch; c += 32) row[c] = (float)wl[c];
        if (lane == 0 && A.final_t) A.final_t[pix] = (float)T;
        if (A.proj_cb && A.relevancy_raw && lane == 0) {
            const int nv = 1 + A.n_canon;
            for (int b = 0; b < A.n_levels; ++b) {
                const double* P = A.proj_cb + (size_t)b * A.L * nv;
                double best = INFINITY;
                for (int j = 1; j < nv; ++j) {
                    double dj = 0.0;
                    for (int l = 0; l < A.L; ++l) {
                        const int c = b * A.L + l;
                        dj = fma((double)(local ? (float)wl[c] : row[c]), P[l * nv] - P[l * nv + j], dj);
                    }
                    best = np_minimum(best, sigmoid2(dj));
                }
                A.relevancy_raw[(size_t)b * A.W * A.H + pix] = best;
            }
        }
        __syncwarp();
    }
}

int launch_blend(const BlendArgs& a, cudaStream_t st) {
    if (a.C > kMaxC) return -2;
    if (a.proj_cb && a.n_ch > kChBlock) return -3;  // fused relevancy needs every channel in one CTA
    int n_tiles = a.n_band_tiles;
    int ch_block = a.n_ch < kChBlock ? a.n_ch : kChBlock;
    int nblk = (a.n_ch + ch_block - 1) / ch_block;
    size_t smem = sizeof(BlendSmem) + (size_t)ch_block * kAccPitch * sizeof(float);
    const bool fast = (a.C == 12 && nblk == 1);
    const int nc = a.proj_cb ? a.n_canon : 0;
    void (*kern)(BlendArgs, int);
    int ki;
    if (fast && !a.proj_cb) { kern = k_blend<12, true, 0>; ki = 0; }
    else if (fast && nc == 4) { kern = k_blend<12, true, 4>; ki = 1; }
    else if (fast) { kern = k_blend<12, true, -1>; ki = 2; }
    else { kern = k_blend<0, false, -1>; ki = 3; }
    static size_t configured[4] = {0, 0, 0, 0};
    if (smem > configured[ki]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured[ki] = smem;
    }
    if (n_tiles > 0) kern<<<dim3(2 * n_tiles, nblk), kCTAThreads, smem, st>>>(a, ch_block);
    if (n_tiles > 0 && a.fixup_list && a.early_exit) k_blend_fixup<<<296, 32 * kFixWarps, 0, st>>>(a);
    return 0;  // (relevancy for n_ch > one channel block: launch_relevancy_from_cmap by the caller)
}

}  // namespace sf
