// sf_blend.cu -- K5/K6 (+ fused K7): per-tile front-to-back blending with
// top-K sparse scatter, optionally followed in the same CTA by the codebook
// decode of the finished tile on the tcgen05 tensor cores.
//
// Reference: tile_blend_weights (rasterizer.py:133-181) and the scatter loop
// of _splat_levels (sparse_splat.py:138-150):
//     alpha_i = min(o_i * exp(-q_i / 2), 0.99), alpha_i = 0 if q_i > 9
//     e_i = alpha_i * T_i  counted iff T_i >= 1e-4,  T_{i+1} = T_i (1 - alpha_i)
//     W[p, cat_idx[i]] += e_i[p] * cat_vals[i]
// and decode (sparse_splat.py:183-199): F_b = W_b @ atoms_b per level.
//
// B200 mapping (K5).  One CTA per half tile (16x8 pixels): four
// consumer warps own an 8x4 pixel patch each, one producer warp streams the
// tile's depth-ordered list through a 2-stage cp.async/mbarrier ring.  fp32
// alpha / transmittance with a guard band in which the reference's fp64 q
// decides membership; early-exit decisions fp32 cannot certify are replayed
// in fp64 by k_blend_fixup.  The coefficient accumulator is fp32 in shared
// memory, acc[channel][slot] with a 129-float pitch (conflict-free scatter).
//
// Fused decode (DEC).  Decode is HBM-store bound (9.56 GB of fp32 features
// per 1440x1080 frame) while blending is issue bound, so the decode of a
// finished tile runs inside the blend CTA: with two CTAs per SM one CTA's
// feature stores drain while the other blends, and the coefficient map never
// round-trips HBM.  Per level b: consumer thread = pixel = TMEM lane splits
// its 64 coefficients into tf32 hi/lo and stores them to TMEM (A operand);
// the producer warp streams pre-swizzled codebook chunks (32 output columns,
// hi + lo, 16 KB) by bulk copy into the freed level-0 accumulator space and
// issues 3xTF32 tcgen05.mma (A from TMEM, B from SMEM) into four 32-column
// TMEM accumulators; consumer warps drain them (tcgen05.ld) straight to HBM,
// one 128-byte line per pixel per chunk.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "sf_common.cuh"
#include "sf_blend_dev.cuh"

namespace sf {

// One CTA per half tile (16x8 pixels = 4 warp patches of 8x4): ~110 KB of
// shared memory, so two CTAs share an SM and one's list start-up and
// epilogue overlap the other's blending.
constexpr int kBlendThreads = 128;  // consumer threads: one per pixel
constexpr int kConsumerWarps = kBlendThreads / 32;
constexpr int kCTAThreads = kBlendThreads + 32;  // + one producer warp
constexpr int kTilePixels = 128;    // pixels per CTA (half a 16x16 tile)
constexpr int kStages = 3;          // batch ring between the producer and the consumer warps
constexpr int kBatch = 32;
constexpr int kAccPitch = 129;
constexpr int kMaxC = 16;            // channels per Gaussian (levels*K) supported
constexpr int kStageChan = 3072;     // scatter-plan bytes per stage: 32 records of C <= 12, 24 of C <= 16
constexpr int kChBlock = 192;        // accumulator channels per CTA (smem bound)
static_assert(kChanWord == kAccPitch * 4, "channel words are accumulator byte offsets");


struct __align__(16) BlendStage {
    GeomF32 g[kBatch];
    uint32_t row[kBatch];
    unsigned char chan[kStageChan];
};
__host__ __device__ constexpr int batch_cap(int cs) { return kStageChan / cs < kBatch ? kStageChan / cs : kBatch; }

// fused decode (DEC).  TMEM columns per CTA (two CTAs per SM share 512):
// two A slots of 64 columns (fp16 hi [0, 32) + lo [32, 64), pairs per
// column) -- level b uses slot b & 1 -- then two 64-column fp32 accumulators.
// A-from-TMEM MMAs read 4 KB of A per K step at ~64 B/clk, so N = 64 keeps the
// tensor core at its A-read floor; the A slots free the accumulator space
// level by level for the codebook ring and the output staging.
constexpr int kDecTmemCols = 256;
#ifndef SF_DEC_N
#define SF_DEC_N 64
#endif
#ifndef SF_DEC_ACC
#define SF_DEC_ACC 2
#endif
constexpr int kDecN = SF_DEC_N;               // output columns per chunk (MMA N)
constexpr int kDecAcc = SF_DEC_ACC;           // TMEM accumulators of kDecN columns
constexpr int kDecAccCol = 128;
constexpr int kDecChunkBytes = 2 * kDecN * 128;  // B chunk: {hi, lo} x kDecN rows (n) x 64 fp16 (128 B, SW128)
static_assert(kDecAccCol + kDecAcc * kDecN <= 256, "accumulators exceed the CTA's TMEM columns");
#ifndef SF_DEC_STAGES
#define SF_DEC_STAGES 2
#endif
#ifndef SF_DEC_BOXES
#define SF_DEC_BOXES 2
#endif
constexpr int kDecStages = SF_DEC_STAGES;     // B chunk ring at the start of the accumulator space
constexpr int kDecBoxes = SF_DEC_BOXES;       // output boxes per consumer warp
#ifndef SF_DEC_BOXCOLS
#define SF_DEC_BOXCOLS 32
#endif
#ifndef SF_DEC_BATCHED
#define SF_DEC_BATCHED 1
#endif
constexpr int kDecBoxCols = SF_DEC_BOXCOLS;   // output box: 8 x 4 pixels (a warp's patch) x 32 fp32 (SW128) or 16 (SW64)
constexpr int kDecOutBytes = 8 * 4 * kDecBoxCols * 4;
constexpr int kDecMaxLevels = 3;

struct __align__(16) BlendSmem {
    BlendStage st[kStages];
    uint64_t full[kStages];   // producer -> consumers: batch staged (count 1)
    uint64_t empty[kStages];  // consumers -> producer: batch consumed (one arrival per consumer warp)
    int nb[kStages];          // batch size; 0 = end of the tile's stream
    int n_done_warps;         // consumer warps whose pixels all saturated
    // fused decode
    uint64_t a_ready;              // consumers -> issuer: A of levels 0-1 (phase 0), level 2 (phase 1) in TMEM
    uint64_t a_free;               // MMAs of level 0 done: its TMEM slot takes level 2 (tcgen05.commit)
    uint64_t b_full[kDecStages];   // codebook chunk landed (tx count)
    uint64_t acc_full[kDecAcc];    // accumulator complete (tcgen05.commit)
    uint64_t acc_empty[kDecAcc];   // accumulator drained (4 warp arrivals)
    uint32_t tmem_base;
};


// Issue the cp.async copies of one batch (nb records) into stage buffer S
// (called by the 32 lanes of the producer warp; lane j holds record j's row).
__device__ __forceinline__ void stage_batch(BlendStage& S, const BlendArgs& A, uint32_t rows, int nb, int cs) {
    constexpr int gchunks = (int)(sizeof(GeomF32) / 16);  // 2
    const int cchunks = cs / 16;
    const int per = gchunks + cchunks;
    const int lane = (int)(threadIdx.x & 31);
    const int n = nb * per;
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int idx = i0 + lane;
        const int j = min(idx / per, 31), c = idx - j * per;
        const uint32_t r = __shfl_sync(0xffffffffu, rows, j);
        if (idx < n) {
            if (c < gchunks) {
                cp_async16(reinterpret_cast<char*>(&S.g[j]) + 16 * c,
                           reinterpret_cast<const char*>(A.geom + r) + 16 * c);
            } else {
                const int cc = c - gchunks;
                cp_async16(S.chan + j * cs + 16 * cc, A.chan + (size_t)r * cs + 16 * cc);
            }
        }
    }
    if (lane < nb) S.row[lane] = rows;
}


__host__ __device__ constexpr int acc_bytes(int nch) { return (nch * kAccPitch * 4 + 15) / 16 * 16; }

// CT: channels per Gaussian (0 = runtime), SINGLE: one channel block,
// NC: canonical phrases of the fused relevancy (0 = none, -1 = runtime count),
// DEC: fused 3xTF32 decode of the finished tile into A.features.
// Shared memory: [accumulator (1024-aligned when DEC)][BlendSmem].
template <int CT, bool SINGLE, int NC, bool DEC>
__global__ void __launch_bounds__(kCTAThreads, 2)
k_blend(BlendArgs A, int ch_block, const __grid_constant__ CUtensorMap fmap) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t mis = DEC ? ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u) : 0u;
    float* acc = reinterpret_cast<float*>(smem_raw + mis);
    BlendSmem& S = *reinterpret_cast<BlendSmem*>(smem_raw + mis + acc_bytes(ch_block));

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
    // fused relevancy: this thread's share of the logit-difference vectors
    // Pd = P_q - P_cj, loaded now so the global latency hides under the blend
    constexpr int kPdRegs = 6;
    double pd_pre[kPdRegs];
    if (NC != 0 && A.proj_cb) {
        const int nc = NC > 0 ? NC : A.n_canon, nv = 1 + A.n_canon;
        const int np = A.n_levels * A.L * nc;
#pragma unroll
        for (int u = 0; u < kPdRegs; ++u) {
            const int i = threadIdx.x + u * kCTAThreads;
            const int j = i % nc, bl = i / nc;
            pd_pre[u] = i < np ? A.proj_cb[(size_t)bl * nv] - A.proj_cb[(size_t)bl * nv + 1 + j] : 0.0;
        }
    }
    if (threadIdx.x == 0) {
        for (int st = 0; st < kStages; ++st) {
            bar_init(&S.full[st], 33);  // 32 cp.async arrivals + the producer's release of rows / nb
            bar_init(&S.empty[st], kConsumerWarps);
        }
        S.n_done_warps = 0;
        if (DEC) {
            bar_init(&S.a_ready, kConsumerWarps);
            bar_init(&S.a_free, 1);
            for (int i = 0; i < kDecStages; ++i) {
                bar_init(&S.b_full[i], 1);
            }
            for (int i = 0; i < kDecAcc; ++i) {
                bar_init(&S.acc_full[i], 1);
                bar_init(&S.acc_empty[i], kConsumerWarps);
            }
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (DEC && threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&S.tmem_base)),
                     "n"(kDecTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < nchb * kAccPitch; i += kCTAThreads) acc[i] = 0.f;
    if (DEC) tc_before();
    __syncthreads();
    if (DEC) tc_after();
    if (A.timeline && threadIdx.x == 0) A.timeline[4 * (blockIdx.x + gridDim.x * blockIdx.y)] = gtimer();

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
        // Entry rows are loaded two batches ahead and the next batch's records
        // are prefetched into L2, so a batch's cp.async gathers hit L2.  The
        // producer never waits for its gathers: each lane's
        // cp.async.mbarrier.arrive fires the stage's `full` barrier when its
        // copies land (32 arrivals + lane 0's arrive after rows and nb).
        const int pl = threadIdx.x & 31;
        const int bcap = batch_cap(cs);
        auto entry = [&](uint32_t i) -> uint32_t { return (i < end && pl < bcap) ? __ldg(A.entries + i) : 0u; };
        uint32_t e_cur = entry(beg + pl), e_next = entry(beg + bcap + pl);
        if (beg + pl < end && pl < bcap) prefetch_records(A, e_cur, cs);
        for (int bi = 0;; ++bi) {
            const int st = bi % kStages;
            const uint32_t base = beg + (uint32_t)bi * bcap;
            const uint32_t e_n2 = entry(base + 2 * bcap + pl);
            if (base + bcap + pl < end && pl < bcap) prefetch_records(A, e_next, cs);
            if (bi >= kStages) bar_wait(&S.empty[st], ((bi / kStages) - 1) & 1);
            const bool all_done = *reinterpret_cast<volatile int*>(&S.n_done_warps) == kConsumerWarps;
            const int nb = (base < end && !all_done) ? (int)min((uint32_t)bcap, end - base) : 0;
            BlendStage& B = S.st[st];
            if (nb) stage_batch(B, A, e_cur, nb, cs);
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(&S.full[st]))
                         : "memory");
            if (pl == 0) S.nb[st] = nb;
            __syncwarp();
            if (pl == 0) bar_arrive(&S.full[st]);
            if (nb == 0) break;
            e_cur = e_next;
            e_next = e_n2;
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
            // Candidates go in groups of kGroup: the group's alphas are computed
            // first, branch-free (independent work, high ILP); the rare pixels
            // inside a guard band take the exact fp64 test afterwards; then the
            // sequential part -- transmittance and scatter -- walks the group.
            uint32_t wmask = wcand;
            while (wmask) {
                constexpr int kGroup = 8;
                int jj[kGroup];
                float alv[kGroup];
                uint32_t amb = 0;
#pragma unroll
                for (int u = 0; u < kGroup; ++u) {
                    jj[u] = wmask ? __ffs(wmask) - 1 : -1;
                    wmask &= wmask - 1;
                }
#pragma unroll
                for (int u = 0; u < kGroup; ++u) {
                    bool g = false;
                    alv[u] = jj[u] >= 0 ? blend_alpha_fast(B.g[jj[u] & 31], pxf, pyf, g) : 0.f;
                    amb |= (g ? 1u : 0u) << u;
                }
                if (__any_sync(0xffffffffu, amb != 0)) {
                    for (int u = 0; u < kGroup; ++u)
                        if (amb & (1u << u))
                            alv[u] = blend_alpha_exact(B.g[jj[u]], A.geom + B.row[jj[u]], pxd, pyd);
                }
                if (CT > 0 && CT % 4 == 0 && SINGLE) {
                    // Branch-free walk: every member scatters (ef = 0 leaves the
                    // accumulator unchanged), and the next member's channel words
                    // and values are loaded before this member's stores, so the
                    // only chain is acc load -> FMA -> store through shared memory.
                    constexpr int NH = CT > 0 ? CT : 4;
                    char* accs = reinterpret_cast<char*>(acc + slot);
                    uint32_t oo[NH], on[NH];
                    float vv[NH], vn[NH];
                    auto load_rec = [&](int j, uint32_t (&o)[NH], float (&v)[NH]) {
                        const unsigned char* rec = B.chan + j * cs;
                        const uint4* oh = reinterpret_cast<const uint4*>(rec);
                        const float4* vh = reinterpret_cast<const float4*>(rec + voff);
#pragma unroll
                        for (int e = 0; e < NH / 4; ++e) {
                            const uint4 o4 = oh[e];
                            const float4 v4 = vh[e];
                            o[4 * e] = o4.x, o[4 * e + 1] = o4.y, o[4 * e + 2] = o4.z, o[4 * e + 3] = o4.w;
                            v[4 * e] = v4.x, v[4 * e + 1] = v4.y, v[4 * e + 2] = v4.z, v[4 * e + 3] = v4.w;
                        }
                    };
                    load_rec(jj[0], oo, vv);
#pragma unroll
                    for (int u = 0; u < kGroup; ++u) {
                        if (jj[u] < 0) break;
                        if (u + 1 < kGroup && jj[u + 1 < kGroup ? u + 1 : u] >= 0)
                            load_rec(jj[u + 1 < kGroup ? u + 1 : u], on, vn);
                        const float al = alv[u];
                        const bool live = al > 0.f && !done;
                        const float ef = live ? al * T : 0.f;
                        if (live) {
                            Tprev = T;
                            T = fmaf(-al, T, T);
                            eb = fmaf(al, rcp_approx(1.f - al), eb);  // 1 - al in [0.01, 1]: no denormals
                            ++ncontrib;
                            if (A.early_exit && T < (float)SF_EARLY_EXIT_T) done = true;
                        }
                        float av[NH];
#pragma unroll
                        for (int e = 0; e < NH; ++e) av[e] = *reinterpret_cast<const float*>(accs + oo[e]);
#pragma unroll
                        for (int e = 0; e < NH; ++e) av[e] = fmaf(ef, vv[e], av[e]);
#pragma unroll
                        for (int e = 0; e < NH; ++e) *reinterpret_cast<float*>(accs + oo[e]) = av[e];
#pragma unroll
                        for (int e = 0; e < NH; ++e) oo[e] = on[e], vv[e] = vn[e];
                    }
                    continue;
                }
#pragma unroll
                for (int u = 0; u < kGroup; ++u) {
                    if (jj[u] < 0) break;
                    const int j = jj[u];
                    const float al = alv[u];
                    float ef = 0.f;
                    if (al > 0.f && !done) {
                        ef = al * T;
                        Tprev = T;
                        T = fmaf(-al, T, T);
                        eb = fmaf(al, rcp_approx(1.f - al), eb);  // 1 - al in [0.01, 1]: no denormals
                        ++ncontrib;
                        if (A.early_exit && T < (float)SF_EARLY_EXIT_T) done = true;
                    }
                    if (__any_sync(0xffffffffu, ef > 0.f)) {
                        const unsigned char* rec = B.chan + j * cs;
                        const float* val = reinterpret_cast<const float*>(rec + voff);
                        char* accs = reinterpret_cast<char*>(acc + slot);
                        if (CT > 0 && CT % 4 == 0 && SINGLE) {
                            // channel words are accumulator byte offsets; a Gaussian's
                            // channels are distinct: all loads, then FMAs, then stores
                            constexpr int NH = CT > 0 ? CT : 4;
                            const uint4* oh = reinterpret_cast<const uint4*>(rec);
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
                            const uint32_t* words = reinterpret_cast<const uint32_t*>(rec);
                            for (int k = 0; k < C; ++k) {
                                const int ch = chan_id(words[k]) - ch0;
                                if ((unsigned)ch < (unsigned)nchb) {
                                    float* a = reinterpret_cast<float*>(accs + (size_t)ch * kChanWord);
                                    *a = fmaf(ef, val[k], *a);
                                }
                            }
                        }
                    }
                }
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
    // no contribution anywhere in the half tile: its decoded features are zero
    const bool any_contrib = __syncthreads_or(ncontrib > 0);

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
    if (A.timeline && threadIdx.x == 0) A.timeline[4 * (blockIdx.x + gridDim.x * blockIdx.y) + 1] = gtimer();
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
            if (np <= kPdRegs * kCTAThreads) {
#pragma unroll
                for (int u = 0; u < kPdRegs; ++u) {
                    const int i = threadIdx.x + u * kCTAThreads;
                    if (i < np) Pd[i] = pd_pre[u];
                }
            } else {
                for (int i = threadIdx.x; i < np; i += kCTAThreads) {
                    const int j = i % nc, bl = i / nc;
                    Pd[i] = A.proj_cb[(size_t)bl * nv] - A.proj_cb[(size_t)bl * nv + 1 + j];
                }
            }
            __syncthreads();
        }
        if (DEC && NC == 4 && fits && A.n_levels == 3 && A.L == 64) {
            // computed level by level inside the decode's A conversion (same reads)
        } else if (inside && NC == 4 && fits && A.n_levels == 3 && A.L == 64) {
            // the three levels together: 12 independent fp64 accumulation chains
            double d[3][4];
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
                for (int j = 0; j < 4; ++j) d[b][j] = 0.0;
#pragma unroll 2
            for (int l = 0; l < 64; ++l) {
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    const double w = (double)acc[(b * 64 + l) * kAccPitch + slot];
                    const double* Pl = Pd + (size_t)(b * 64 + l) * 4;
                    const double2 p01 = *reinterpret_cast<const double2*>(Pl);
                    const double2 p23 = *reinterpret_cast<const double2*>(Pl + 2);
                    d[b][0] = fma(w, p01.x, d[b][0]);
                    d[b][1] = fma(w, p01.y, d[b][1]);
                    d[b][2] = fma(w, p23.x, d[b][2]);
                    d[b][3] = fma(w, p23.y, d[b][3]);
                }
            }
#pragma unroll
            for (int b = 0; b < 3; ++b)  // sigmoid is monotone: min_j sigmoid(d_j) = sigmoid(min_j d_j)
                A.relevancy_raw[(size_t)b * A.W * A.H + (size_t)py * A.W + px] =
                    sigmoid2(np_minimum(np_minimum(d[b][0], d[b][1]), np_minimum(d[b][2], d[b][3])));
        } else if (inside) {
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
    if (DEC) {
        // ---------------- fused decode: F_b = W_b @ atoms_b on tcgen05 ----------------
        // 3-term fp16 split: W = Wh + Wl, atoms = Bh + Bl (each rounded to
        // fp16), F ~= Wh Bh + Wh Bl + Wl Bh accumulated in fp32 (error ~2^-22
        // |W||B|, plus 2^-25 absolute for subnormal low parts, which the
        // per-level power-of-two codebook scale keeps below 2^-19 max|B|).
        // Levels 0 and 1 go to TMEM first, freeing accumulator bytes
        // [0, 64 KB) for the codebook ring (2 x 16 KB) and the per-warp output
        // boxes (2 x 4 KB each); level 2 replaces level 0 once level 0's MMAs
        // are done.
        const int nchunk = A.D / kDecN;
        const int total = A.n_levels * nchunk;
        const uint32_t tm = S.tmem_base;
        unsigned char* bring = reinterpret_cast<unsigned char*>(acc);
        unsigned char* obuf = bring + kDecStages * kDecChunkBytes;  // kDecBoxes output boxes per consumer warp
        static_assert(kDecStages * kDecChunkBytes + kConsumerWarps * kDecBoxes * kDecOutBytes <= 64 * 128 * kAccPitch * 4,
                      "ring + boxes must fit in the accumulator rows of levels 0-1");
        if (consumer) {
            const uint32_t lane_off = (uint32_t)(cw * 32) << 16;  // this warp's TMEM lane quarter
            // level b's coefficients (this thread's pixel) -> fp16 hi/lo pairs in A slot b & 1
            // fused relevancy rides on the conversion's reads (Pd staged in S.st)
            const bool rel = NC == 4 && A.proj_cb && A.n_levels == 3 && A.L == 64 &&
                             A.n_levels * A.L * 4 * (int)sizeof(double) <= (int)sizeof(S.st);
            const double* Pd = reinterpret_cast<const double*>(&S.st[0]);
            auto convert = [&](int b, bool with_rel) {
                const bool rel_b = rel && with_rel;
                // even / odd K in separate chains (8 independent fp64 FMA chains)
                double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0, e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll 1
                for (int kb = 0; kb < 2; ++kb) {
                    uint32_t hi[16], lo[16];
                    const float* src = acc + (b * 64 + kb * 32) * kAccPitch + slot;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float x0 = src[(2 * k) * kAccPitch], x1 = src[(2 * k + 1) * kAccPitch];
                        if (rel_b) {
                            const double* P0 = Pd + (size_t)(b * 64 + kb * 32 + 2 * k) * 4;
                            const double2 a01 = *reinterpret_cast<const double2*>(P0);
                            const double2 a23 = *reinterpret_cast<const double2*>(P0 + 2);
                            const double2 b01 = *reinterpret_cast<const double2*>(P0 + 4);
                            const double2 b23 = *reinterpret_cast<const double2*>(P0 + 6);
                            const double w0 = (double)x0, w1 = (double)x1;
                            d0 = fma(w0, a01.x, d0), d1 = fma(w0, a01.y, d1);
                            d2 = fma(w0, a23.x, d2), d3 = fma(w0, a23.y, d3);
                            e0 = fma(w1, b01.x, e0), e1 = fma(w1, b01.y, e1);
                            e2 = fma(w1, b23.x, e2), e3 = fma(w1, b23.y, e3);
                        }
                        const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
                        const __half l0 = __float2half_rn(x0 - __half2float(h0));
                        const __half l1 = __float2half_rn(x1 - __half2float(h1));
                        hi[k] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
                        lo[k] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
                    }
                    const uint32_t col = (uint32_t)(64 * (b & 1) + 16 * kb);
                    tmem_st16(tm + lane_off + col, hi);
                    tmem_st16(tm + lane_off + col + 32, lo);
                }
                // sigmoid is monotone: min_j sigmoid(d_j) = sigmoid(min_j d_j)
                d0 += e0, d1 += e1, d2 += e2, d3 += e3;
                if (rel_b && inside)
                    A.relevancy_raw[(size_t)b * A.W * A.H + (size_t)py * A.W + px] =
                        sigmoid2(np_minimum(np_minimum(d0, d1), np_minimum(d2, d3)));
            };
            for (int b = 0; b < A.n_levels && b < 2; ++b) convert(b, true);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");

            proxy_fence();  // accumulator reads precede the bulk copies / boxes written over them
            tc_before();
            __syncwarp();
            if (lane == 0) bar_arrive(&S.a_ready);
            if (A.timeline && threadIdx.x == 0) A.timeline[4 * (blockIdx.x + gridDim.x * blockIdx.y) + 2] = gtimer();
            if (rel && inside) {
                // level 2's relevancy while the tensor cores start on level 0: its
                // accumulator rows stay intact until level 2 is converted
                double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0, e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
                const float* src = acc + 128 * kAccPitch + slot;
#pragma unroll 2
                for (int l = 0; l < 64; l += 2) {
                    const double w = (double)src[l * kAccPitch], v = (double)src[(l + 1) * kAccPitch];
                    const double* P0 = Pd + (size_t)(128 + l) * 4;
                    const double2 a01 = *reinterpret_cast<const double2*>(P0);
                    const double2 a23 = *reinterpret_cast<const double2*>(P0 + 2);
                    const double2 b01 = *reinterpret_cast<const double2*>(P0 + 4);
                    const double2 b23 = *reinterpret_cast<const double2*>(P0 + 6);
                    d0 = fma(w, a01.x, d0), d1 = fma(w, a01.y, d1);
                    d2 = fma(w, a23.x, d2), d3 = fma(w, a23.y, d3);
                    e0 = fma(v, b01.x, e0), e1 = fma(v, b01.y, e1);
                    e2 = fma(v, b23.x, e2), e3 = fma(v, b23.y, e3);
                }
                d0 += e0, d1 += e1, d2 += e2, d3 += e3;
                A.relevancy_raw[(size_t)2 * A.W * A.H + (size_t)py * A.W + px] =
                    sigmoid2(np_minimum(np_minimum(d0, d1), np_minimum(d2, d3)));
            }

            // drain, each warp on its own: TMEM -> swizzled box (its 8 x 4 pixel
            // patch x 32 fp32, row = lane) -> TMA store by lane 0; no CTA barriers
            unsigned char* wbox = obuf + cw * kDecBoxes * kDecOutBytes;
            const int bx = x0 + (warp & 1) * 8, by = y0 + (warp >> 1) * 4;
            float scl[kDecMaxLevels];
#pragma unroll
            for (int b = 0; b < kDecMaxLevels; ++b) scl[b] = b < A.n_levels ? A.dec_scale[b] : 1.f;
            int nbox = 0;
            constexpr int kBoxesPerChunk = kDecN / kDecBoxCols;
            if (!any_contrib) {
                // empty half tile: zero boxes, stored for every chunk (no MMAs, no drains)
                for (int i = lane; i < kDecBoxes * kDecOutBytes / 16; i += 32)
                    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(smem_addr(wbox) + 16 * i), "r"(0u)
                                 : "memory");
                proxy_fence();
                __syncwarp();
                if (lane == 0) {
                    for (int g = 0; g < total; ++g) {
                        const int b = g / nchunk, c = g - b * nchunk;
                        for (int q = 0; q < kBoxesPerChunk; ++q)
                            tma_store_4d(&fmap, wbox + (q % kDecBoxes) * kDecOutBytes, c * kDecN + kDecBoxCols * q, bx,
                                         by, b);
                    }
                    bulk_commit();
                }
            }
            for (int g = 0; g < total && any_contrib; ++g) {
                const int t = g & (kDecAcc - 1), b = g / nchunk, c = g - b * nchunk;
                if (c == 0 && b == 1 && A.n_levels > 2) {
                    // level 0's MMAs are done (its chunks were drained): level 2 -> slot 0
                    bar_wait(&S.a_free, 0);
                    tc_after();
                    convert(2, false);
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    tc_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(&S.a_ready);
                }
                bar_wait(&S.acc_full[t], (g / kDecAcc) & 1);
                if (cw == 0 && lane == 0 && g + kDecStages < total) {
                    // chunk g's MMAs are complete: its codebook stage takes chunk g + kDecStages
                    const int sg = g % kDecStages;
                    bar_expect_tx(&S.b_full[sg], kDecChunkBytes);
                    bulk_g2s(bring + sg * kDecChunkBytes,
                             reinterpret_cast<const unsigned char*>(A.dec_b) + (size_t)(g + kDecStages) * kDecChunkBytes,
                             kDecChunkBytes, &S.b_full[sg]);
                }
                tc_after();
                uint32_t v[kDecN];
#pragma unroll
                for (int h = 0; h < kDecN / 32; ++h) {
                    uint32_t (&vh)[32] = *reinterpret_cast<uint32_t(*)[32]>(&v[32 * h]);
                    tmem_ld32(tm + lane_off + (uint32_t)(kDecAccCol + t * kDecN + 32 * h), vh);
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                tc_before();
                __syncwarp();
                if (lane == 0) bar_arrive(&S.acc_empty[t]);
                const float sc = b == 0 ? scl[0] : (b == 1 ? scl[1] : scl[2]);
                if (sc != 1.f) {
#pragma unroll
                    for (int i = 0; i < kDecN; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * sc);
                }
#pragma unroll
                auto fill_box = [&](unsigned char* box, int q) {
                    const uint32_t row = smem_addr(box) + lane * (kDecBoxCols * 4);
#pragma unroll
                    for (int u = 0; u < kDecBoxCols / 4; ++u) {
                        // 128-byte swizzle: unit u of row r at u ^ (r & 7); 64-byte: u ^ ((r >> 1) & 3)
                        const int pu = kDecBoxCols == 32 ? (u ^ (lane & 7)) : (u ^ ((lane >> 1) & 3));
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + (pu << 4)),
                                     "r"(v[kDecBoxCols * q + 4 * u]), "r"(v[kDecBoxCols * q + 4 * u + 1]),
                                     "r"(v[kDecBoxCols * q + 4 * u + 2]), "r"(v[kDecBoxCols * q + 4 * u + 3])
                                     : "memory");
                    }
                };
                if (SF_DEC_BATCHED && kDecBoxes == kBoxesPerChunk) {
                    // one box per chunk column block: the previous chunk's stores
                    // must have left the boxes; one fence and one commit per chunk
                    if (lane == 0) bulk_wait_read<0>();
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < kBoxesPerChunk; ++q) fill_box(wbox + q * kDecOutBytes, q);
                    proxy_fence();
                    __syncwarp();
                    if (lane == 0) {
#pragma unroll
                        for (int q = 0; q < kBoxesPerChunk; ++q)
                            tma_store_4d(&fmap, wbox + q * kDecOutBytes, c * kDecN + kDecBoxCols * q, bx, by, b);
                        bulk_commit();
                    }
                } else {
                    for (int q = 0; q < kBoxesPerChunk; ++q, ++nbox) {
                        if (lane == 0) bulk_wait_read<kDecBoxes - 1>();  // the store issued kDecBoxes ago has left this box
                        __syncwarp();
                        unsigned char* box = wbox + (nbox % kDecBoxes) * kDecOutBytes;
                        fill_box(box, q);
                        proxy_fence();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_4d(&fmap, box, c * kDecN + kDecBoxCols * q, bx, by, b);
                            bulk_commit();
                        }
                    }
                }
            }
            if (lane == 0) bulk_wait_read<0>();  // the boxes may be released once read; the writes complete with the grid
        } else {
            // issuer: the whole producer warp walks the chunk ring; lane 0 issues.
            // Per chunk 3 x 4 MMAs (128 x 64 x 16, fp16 -> fp32, A from TMEM).
            const uint32_t idesc = (1u << 4) | ((uint32_t)(kDecN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            const unsigned char* img = reinterpret_cast<const unsigned char*>(A.dec_b);
            const bool leader = lane == 0;
            const uint64_t desc0 = sw128_desc(smem_addr(bring));
            const int n_issue = any_contrib ? total : 0;  // empty half tile: nothing to multiply
            if (n_issue) bar_wait(&S.a_ready, 0);
            tc_after();
            if (leader && n_issue)
                for (int g = 0; g < kDecStages && g < total; ++g) {
                    bar_expect_tx(&S.b_full[g], kDecChunkBytes);
                    bulk_g2s(bring + g * kDecChunkBytes, img + (size_t)g * kDecChunkBytes, kDecChunkBytes,
                             &S.b_full[g]);
                }
            __syncwarp();
            for (int g = 0; g < n_issue; ++g) {
                const int s = g % kDecStages, t = g & (kDecAcc - 1), b = g / nchunk, c = g - b * nchunk;
                if (c == 0 && b >= 2) {  // level b's A replaced level b - 2's in its slot
                    bar_wait(&S.a_ready, (b - 1) & 1);
                    tc_after();
                }
                bar_wait(&S.b_full[s], (g / kDecStages) & 1);
                if (g >= kDecAcc) bar_wait(&S.acc_empty[t], ((g / kDecAcc) - 1) & 1);
                tc_after();
                if (leader) {
                    const uint32_t d = tm + (uint32_t)(kDecAccCol + t * kDecN);
                    const uint64_t bd = desc0 + (uint64_t)((s * kDecChunkBytes) >> 4);
                    const uint32_t ah0 = tm + (uint32_t)(64 * (b & 1));
#pragma unroll
                    for (int k = 0; k < 4; ++k) {  // K steps of 16: Wl Bh + Wh Bl + Wh Bh
                        const uint64_t bh = bd + 2 * k, bl = bh + ((kDecChunkBytes / 2) >> 4);
                        const uint32_t ah = ah0 + (uint32_t)(8 * k), al = ah + 32;
                        mma_f16_tmem_a(d, al, bh, idesc, k > 0 ? 1u : 0u);
                        mma_f16_tmem_a(d, ah, bl, idesc, 1u);
                        mma_f16_tmem_a(d, ah, bh, idesc, 1u);
                    }
                    mma_commit(&S.acc_full[t]);
                    if (c == nchunk - 1 && b + 2 < A.n_levels) mma_commit(&S.a_free);
                }
                __syncwarp();
            }
        }
        tc_before();
        __syncthreads();
        if (threadIdx.x < 32) {
            tc_after();
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(kDecTmemCols));
        }
        if (A.timeline && threadIdx.x == 0) A.timeline[4 * (blockIdx.x + gridDim.x * blockIdx.y) + 3] = gtimer();
    }
}

// Codebook chunks of the fused decode, pre-swizzled so one linear bulk copy
// lands the SW128 K-major fp16 operand image: for level b and output columns
// [64 c, 64 c + 64): {hi, lo} x 64 rows (n) x 64 fp16 (128 B), 16-byte unit j
// of row n stored at unit j ^ (n & 7).  The level's atoms are first scaled by
// a power of two 2^s (s = 0 unless max |atom| lies outside [2^-6, 2^8)), so
// both fp16 parts stay normal; dec_scale[b] = 2^-s undoes it in the epilogue.
// One CTA per (level, chunk).
__global__ void __launch_bounds__(256) k_dec_codebook_image(const float* __restrict__ cb, LevelSelDev lv, int L,
                                                            int D, unsigned char* __restrict__ out,
                                                            float* __restrict__ scale_out) {
    const int nchunk = D / kDecN;
    const int b = blockIdx.x / nchunk, c = blockIdx.x % nchunk;
    const float* atoms = cb + (size_t)lv.lv[b] * L * D;
    __shared__ float red[8];
    float m = 0.f;
    for (int i = threadIdx.x; i < L * D; i += blockDim.x) m = fmaxf(m, fabsf(atoms[i]));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = red[0];
    for (int i = 1; i < 8; ++i) m = fmaxf(m, red[i]);
    int e = 0;
    if (m > 0.f && (m < 0x1p-6f || m >= 0x1p8f)) {
        frexpf(m, &e);  // m = f 2^e, f in [0.5, 1): scale by 2^-e
        e = -e;
    }
    if (c == 0 && threadIdx.x == 0) scale_out[b] = ldexpf(1.f, -e);
    unsigned char* dst = out + (size_t)blockIdx.x * kDecChunkBytes;
    for (int i = threadIdx.x; i < kDecN * 64; i += blockDim.x) {
        const int n = i / 64, k = i % 64;
        const float x = ldexpf(atoms[(size_t)k * D + c * kDecN + n], e);
        const __half h = __float2half_rn(x);
        const __half l = __float2half_rn(x - __half2float(h));
        const int off = n * 128 + (((k >> 3) ^ (n & 7)) << 4) + (k & 7) * 2;
        *reinterpret_cast<__half*>(dst + off) = h;
        *reinterpret_cast<__half*>(dst + kDecChunkBytes / 2 + off) = l;
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
    ensure_smem_attr((const void*)k_relevancy_from_cmap<0>, 200 * 1024);
    ensure_smem_attr((const void*)k_relevancy_from_cmap<4>, 200 * 1024);
    const int blocks = (int)std::min<int64_t>(ceil_div(P, 256), 148 * 8);
    if (vec && n_canon == 4)
        k_relevancy_from_cmap<4><<<blocks, 256, smem, st>>>(P, n_ch, cmap, proj_cb, n_levels, L, n_canon, out,
                                                            out_stride);
    else
        k_relevancy_from_cmap<0><<<blocks, 256, smem, st>>>(P, n_ch, cmap, proj_cb, n_levels, L, n_canon, out,
                                                            out_stride);
}

// Relevancy of many prompts over one coefficient map (query sweep).  The map
// is read once: a CTA (one level: blockIdx.y) stages 256 pixels x L
// coefficients in shared memory (level-major, pixel-contiguous).  First each
// thread forms its pixel's canonical logits (<= 8) and keeps their max; then
// a thread takes 4 consecutive pixels x one block of 8 prompt columns (a 4 x 8
// register tile of fp64 FMA chains over l, 5 shared loads per 32 FMAs).
// rel = sigmoid(l_q - max_j l_j) = sigmoid(min_j (l_q - l_j)), the two-branch
// sigmoid of query.py:65-84; same value as the single-query Pd = P_q - P_cj
// form up to rounding (~1e-16 of the logits).
constexpr int kSwPx = 256, kSwThreads = 256, kSwCols = 8;  // pixels per tile, threads, columns per block
static_assert(kSwThreads == kSwPx, "the canonical pass maps one thread to one pixel");

__global__ void __launch_bounds__(kSwThreads, 2) k_relevancy_sweep(int64_t P, int n_ch, const float* __restrict__ cmap,
                                                                const double* __restrict__ proj, int n_levels, int L,
                                                                int nq, int nc, double* __restrict__ out,
                                                                int64_t pstride, int64_t lstride) {
    extern __shared__ __align__(16) unsigned char sw_smem[];
    const int nqp = (nq + kSwCols - 1) / kSwCols * kSwCols, nvp = nqp + kSwCols, nv = nq + nc;
    double* pj = reinterpret_cast<double*>(sw_smem);       // [L][nvp]: prompts, pad, canonicals, pad
    float* ws = reinterpret_cast<float*>(pj + (size_t)L * nvp);  // [L][kSwPx]
    double* lcs = reinterpret_cast<double*>(ws + (size_t)L * kSwPx);  // [kSwPx] max canonical logit
    const int t = threadIdx.x;
    const int b = blockIdx.y;  // one level per CTA: its projected codebook is loaded once
    for (int i = t; i < L * nvp; i += kSwThreads) {
        const int l = i / nvp, v = i % nvp;
        const double* src = proj + ((size_t)b * L + l) * nv;
        pj[i] = v < nq ? src[v] : ((v >= nqp && v - nqp < nc) ? src[nq + v - nqp] : 0.0);
    }
    for (int64_t base = (int64_t)blockIdx.x * kSwPx; base < P; base += (int64_t)gridDim.x * kSwPx) {
        const int np = (int)(P - base < kSwPx ? P - base : kSwPx);
        {
            __syncthreads();
            for (int h = 0; h < kSwPx / kSwThreads; ++h) {
                const int px = t + h * kSwThreads;
                if (px >= np) continue;
                const float4* src = reinterpret_cast<const float4*>(cmap + (size_t)(base + px) * n_ch + b * L);
#pragma unroll 8
                for (int k = 0; k < L / 4; ++k) {
                    const float4 v = __ldg(src + k);
                    ws[(4 * k + 0) * kSwPx + px] = v.x;
                    ws[(4 * k + 1) * kSwPx + px] = v.y;
                    ws[(4 * k + 2) * kSwPx + px] = v.z;
                    ws[(4 * k + 3) * kSwPx + px] = v.w;
                }
            }
            __syncthreads();
            // canonical logits: thread = pixel, 8 columns (the canonical block)
            {
                double lc[kSwCols];
#pragma unroll
                for (int c = 0; c < kSwCols; ++c) lc[c] = 0.0;
#pragma unroll 2
                for (int l = 0; l < L; ++l) {
                    const double w = ws[l * kSwPx + t];
                    const double2* pr = reinterpret_cast<const double2*>(pj + (size_t)l * nvp + nqp);
#pragma unroll
                    for (int c2 = 0; c2 < kSwCols / 2; ++c2) {
                        const double2 pv = pr[c2];
                        lc[2 * c2] = fma(w, pv.x, lc[2 * c2]);
                        lc[2 * c2 + 1] = fma(w, pv.y, lc[2 * c2 + 1]);
                    }
                }
                // min_j (l_q - l_j) = l_q - max_j l_j exactly (rounded subtraction is
                // monotone); NaN propagates as through np.minimum
                double mx = lc[0];
#pragma unroll
                for (int c = 1; c < kSwCols; ++c)
                    if (c < nc) mx = (mx != mx || lc[c] != lc[c]) ? NAN : fmax(mx, lc[c]);
                lcs[t] = mx;
            }
            __syncthreads();
            // prompt logits: thread = 4 consecutive pixels x one 8-column block
            // (4 x 8 register tile: 5 shared loads per 32 FMAs)
            const int pg = t % (kSwPx / 4), cg = t / (kSwPx / 4);
            const int px0 = 4 * pg;
            for (int cb = cg; cb * kSwCols < nq; cb += kSwThreads / (kSwPx / 4)) {
                const int c0 = cb * kSwCols;
                double acc[4][kSwCols];
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int j = 0; j < kSwCols; ++j) acc[r][j] = 0.0;
#pragma unroll 2
                for (int l = 0; l < L; ++l) {
                    const float4 w4 = *reinterpret_cast<const float4*>(ws + l * kSwPx + px0);
                    const double w[4] = {w4.x, w4.y, w4.z, w4.w};
                    const double2* pr = reinterpret_cast<const double2*>(pj + (size_t)l * nvp + c0);
#pragma unroll
                    for (int j2 = 0; j2 < kSwCols / 2; ++j2) {
                        const double2 pv = pr[j2];
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            acc[r][2 * j2] = fma(w[r], pv.x, acc[r][2 * j2]);
                            acc[r][2 * j2 + 1] = fma(w[r], pv.y, acc[r][2 * j2 + 1]);
                        }
                    }
                }
                const double2 m01 = *reinterpret_cast<const double2*>(lcs + px0);
                const double2 m23 = *reinterpret_cast<const double2*>(lcs + px0 + 2);
                const double lmax[4] = {m01.x, m01.y, m23.x, m23.y};
#pragma unroll
                for (int j = 0; j < kSwCols; ++j) {
                    if (c0 + j >= nq) break;
                    double v[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) v[r] = sigmoid2(acc[r][j] - lmax[r]);
                    double* o = out + (size_t)(c0 + j) * pstride + (size_t)b * lstride + base + px0;
                    if (px0 + 3 < np && (((uintptr_t)o) & 15) == 0) {
                        reinterpret_cast<double2*>(o)[0] = make_double2(v[0], v[1]);
                        reinterpret_cast<double2*>(o)[1] = make_double2(v[2], v[3]);
                    } else {
#pragma unroll
                        for (int r = 0; r < 4; ++r)
                            if (px0 + r < np) o[r] = v[r];
                    }
                }
            }
        }
    }
}

int launch_relevancy_sweep(int64_t P, int n_ch, const float* cmap, const double* proj, int n_levels, int L, int nq,
                           int n_canon, double* out, int64_t out_prompt_stride, int64_t out_level_stride,
                           cudaStream_t st) {
    const int nvp = (nq + kSwCols - 1) / kSwCols * kSwCols + kSwCols;
    const size_t smem = sizeof(double) * (size_t)L * nvp + sizeof(float) * (size_t)L * kSwPx +
                        sizeof(double) * kSwPx;
    if (n_canon < 1 || n_canon > kSwCols || L % 4 || n_ch % 4 || (uintptr_t)cmap % 16 || smem > 200 * 1024)
        return 1;
    if (P == 0 || nq == 0) return 0;
    ensure_smem_attr((const void*)k_relevancy_sweep, 200 * 1024);
    const int blocks = (int)std::min<int64_t>(ceil_div(P, kSwPx), std::max(1, 148 * 2 / n_levels));  // one wave
    k_relevancy_sweep<<<dim3(blocks, n_levels), kSwThreads, smem, st>>>(P, n_ch, cmap, proj, n_levels, L, nq, n_canon, out,
                                                        out_prompt_stride, out_level_stride);
    return 0;
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
        // list rows are loaded two chunks ahead, their geometry one chunk ahead
        struct G64 {
            double mx, my, a, b, c;
            float o;
        };
        auto ld_geo = [&](uint32_t r) {
            const GeomRec* g = A.geom + r;
            return G64{g->mx, g->my, g->a64, g->b64, g->c64, g->opacity};
        };
        uint32_t r_cur = (beg + lane < end) ? A.entries[beg + lane] : 0u;
        uint32_t r_nxt = (beg + 32 + lane < end) ? A.entries[beg + 32 + lane] : 0u;
        G64 g_cur = (beg + lane < end) ? ld_geo(r_cur) : G64{};
        for (uint32_t i0 = beg; i0 < end && T >= SF_EARLY_EXIT_T; i0 += 32) {
            const uint32_t i = i0 + lane;
            const uint32_t r_n2 = (i + 64 < end) ? A.entries[i + 64] : 0u;
            const G64 g_nxt = (i + 32 < end) ? ld_geo(r_nxt) : G64{};
            double al = 0.0;
            const uint32_t r = r_cur;
            if (i < end) {
                const G64& g = g_cur;
                double ddx = __dadd_rn(pxd, -g.mx), ddy = __dadd_rn(pyd, -g.my);
                double t1 = __dmul_rn(__dmul_rn(g.a, ddx), ddx);
                double t2 = __dmul_rn(__dmul_rn(__dmul_rn(2.0, g.b), ddx), ddy);
                double t3 = __dmul_rn(__dmul_rn(g.c, ddy), ddy);
                double q = __dadd_rn(__dadd_rn(t1, t2), t3);
                if (q <= SF_CUTOFF)
                    al = np_minimum(__dmul_rn((double)g.o, exp(__dmul_rn(-0.5, q))), SF_ALPHA_CLAMP);
            }
            r_cur = r_nxt;
            r_nxt = r_n2;
            g_cur = g_nxt;
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
            // Ordered accumulation (deterministic, the reference's order,
            // sparse_splat.py:144-147): entries in list order, a channel is
            // owned by lane ch % 32, so each channel's sum runs in depth order.
            const double e_mine = counted ? __dmul_rn(al, Tb) : 0.0;
            unsigned live = __ballot_sync(0xffffffffu, counted);
            while (live) {
                const int j = __ffs(live) - 1;
                live &= live - 1;
                const double e = __shfl_sync(0xffffffffu, e_mine, j);
                const uint32_t rj = __shfl_sync(0xffffffffu, r, j);
                const unsigned char* rec = A.chan + (size_t)rj * cs;
                const uint32_t* words = reinterpret_cast<const uint32_t*>(rec);
                const float* val = reinterpret_cast<const float*>(rec + voff);
                for (int k = 0; k < C; ++k) {
                    const int ch = chan_id(words[k]);
                    if ((ch & 31) == lane) {
                        if (local) wl[ch] += e * (double)val[k];
                        else row[ch] += (float)(e * (double)val[k]);
                    }
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
        if (local && A.features) {
            // the fused decode used the fp32 tile: redo this pixel's features
            // from the exact coefficients (fp32 FMA over L = 64 terms: ~4e-6
            // relative, inside the 3-term tensor-core tolerance); lanes own
            // columns n = lane + 32 i, so codebook rows are read coalesced
            for (int b = 0; b < A.n_levels; ++b) {
                const float* cb = A.codebooks + (size_t)A.lv.lv[b] * A.L * A.D;
                float* fo = A.features + (size_t)b * A.feat_level_stride + pix * A.D;
                for (int n0 = 0; n0 < A.D; n0 += 32 * 8) {
                    float f[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) f[i] = 0.f;
                    for (int l = 0; l < A.L; ++l) {
                        const float w = (float)wl[b * A.L + l];
                        const float* row = cb + (size_t)l * A.D + n0 + lane;
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            if (n0 + lane + 32 * i < A.D) f[i] = fmaf(w, __ldg(row + 32 * i), f[i]);
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if (n0 + lane + 32 * i < A.D) fo[n0 + lane + 32 * i] = f[i];
                }
            }
        }
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

bool blend_dec_supported(int n_levels, int L, int K, int D) {
    return L == 64 && n_levels * K == 12 && n_levels <= kDecMaxLevels && n_levels * L <= kChBlock && D >= kDecN &&
           D % kDecN == 0;
}
size_t blend_dec_image_bytes(int n_levels, int D) {
    return (size_t)n_levels * (D / kDecN) * kDecChunkBytes + 64;  // + per-level scales
}
void launch_dec_codebook_image(const float* codebooks, const LevelSelDev& lv, int L, int D, void* out,
                               cudaStream_t st) {
    unsigned char* img = (unsigned char*)out;
    float* scale = (float*)(img + (size_t)lv.n * (D / kDecN) * kDecChunkBytes);
    k_dec_codebook_image<<<lv.n * (D / kDecN), 256, 0, st>>>(codebooks, lv, L, D, img, scale);
}

// features (n_levels, H, W, D) fp32 as a 4-D TMA map: boxes of kDecBoxCols
// columns x 8 x 4 pixels of one level (a warp's fused-decode store box)
int make_feature_map(CUtensorMap* map, float* f, int D, int W, int H, int n_levels) {
    static const PFN_cuTensorMapEncodeTiled_v12000 enc = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)p;
    }();
    if (!enc) return -1;
    cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n_levels};
    cuuint64_t strides[3] = {(cuuint64_t)D * 4, (cuuint64_t)W * D * 4, (cuuint64_t)H * W * D * 4};
    cuuint32_t box[4] = {(cuuint32_t)kDecBoxCols, 8, 4, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, f, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     kDecBoxCols == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

// Transpose of the splat (train.py:324-330, the blend weights being constants
// of the coefficient optimisation):
//     ghat[b][row][k] = sum over pixels p of e_row(p) * dL/dW[p][b L + idx_bk]
// One 128-thread CTA per half tile, thread = pixel.  The tile's dL/dW rows sit
// in shared memory as dw[channel][pixel]; the list streams through in
// batches of 32 records; each warp walks its candidates (patch culling as in
// k_blend), recomputes alpha / T / e with the blend's rule, and reduces
// e * dW over its 32 pixels with shuffles into per-batch shared sums, which
// are added to ghat once per CTA and record.
constexpr int kTrBatch = 32;
__global__ void __launch_bounds__(128) k_splat_transpose(BlendArgs A, const float* __restrict__ dW,
                                                         float* __restrict__ ghat, int K, int64_t G) {
    extern __shared__ __align__(16) unsigned char smem_tr[];
    const int n_ch = A.n_ch, C = A.C;
    const int cs = chan_rec_bytes(C), voff = chan_val_offset(C);
    float* dw = reinterpret_cast<float*>(smem_tr);                                   // [n_ch][kAccPitch]
    GeomF32* g = reinterpret_cast<GeomF32*>(smem_tr + acc_bytes(n_ch));              // [32]
    uint32_t* rows = reinterpret_cast<uint32_t*>(g + kTrBatch);                      // [32]
    unsigned char* rec = reinterpret_cast<unsigned char*>(rows + kTrBatch);          // [32][cs]
    float* gsum = reinterpret_cast<float*>(rec + kTrBatch * cs);                     // [32][C]
    const int tile = A.tile0 + (blockIdx.x >> 1), half = blockIdx.x & 1;
    const int tx = tile % A.tiles_x, ty = tile / A.tiles_x;
    const int x0 = tx * SF_TILE, y0 = ty * SF_TILE;
    const int slot = threadIdx.x, lane = slot & 31, cw = slot >> 5;
    const int warp = half * kConsumerWarps + cw;
    const int px = x0 + (warp & 1) * 8 + (lane & 7), py = y0 + (warp >> 1) * 4 + (lane >> 3);
    const bool inside = px < A.W && py < A.H;
    if (A.stats[SF_STAT_OVERFLOW]) return;
    for (int i = threadIdx.x; i < kTilePixels * n_ch; i += blockDim.x) {
        const int sl = i / n_ch, c = i - sl * n_ch;
        const int w8 = half * kConsumerWarps + (sl >> 5), l8 = sl & 31;
        const int gx = x0 + (w8 & 1) * 8 + (l8 & 7), gy = y0 + (w8 >> 1) * 4 + (l8 >> 3);
        dw[c * kAccPitch + sl] = (gx < A.W && gy < A.H) ? dW[((size_t)gy * A.W + gx) * n_ch + c] : 0.f;
    }
    const float pxf = (float)px, pyf = (float)py;
    const double pxd = (double)px, pyd = (double)py;
    const float pdx0 = (float)(x0 + (warp & 1) * 8), pdy0 = (float)(y0 + (warp >> 1) * 4);
    float T = 1.f;
    bool done = !inside;
    const uint32_t beg = A.tile_offsets[tile], end = A.tile_offsets[tile + 1];
    for (uint32_t base = beg; base < end; base += kTrBatch) {
        const int nb = (int)min((uint32_t)kTrBatch, end - base);
        __syncthreads();  // previous batch flushed
        for (int i = threadIdx.x; i < nb; i += blockDim.x) {
            const uint32_t r = A.entries[base + i];
            rows[i] = r;
            g[i] = *reinterpret_cast<const GeomF32*>(A.geom + r);
        }
        for (int i = threadIdx.x; i < nb * cs / 16; i += blockDim.x) {
            const int j = i / (cs / 16), q = i - j * (cs / 16);
            reinterpret_cast<uint4*>(rec + j * cs)[q] =
                reinterpret_cast<const uint4*>(A.chan + (size_t)A.entries[base + j] * cs)[q];
        }
        for (int i = threadIdx.x; i < kTrBatch * C; i += blockDim.x) gsum[i] = 0.f;
        __syncthreads();
        uint32_t wmask = __ballot_sync(0xffffffffu, lane < nb && patch_may_hit(g[lane & 31], pdx0, pdy0));
        if (__all_sync(0xffffffffu, done)) wmask = 0;
        while (wmask) {
            const int j = __ffs(wmask) - 1;
            wmask &= wmask - 1;
            bool amb = false;
            float al = blend_alpha_fast(g[j], pxf, pyf, amb);
            if (amb) al = blend_alpha_exact(g[j], A.geom + rows[j], pxd, pyd);
            float e = 0.f;
            if (al > 0.f && !done) {
                e = al * T;
                T = fmaf(-al, T, T);
                if (A.early_exit && T < (float)SF_EARLY_EXIT_T) done = true;
            }
            if (!__any_sync(0xffffffffu, e > 0.f)) continue;
            const uint32_t* words = reinterpret_cast<const uint32_t*>(rec + j * cs);
            for (int k = 0; k < C; ++k) {
                float v = e * dw[chan_id(words[k]) * kAccPitch + slot];
#pragma unroll
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) atomicAdd(&gsum[j * C + k], v);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nb * C; i += blockDim.x) {
            const int j = i / C, k = i - j * C;
            const float v = gsum[i];
            if (v != 0.f) atomicAdd(&ghat[((size_t)(k / K) * G + rows[j]) * K + (k % K)], v);
        }
        if (__syncthreads_and(done)) break;
    }
}

int launch_splat_transpose(const BlendArgs& a, const float* dW, float* ghat, int K, int64_t G, cudaStream_t st) {
    if (a.n_ch > kChBlock || a.C > kMaxC || a.C % K) return -1;
    const int cs = chan_rec_bytes(a.C);
    const size_t smem = acc_bytes(a.n_ch) + kTrBatch * (sizeof(GeomF32) + 4 + cs + 4 * a.C);
    ensure_smem_attr((const void*)k_splat_transpose, smem);
    if (a.n_band_tiles > 0) k_splat_transpose<<<2 * a.n_band_tiles, 128, smem, st>>>(a, dW, ghat, K, G);
    return 0;
}

// CTA-per-pixel variant of k_blend_fixup (accumulators in one CTA's shared
// memory, n_ch <= kChBlock): 8 warps take 8 consecutive 32-entry chunks of
// the list per round, so a long replay takes 1/8 of the sequential chunk
// steps.  T before an entry = T before the round x the product of the earlier
// warps' (1 - alpha) x the warp's exclusive prefix product.
constexpr int kFxWarps = 8;
__global__ void __launch_bounds__(32 * kFxWarps, 3) k_blend_fixup_cta(BlendArgs A) {
    __shared__ double wl[kChBlock];
    __shared__ float wf[kChBlock];
    __shared__ double pv[32 * kFxWarps][kMaxC];
    __shared__ uint8_t chs[32 * kFxWarps][kMaxC];
    __shared__ uint16_t live_list[32 * kFxWarps];  // the round's adding entries, in list order
    __shared__ int wcnt[kFxWarps];
    __shared__ double wtot[kFxWarps];
    __shared__ double Tround, Tfinal;
    __shared__ unsigned int last_counted;
    const uint32_t count = min(*A.fixup_count, A.fixup_capacity);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        const_cast<int64_t*>(A.stats)[SF_STAT_FIXUPS] = (int64_t)*A.fixup_count;
    const int C = A.C;
    const int cs = chan_rec_bytes(C);
    const int voff = chan_val_offset(C);
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    const int kper = C / A.n_levels;  // plan slots per level (level-major plan, launch_pack_channels)
    constexpr double thr = SF_EARLY_EXIT_T;
    for (uint32_t idx = blockIdx.x; idx < count; idx += gridDim.x) {
        const uint32_t code = A.fixup_list[idx];
        const int tile = (int)(code >> 8), slot = (int)(code & 255u);
        const int w8 = slot >> 5, l8 = slot & 31;
        const int px = (tile % A.tiles_x) * SF_TILE + (w8 & 1) * 8 + (l8 & 7);
        const int py = (tile / A.tiles_x) * SF_TILE + (w8 >> 1) * 4 + (l8 >> 3);
        const size_t pix = (size_t)py * A.W + px;
        for (int c = tid; c < A.n_ch; c += blockDim.x) wl[c] = 0.0;
        if (tid == 0) {
            Tround = 1.0;
            Tfinal = -1.0;
        }
        __syncthreads();
        const double pxd = (double)px, pyd = (double)py;
        const uint32_t beg = A.tile_offsets[tile], end = A.tile_offsets[tile + 1];
        // the next round's entry is loaded (and its record prefetched) one round ahead
        uint32_t r_next = (beg + (uint32_t)tid < end) ? A.entries[beg + tid] : 0u;
        for (uint32_t r0 = beg; r0 < end; r0 += 32 * kFxWarps) {
            const double T = Tround;
            const uint32_t i = r0 + (uint32_t)(wid * 32 + lane);
            double al = 0.0;
            uint32_t r = r_next;
            {
                const uint32_t i2 = i + 32 * kFxWarps;
                r_next = i2 < end ? A.entries[i2] : 0u;
                if (i2 < end) {
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(A.geom + r_next));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(A.geom + r_next) + 64));
                }
            }
            if (i < end) {
                const GeomRec* g = A.geom + r;
                // fp32 pre-test: outside its guard band q32 > 9 certifies q > 9
                // (alpha = 0), so only the entries that touch the pixel take
                // the fp64 path (the fp32 record is 32 of the 80 bytes)
                bool amb = false;
                const float a32 = blend_alpha_fast(*reinterpret_cast<const GeomF32*>(g), (float)px, (float)py, amb);
                if (a32 > 0.f || amb) {
                    double ddx = __dadd_rn(pxd, -g->mx), ddy = __dadd_rn(pyd, -g->my);
                    double t1 = __dmul_rn(__dmul_rn(g->a64, ddx), ddx);
                    double t2 = __dmul_rn(__dmul_rn(__dmul_rn(2.0, g->b64), ddx), ddy);
                    double t3 = __dmul_rn(__dmul_rn(g->c64, ddy), ddy);
                    double q = __dadd_rn(__dadd_rn(t1, t2), t3);
                    if (q <= SF_CUTOFF)
                        al = np_minimum(__dmul_rn((double)g->opacity, exp(__dmul_rn(-0.5, q))), SF_ALPHA_CLAMP);
                }
            }
            const double f = __dadd_rn(1.0, -al);
            double incl = f;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl = __dmul_rn(v, incl);
            }
            if (lane == 31) wtot[wid] = incl;
            if (tid == 0) last_counted = 0u;
            __syncthreads();
            double pre = 1.0;
            for (int v = 0; v < wid; ++v) pre = __dmul_rn(pre, wtot[v]);
            double excl = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane == 0) excl = 1.0;
            const double Tb = __dmul_rn(__dmul_rn(T, pre), excl);
            const bool live = (i < end) && (Tb >= thr);
            // Ordered accumulation (deterministic, and the reference's order,
            // sparse_splat.py:144-147): entry t stages its C channel ids and
            // products e v; then thread c owns channel c and adds the round's
            // products to it in list order (only level c / L's K slots can hold c).
            const bool adds = live && al > 0.0;
            const uint32_t abal = __ballot_sync(0xffffffffu, adds);
            if (lane == 0) wcnt[wid] = __popc(abal);
            if (adds) {
                const double e = __dmul_rn(al, Tb);
                const unsigned char* rec = A.chan + (size_t)r * cs;
                const uint32_t* words = reinterpret_cast<const uint32_t*>(rec);
                const float* val = reinterpret_cast<const float*>(rec + voff);
                for (int k = 0; k < C; ++k) {
                    chs[tid][k] = (uint8_t)chan_id(words[k]);
                    pv[tid][k] = e * (double)val[k];
                }
            }
            const bool stop = __syncthreads_or((i < end) && !(Tb >= thr));
            // compact the adding entries (usually a small fraction of the round)
            int n_add = 0, woff = 0;
#pragma unroll
            for (int v = 0; v < kFxWarps; ++v) {
                woff += v < wid ? wcnt[v] : 0;
                n_add += wcnt[v];
            }
            if (adds) live_list[woff + __popc(abal & ((1u << lane) - 1u))] = (uint16_t)tid;
            __syncthreads();
            if (tid < A.n_ch) {
                const int c = tid, k0 = (c / A.L) * kper;
                double acc = wl[c];
                for (int u = 0; u < n_add; ++u) {
                    const int j = live_list[u];
                    for (int k = k0; k < k0 + kper; ++k)
                        if (chs[j][k] == c) acc += pv[j][k];
                }
                wl[c] = acc;
            }
            if (stop) {
                // final T = T after the last entry still counted (T is non-increasing);
                // none counted in this round: the T the round started with
                if (live) atomicMax(&last_counted, i + 1u);
                __syncthreads();
                if (live && last_counted == i + 1u) Tfinal = __dmul_rn(Tb, f);
                if (tid == 0 && last_counted == 0u) Tfinal = T;
                __syncthreads();
                break;
            }
            if (tid == 0) {
                double p = T;
                for (int v = 0; v < kFxWarps; ++v) p = __dmul_rn(p, wtot[v]);
                Tround = p;
            }
            __syncthreads();
        }
        const double Tend = Tfinal >= 0.0 ? Tfinal : Tround;
        if (A.coeff_map)
            for (int c = tid; c < A.n_ch; c += blockDim.x) A.coeff_map[pix * A.n_ch + c] = (float)wl[c];
        if (tid == 0 && A.final_t) A.final_t[pix] = (float)Tend;
        if (A.features && A.fixup_w && idx < A.fixup_w_capacity) {
            // the features are redone by k_fixup_decode for all replayed pixels at once
            for (int c = tid; c < A.n_ch; c += blockDim.x) A.fixup_w[(size_t)idx * A.n_ch + c] = (float)wl[c];
        } else if (A.features) {
            // the fused decode used the fp32 tile: redo this pixel's features from
            // the exact coefficients (fp32 FMA over L terms, ~4e-6 relative);
            // 8 outputs per thread at a time, as independent FMA chains
            for (int c = tid; c < A.n_ch; c += blockDim.x) wf[c] = (float)wl[c];
            __syncthreads();
            const int total = A.n_levels * A.D;
            for (int base = tid; base < total; base += 8 * blockDim.x) {
                float fv[8];
                const float* cbp[8];
                int wo[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int bn = min(base + k * (int)blockDim.x, total - 1);
                    const int b = bn / A.D, n = bn - b * A.D;
                    cbp[k] = A.codebooks + (size_t)A.lv.lv[b] * A.L * A.D + n;
                    wo[k] = b * A.L;
                    fv[k] = 0.f;
                }
                // 4 codebook rows in flight per chain (the loads are L2 hits:
                // latency, not bandwidth, bounds this loop)
                int l = 0;
                for (; l + 4 <= A.L; l += 4) {
                    float cv[4][8];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int k = 0; k < 8; ++k) cv[u][k] = __ldg(cbp[k] + (size_t)(l + u) * A.D);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int k = 0; k < 8; ++k) fv[k] = fmaf(wf[wo[k] + l + u], cv[u][k], fv[k]);
                }
                for (; l < A.L; ++l) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) fv[k] = fmaf(wf[wo[k] + l], __ldg(cbp[k] + (size_t)l * A.D), fv[k]);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int bn = base + k * (int)blockDim.x;
                    if (bn < total) {
                        const int b = bn / A.D, n = bn - b * A.D;
                        A.features[(size_t)b * A.feat_level_stride + pix * A.D + n] = fv[k];
                    }
                }
            }
        }
        if (A.proj_cb && A.relevancy_raw && tid < A.n_levels) {
            const int b = tid, nv = 1 + A.n_canon;
            const double* P = A.proj_cb + (size_t)b * A.L * nv;
            double best = INFINITY;
            for (int j = 1; j < nv; ++j) {
                double dj = 0.0;
                for (int l = 0; l < A.L; ++l) dj = fma((double)(float)wl[b * A.L + l], P[l * nv] - P[l * nv + j], dj);
                best = np_minimum(best, sigmoid2(dj));
            }
            A.relevancy_raw[(size_t)b * A.W * A.H + pix] = best;
        }
        __syncthreads();
    }
}

// Features of the replayed pixels from their exact coefficients (fixup_w,
// written by k_blend_fixup_cta): per CTA 32 pixels x 64 columns of one level,
// the codebook slice and the pixels' coefficients staged in shared memory;
// each output is the same fp32 FMA chain over l as the per-pixel recompute.
// Work items (pixel block, level, column block) are strided over a fixed grid
// (the pixel count is only known on the device).
int device_sm_count();
constexpr int kFdPix = 32, kFdCols = 64;
__global__ void __launch_bounds__(256, 4) k_fixup_decode(BlendArgs A) {
    __shared__ __align__(16) float cb[64][kFdCols];   // L <= 64 rows of the level's codebook slice
    __shared__ float wrow[kFdPix][65];  // the block's pixels' coefficients of the level (padded)
    __shared__ size_t pixs[kFdPix];
    const uint32_t count = min(min(*A.fixup_count, A.fixup_capacity), A.fixup_w_capacity);
    const int nblk = (int)((count + kFdPix - 1) / kFdPix), ncb = A.D / kFdCols;
    const int items = nblk * A.n_levels * ncb;
    const int L = A.L;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int pb = it / (A.n_levels * ncb), rem = it - pb * A.n_levels * ncb;
        const int b = rem / ncb, n0 = (rem - b * ncb) * kFdCols;
        const float* src = A.codebooks + (size_t)A.lv.lv[b] * L * A.D + n0;
        {
            // all loads in flight before the shared-memory stores (L2 latency, not bandwidth)
            float cv[16], wv[8];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int i = threadIdx.x + u * 256, l = i / kFdCols;
                cv[u] = l < L ? __ldg(src + (size_t)l * A.D + (i % kFdCols)) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = threadIdx.x + u * 256, p = i / 64, l = i % 64;
                const uint32_t idx = (uint32_t)(pb * kFdPix + p);
                wv[u] = (idx < count && l < L) ? A.fixup_w[(size_t)idx * A.n_ch + b * L + l] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int i = threadIdx.x + u * 256;
                cb[i / kFdCols][i % kFdCols] = cv[u];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = threadIdx.x + u * 256;
                wrow[i / 64][i % 64] = wv[u];
            }
        }
        if (threadIdx.x < kFdPix) {
            const uint32_t idx = (uint32_t)(pb * kFdPix + threadIdx.x);
            size_t pix = ~(size_t)0;
            if (idx < count) {
                const uint32_t code = A.fixup_list[idx];
                const int tile = (int)(code >> 8), slot = (int)(code & 255u);
                const int w8 = slot >> 5, l8 = slot & 31;
                const int px = (tile % A.tiles_x) * SF_TILE + (w8 & 1) * 8 + (l8 & 7);
                const int py = (tile / A.tiles_x) * SF_TILE + (w8 >> 1) * 4 + (l8 >> 3);
                pix = (size_t)py * A.W + px;
            }
            pixs[threadIdx.x] = pix;
        }
        __syncthreads();
        // thread: pixel t / 8, columns 8 (t % 8) .. + 8
        const int p = threadIdx.x >> 3, c0 = (threadIdx.x & 7) * 8;
        float fv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) fv[k] = 0.f;
#pragma unroll 8
        for (int l = 0; l < L; ++l) {
            const float w = wrow[p][l];
            const float4 q0 = *reinterpret_cast<const float4*>(&cb[l][c0]);  // 16-byte loads: conflict-free rows
            const float4 q1 = *reinterpret_cast<const float4*>(&cb[l][c0 + 4]);
            fv[0] = fmaf(w, q0.x, fv[0]), fv[1] = fmaf(w, q0.y, fv[1]), fv[2] = fmaf(w, q0.z, fv[2]), fv[3] = fmaf(w, q0.w, fv[3]);
            fv[4] = fmaf(w, q1.x, fv[4]), fv[5] = fmaf(w, q1.y, fv[5]), fv[6] = fmaf(w, q1.z, fv[6]), fv[7] = fmaf(w, q1.w, fv[7]);
        }
        if (pixs[p] != ~(size_t)0) {
            float4* dst = reinterpret_cast<float4*>(A.features + (size_t)b * A.feat_level_stride + pixs[p] * A.D + n0 + c0);
            dst[0] = make_float4(fv[0], fv[1], fv[2], fv[3]);
            dst[1] = make_float4(fv[4], fv[5], fv[6], fv[7]);
        }
        __syncthreads();
    }
}

// k_splat_tc (sf_splat_tc.cu) is the frame path for L = 64, <= 3 levels and
// 4 or no canonicals; k_blend serves the other shapes (wide / generic channel
// blocks, other canonical counts).  SF_BLEND_IMPL=legacy forces k_blend
// (A/B comparisons only).
bool splat_tc_supported(const BlendArgs& a);
int launch_splat_tc(const BlendArgs& a, cudaStream_t st);

int launch_blend(const BlendArgs& a, cudaStream_t st) {
    if (a.C > kMaxC) return -2;
    if (a.proj_cb && a.n_ch > kChBlock) return -3;  // fused relevancy needs every channel in one CTA
    const int n_tiles = a.n_band_tiles;
    static const bool legacy = [] {
        const char* e = getenv("SF_BLEND_IMPL");
        return e && strcmp(e, "legacy") == 0;
    }();
    if (!legacy && splat_tc_supported(a)) {
        const int r = launch_splat_tc(a, st);
        if (r) return r;
    } else {
        int ch_block = a.n_ch < kChBlock ? a.n_ch : kChBlock;
        int nblk = (a.n_ch + ch_block - 1) / ch_block;
        const bool dec = a.features != nullptr;
        CUtensorMap fmap;
        memset(&fmap, 0, sizeof(fmap));
        if (dec) {
            if (!blend_dec_supported(a.n_levels, a.L, a.C / a.n_levels, a.D) || nblk != 1 || !a.dec_b) return -4;
            if ((uintptr_t)a.features % 16) return -4;
            if (make_feature_map(&fmap, a.features, a.D, a.W, a.H, a.n_levels)) return -5;
        }
        size_t smem = (dec ? 1024 : 0) + acc_bytes(ch_block) + sizeof(BlendSmem);
        const bool fast = (a.C == 12 && nblk == 1);
        const int nc = a.proj_cb ? a.n_canon : 0;
        void (*kern)(BlendArgs, int, const CUtensorMap);
        if (dec && !a.proj_cb) kern = k_blend<12, true, 0, true>;
        else if (dec && nc == 4) kern = k_blend<12, true, 4, true>;
        else if (dec) kern = k_blend<12, true, -1, true>;
        else if (fast && !a.proj_cb) kern = k_blend<12, true, 0, false>;
        else if (fast && nc == 4) kern = k_blend<12, true, 4, false>;
        else if (fast) kern = k_blend<12, true, -1, false>;
        else kern = k_blend<0, false, -1, false>;
        if (ensure_smem_attr((const void*)kern, smem)) return -6;
        if (n_tiles > 0) kern<<<dim3(2 * n_tiles, nblk), kCTAThreads, smem, st>>>(a, ch_block, fmap);
    }
    if (n_tiles > 0 && a.fixup_list && a.early_exit) {
        if (a.n_ch <= kChBlock) {
            k_blend_fixup_cta<<<1184, 32 * kFxWarps, 0, st>>>(a);
            if (a.features && a.fixup_w) k_fixup_decode<<<4 * device_sm_count(), 256, 0, st>>>(a);
        }
        else k_blend_fixup<<<296, 32 * kFixWarps, 0, st>>>(a);
    }
    return 0;  // (relevancy for n_ch > one channel block: launch_relevancy_from_cmap by the caller)
}

}  // namespace sf
