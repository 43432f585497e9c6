// sf_splat_tc.cu -- K5/K6 + K7 as one persistent, warp-specialised kernel:
// the sparse-coefficient splat AND the codebook decode on the tcgen05 tensor
// cores, with the decode of half tile i overlapping the blend of half tile i+1.
//
// Reference: tile_blend_weights (rasterizer.py:133-181), the scatter of
// _splat_levels (sparse_splat.py:138-150) and decode (sparse_splat.py:183-199):
//     e_i(p) = alpha_i(p) T_i(p)  (counted iff T_i >= 1e-4),  T_{i+1} = T_i (1 - alpha_i)
//     W[p, cat_idx[i]] += e_i(p) cat_vals[i]           F_b = W_b @ atoms_b
//
// The scatter is a GEMM.  For a batch of 32 list entries the per-pixel blend
// weights form E (128 pixels x 32 entries) and the entries' sparse codes form
// V (32 entries x 192 channels, 12 nonzeros per row), so W += E V -- one
// 128 x 192 x 32 tensor-core product per batch replaces 12 x 32 dependent
// shared-memory read-modify-writes per pixel (the old kernel's latency chain).
// Precision: E and V are scaled by 2^12 and split into fp16 hi + lo; the MMA
// sums Eh Vh + Eh Vl + El Vh in fp32 (relative error ~2^-22 per product; the
// scaling keeps the lo parts normal down to 2^-15, below which the absolute
// error is < 2^-37).  W' = 2^24 W exactly.
//
// CTA = one SM (persistent, half tiles blockIdx.x + i gridDim.x), 10 warps:
//   warps 0-3  blend: pixel = TMEM lane (warp w owns lanes 32w..32w+31, an
//              8x4 patch).  Per batch: conservative patch test (ballot), fp32
//              alpha with the fp64 guard band, T walk, e -> E rows (fp16
//              hi/lo, 16-byte stores).  Per tile: W from TMEM, fused
//              relevancy (fp64), final T, early-exit ambiguity list, and the
//              in-place conversion of W into the decode's A operand.
//   warps 4-7  drain (DEC): accumulator -> registers -> 128B-swizzled boxes ->
//              TMA stores of features[level][y][x][col].
//   warp 8     producer: tile lists -> record ring (cp.async), sparse codes
//              -> dense V^T stage (scatter of 12 hi/lo pairs per entry; the
//              previous batch's 12 positions are cleared, not the whole stage).
//   warp 9     MMA issuer (one thread): E V batches into the W slot of the
//              blending tile, 3-term fp16 decode chunks (A = W from TMEM,
//              B = codebook chunk by bulk copy) of the previous tile.
// TMEM (512 columns): W/A slots [0,192) and [192,384) alternate by tile;
// two 64-column decode accumulators at [384,512).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "sf_blend_dev.cuh"
#include "sf_common.cuh"

namespace sf {
namespace tcs {

constexpr int kThreads = 320;
constexpr int kBlendWarps = 4;   // warps 0-3
constexpr int kDrainWarp0 = 4;   // warps 4-7
constexpr int kProdWarp = 8;
constexpr int kMmaWarp = 9;
constexpr int kStages = 3;
constexpr int kBatch = 32;
constexpr int kMaxLevels = 3;
constexpr int kMaxCh = 64 * kMaxLevels;
constexpr int kSlotCols = 192;
constexpr int kAccCol0 = 2 * kSlotCols;  // 384
constexpr int kDecN = 64;
constexpr int kChunkBytes = 2 * kDecN * 128;  // codebook chunk: {hi, lo} x 64 n x 64 k fp16, SW128
constexpr int kBStages = 2;
constexpr int kBoxCols = 32;
constexpr int kBoxBytes = 8 * 4 * kBoxCols * 4;  // 8 x 4 pixels x 32 fp32
constexpr int kEBytes = 128 * kBatch * 2;         // 8 KB per part
constexpr int kVBytes = kMaxCh * kBatch * 2;      // 12 KB per part
constexpr float kScale = 4096.f;                  // 2^12 on E, V and the decode's A
constexpr float kInvW = 1.f / 16777216.f;         // W = W' 2^-24
constexpr uint32_t kMaxC = 16;

struct __align__(1024) Smem {
    unsigned char bring[kBStages][kChunkBytes];  // decode B ring (SW128, 1024-aligned)
    unsigned char box[4][2][kBoxBytes];          // drain boxes (SW128, 1024-aligned)
    unsigned char ehi[kStages][kEBytes];         // E operand (K-major, no swizzle)
    unsigned char elo[kStages][kEBytes];
    unsigned char vhi[kStages][kVBytes];         // V^T operand (K-major, no swizzle)
    unsigned char vlo[kStages][kVBytes];
    GeomF32 g[kStages][kBatch];
    uint32_t row[kStages][kBatch];
    double pd[kMaxCh * 4];  // fused relevancy: Pd_j = P_q - P_cj per (level, l)
    int nb[kStages];
    int done_count;
    uint32_t contrib[2];   // per W slot: bit w = blend warp w's pixels got a contribution
    uint32_t dq_info[2];   // MMA -> drains, per tile in order: contrib of the tile
    uint64_t rec_full[kStages], ev_full[kStages], ev_empty[kStages];
    uint64_t w_full[2], a_ready[2], slot_free[2];
    uint64_t dq_full[2], dq_empty[2];
    uint64_t b_full[kBStages], acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};

__device__ __forceinline__ bool bar_test(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// K-major, no-swizzle operand: 8-row x 16-byte core matrices, K-adjacent ones
// 128 B apart (LBO), 8-row groups 512 B apart (SBO); 32 K per row group
__device__ __forceinline__ uint64_t ns_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)(128 >> 4) << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// two floats -> packed fp16 hi pair and lo pair (x = hi + lo + O(2^-22 x))
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(x0, x1);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t a, uint16_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(v) : "memory");
}
// byte offset of element (row r, k) in a K-major no-swizzle operand
__device__ __forceinline__ uint32_t ns_off(int r, int k) {
    return (uint32_t)((r >> 3) * 512 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

// development aid (SF_TC_PROGRESS=<mapped host address>): per CTA and role,
// the role's position, readable by the host while the kernel runs
__device__ __forceinline__ void progress(const BlendArgs& A, int role, uint32_t a, uint32_t b) {
    if (A.timeline)
        *reinterpret_cast<volatile uint64_t*>(A.timeline + (size_t)blockIdx.x * 16 + role) =
            ((uint64_t)a << 32) | (uint64_t)b | (1ull << 63);
}

template <int NC, bool DEC>
__global__ void __launch_bounds__(kThreads, 1) k_splat_tc(BlendArgs A, const __grid_constant__ CUtensorMap fmap) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t mis = (1024u - (smem_addr(smem_raw) & 1023u)) & 1023u;
    Smem& S = *reinterpret_cast<Smem*>(smem_raw + mis);
    if (A.stats[SF_STAT_OVERFLOW]) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_half = 2 * A.n_band_tiles;
    const int n_levels = A.n_levels, n_ch = A.n_ch;
    const int dchunks = DEC ? A.D / kDecN : 0;  // chunks per level
    const int nchunk = n_levels * dchunks;      // decode chunks per half tile
    const int n_my = (int)blockIdx.x < n_half ? (n_half - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            bar_init(&S.rec_full[s], 33);  // 32 cp.async arrivals + the producer's release of rows / nb
            bar_init(&S.ev_full[s], kBlendWarps + 1);
            bar_init(&S.ev_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            bar_init(&S.w_full[i], 1);
            bar_init(&S.a_ready[i], kBlendWarps);
            bar_init(&S.slot_free[i], DEC ? 1 : kBlendWarps);
            bar_init(&S.acc_full[i], 1);
            bar_init(&S.acc_empty[i], 4);
            bar_init(&S.dq_full[i], 1);
            bar_init(&S.dq_empty[i], 4);
        }
        for (int i = 0; i < kBStages; ++i) bar_init(&S.b_full[i], 1);
        S.done_count = 0;
        S.contrib[0] = S.contrib[1] = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // V stages start (and, between batches, are returned to) all zero
    {
        const uint32_t v0 = smem_addr(&S.vhi[0][0]);
        constexpr int n16 = 2 * kStages * kVBytes / 16;
        static_assert(offsetof(Smem, vlo) == offsetof(Smem, vhi) + kStages * kVBytes, "V parts adjacent");
        for (int i = threadIdx.x; i < n16; i += kThreads) sts128(v0 + 16 * i, 0u, 0u, 0u, 0u);
    }
    if (NC == 4 && A.proj_cb) {
        const int nv = 1 + A.n_canon;
        for (int i = threadIdx.x; i < n_ch * 4; i += kThreads) {
            const int j = i & 3, bl = i >> 2;
            S.pd[i] = A.proj_cb[(size_t)bl * nv] - A.proj_cb[(size_t)bl * nv + 1 + j];
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&S.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    proxy_fence();
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tm = S.tmem_base;

    if (warp == kProdWarp) {
        // ---------------- producer: records -> ring, sparse codes -> V^T ----------------
        const int C = A.C;
        const int cs = chan_rec_bytes(C), voff = chan_val_offset(C);
        const uint32_t vh0 = smem_addr(&S.vhi[0][0]), vl0 = smem_addr(&S.vlo[0][0]);
        // channel ids (u8) this lane wrote into the stage used 1, 2, 3 batches ago
        uint32_t old0[4] = {~0u, ~0u, ~0u, ~0u}, old1[4] = {~0u, ~0u, ~0u, ~0u}, old2[4] = {~0u, ~0u, ~0u, ~0u};
        int bs = 0;
        for (int it = 0; it < n_my; ++it) {
            const int ht = (int)blockIdx.x + it * (int)gridDim.x;
            const int tile = A.tile0 + (ht >> 1);
            const uint32_t beg = A.tile_offsets[tile], end = A.tile_offsets[tile + 1];
            auto entry = [&](uint32_t i) -> uint32_t { return i < end ? __ldg(A.entries + i) : 0u; };
            auto load_chan = [&](uint32_t r, bool ok, uint4 (&w)[4], float4 (&v)[4]) {
                const unsigned char* rec = A.chan + (size_t)r * cs;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const bool in = ok && 4 * q < C;
                    w[q] = in ? __ldg(reinterpret_cast<const uint4*>(rec) + q) : make_uint4(0, 0, 0, 0);
                    v[q] = in ? __ldg(reinterpret_cast<const float4*>(rec + voff) + q) : make_float4(0, 0, 0, 0);
                }
            };
            uint32_t e_cur = entry(beg + lane), e_next = entry(beg + kBatch + lane);
            if (beg + lane < end) prefetch_records(A, e_cur, cs);
            uint4 wc[4], wn[4];
            float4 vc[4], vn[4];
            load_chan(e_cur, beg + lane < end, wc, vc);
            for (int bi = 0;; ++bi) {
                const int s = bs % kStages;
                const uint32_t base = beg + (uint32_t)bi * kBatch;
                const uint32_t e_n2 = entry(base + 2 * kBatch + lane);
                if (base + kBatch + lane < end) prefetch_records(A, e_next, cs);
                if (bs >= kStages) bar_wait(&S.ev_empty[s], ((bs / kStages) - 1) & 1);
                const bool all_done = *reinterpret_cast<volatile int*>(&S.done_count) == kBlendWarps * (it + 1);
                const int nb = (base < end && !all_done) ? (int)min((uint32_t)kBatch, end - base) : 0;
                if (lane < nb) {
                    cp_async16(&S.g[s][lane], A.geom + e_cur);
                    cp_async16(reinterpret_cast<char*>(&S.g[s][lane]) + 16, reinterpret_cast<const char*>(A.geom + e_cur) + 16);
                    S.row[s][lane] = e_cur;
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(&S.rec_full[s]))
                             : "memory");
                if (lane == 0) S.nb[s] = nb;
                __syncwarp();
                if (lane == 0) bar_arrive(&S.rec_full[s]);
                // the next batch's codes load while this batch's V^T is built
                const bool nxt_ok = nb == kBatch && base + kBatch + lane < end;
                load_chan(e_next, nxt_ok, wn, vn);
                const uint32_t vh = vh0 + s * kVBytes, vl = vl0 + s * kVBytes;
                // clear what this lane wrote into the stage last time (column k = lane)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t n = (old0[q] >> (8 * e)) & 0xFFu;
                        if (n != 0xFFu) {
                            const uint32_t o = ns_off((int)n, lane);
                            sts16(vh + o, 0);
                            sts16(vl + o, 0);
                        }
                    }
                }
                uint32_t nw[4] = {~0u, ~0u, ~0u, ~0u};
                if (lane < nb) {
                    const uint32_t wv[16] = {wc[0].x, wc[0].y, wc[0].z, wc[0].w, wc[1].x, wc[1].y, wc[1].z, wc[1].w,
                                             wc[2].x, wc[2].y, wc[2].z, wc[2].w, wc[3].x, wc[3].y, wc[3].z, wc[3].w};
                    const float fv[16] = {vc[0].x, vc[0].y, vc[0].z, vc[0].w, vc[1].x, vc[1].y, vc[1].z, vc[1].w,
                                          vc[2].x, vc[2].y, vc[2].z, vc[2].w, vc[3].x, vc[3].y, vc[3].z, vc[3].w};
#pragma unroll
                    for (int c = 0; c < (int)kMaxC; c += 2) {
                        if (c < C) {
                            const uint32_t n0 = wv[c] / kChanWord;
                            const bool two = c + 1 < C;
                            const uint32_t n1 = two ? wv[c + 1] / kChanWord : 0u;
                            uint32_t hi, lo;
                            split2(fv[c] * kScale, two ? fv[c + 1] * kScale : 0.f, hi, lo);
                            const uint32_t o0 = ns_off((int)n0, lane);
                            sts16(vh + o0, (uint16_t)(hi & 0xFFFFu));
                            sts16(vl + o0, (uint16_t)(lo & 0xFFFFu));
                            nw[c >> 2] = (nw[c >> 2] & ~(0xFFu << (8 * (c & 3)))) | (n0 << (8 * (c & 3)));
                            if (two) {
                                const uint32_t o1 = ns_off((int)n1, lane);
                                sts16(vh + o1, (uint16_t)(hi >> 16));
                                sts16(vl + o1, (uint16_t)(lo >> 16));
                                nw[(c + 1) >> 2] =
                                    (nw[(c + 1) >> 2] & ~(0xFFu << (8 * ((c + 1) & 3)))) | (n1 << (8 * ((c + 1) & 3)));
                            }
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    old0[q] = old1[q];
                    old1[q] = old2[q];
                    old2[q] = nw[q];
                }
                proxy_fence();
                __syncwarp();
                if (lane == 0) bar_arrive(&S.ev_full[s]);
                ++bs;
                if (lane == 0) progress(A, 0, (uint32_t)it, (uint32_t)bs);
                if (nb == 0) break;
                e_cur = e_next;
                e_next = e_n2;
#pragma unroll
                for (int q = 0; q < 4; ++q) wc[q] = wn[q], vc[q] = vn[q];
            }
        }
    } else if (warp < kBlendWarps) {
        // ---------------- blend warps: E rows per batch, W epilogue per tile ----------------
        const int cw = warp;
        const int m = 32 * cw + lane;  // MMA row = TMEM lane = pixel slot in the half tile
        const uint32_t lane_off = (uint32_t)(32 * cw) << 16;
        const uint32_t eh0 = smem_addr(&S.ehi[0][0]) + (uint32_t)((m >> 3) * 512 + (m & 7) * 16);
        const uint32_t el0 = smem_addr(&S.elo[0][0]) + (uint32_t)((m >> 3) * 512 + (m & 7) * 16);
        const bool rel = NC == 4 && A.proj_cb != nullptr;
        int bs = 0;
        uint32_t zero_mask = 0;  // stages whose E rows of this warp are all zero
        for (int it = 0; it < n_my; ++it) {
            const int ht = (int)blockIdx.x + it * (int)gridDim.x;
            const int slot = it & 1;
            const int tile = A.tile0 + (ht >> 1), half = ht & 1;
            const int x0 = (tile % A.tiles_x) * SF_TILE, y0 = (tile / A.tiles_x) * SF_TILE;
            const int w8 = half * 4 + cw;
            const int px = x0 + (w8 & 1) * 8 + (lane & 7), py = y0 + (w8 >> 1) * 4 + (lane >> 3);
            const bool inside = px < A.W && py < A.H;
            const float pxf = (float)px, pyf = (float)py;
            const double pxd = (double)px, pyd = (double)py;
            const float pdx0 = (float)(x0 + (w8 & 1) * 8), pdy0 = (float)(y0 + (w8 >> 1) * 4);
            float T = 1.f, eb = 0.f, Tprev = 1.f;
            int ncontrib = 0, nbatches = 0;
            bool done = !inside;
            bool warp_done = __all_sync(0xffffffffu, done);
            bool counted = warp_done;
            if (warp_done && lane == 0) atomicAdd(&S.done_count, 1);
            for (;;) {
                const int s = bs % kStages;
                bar_wait(&S.rec_full[s], (bs / kStages) & 1);
                const int nb = *reinterpret_cast<volatile int*>(&S.nb[s]);
                if (nb == 0) {
                    __syncwarp();
                    if (lane == 0) bar_arrive(&S.ev_full[s]);
                    ++bs;
                    break;
                }
                ++nbatches;
                const uint32_t eh = eh0 + s * kEBytes, el = el0 + s * kEBytes;
                if (!warp_done) {
                    const GeomF32* G = S.g[s];
                    const uint32_t wcand = __ballot_sync(0xffffffffu, lane < nb && patch_may_hit(G[lane], pdx0, pdy0));
#pragma unroll
                    for (int g4 = 0; g4 < 4; ++g4) {
                        const uint32_t byte = (wcand >> (8 * g4)) & 0xFFu;
                        uint32_t hw[4] = {0u, 0u, 0u, 0u}, lw[4] = {0u, 0u, 0u, 0u};
                        if (byte) {
                            float alv[8];
                            uint32_t amb = 0;
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                bool gb = false;
                                alv[u] = ((byte >> u) & 1u) ? blend_alpha_fast(G[8 * g4 + u], pxf, pyf, gb) : 0.f;
                                amb |= (gb ? 1u : 0u) << u;
                            }
                            if (__any_sync(0xffffffffu, amb != 0)) {
                                for (int u = 0; u < 8; ++u)
                                    if (amb & (1u << u))
                                        alv[u] = blend_alpha_exact(G[8 * g4 + u], A.geom + S.row[s][8 * g4 + u], pxd, pyd);
                            }
                            float ev[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const float al = alv[u];
                                const bool live = al > 0.f && !done;
                                ev[u] = live ? al * T : 0.f;
                                if (live) {
                                    Tprev = T;
                                    T = fmaf(-al, T, T);
                                    eb = fmaf(al, rcp_approx(1.f - al), eb);  // 1 - al in [0.01, 1]
                                    ++ncontrib;
                                    if (A.early_exit && T < (float)SF_EARLY_EXIT_T) done = true;
                                }
                            }
#pragma unroll
                            for (int i = 0; i < 4; ++i) split2(ev[2 * i] * kScale, ev[2 * i + 1] * kScale, hw[i], lw[i]);
                        }
                        sts128(eh + 128 * g4, hw[0], hw[1], hw[2], hw[3]);
                        sts128(el + 128 * g4, lw[0], lw[1], lw[2], lw[3]);
                    }
                    zero_mask &= ~(1u << s);
                } else if (!((zero_mask >> s) & 1u)) {
#pragma unroll
                    for (int g4 = 0; g4 < 4; ++g4) {
                        sts128(eh + 128 * g4, 0u, 0u, 0u, 0u);
                        sts128(el + 128 * g4, 0u, 0u, 0u, 0u);
                    }
                    zero_mask |= 1u << s;
                }
                proxy_fence();
                __syncwarp();
                if (lane == 0) bar_arrive(&S.ev_full[s]);
                ++bs;
                if (!warp_done && __all_sync(0xffffffffu, done)) {
                    warp_done = true;
                    if (!counted && lane == 0) atomicAdd(&S.done_count, 1);
                    counted = true;
                }
            }
            if (!counted && lane == 0) atomicAdd(&S.done_count, 1);

            // ---- per-tile epilogue ----
            if (inside && A.early_exit && A.fixup_list) {
                // early-exit decisions fp32 cannot certify: replayed in fp64 by k_blend_fixup_cta
                const float tol = fmaf(4e-6f, eb, fmaf(3e-7f, (float)ncontrib, 2e-6f));
                const float thr = (float)SF_EARLY_EXIT_T;
                const bool amb = done ? (Tprev < thr * (1.f + tol) || T > thr * (1.f - tol)) : (T < thr * (1.f + tol));
                if (amb) {
                    const uint32_t k = atomicAdd(A.fixup_count, 1u);
                    if (k < A.fixup_capacity) A.fixup_list[k] = ((uint32_t)tile << 8) | (uint32_t)(half * 128 + m);
                }
            }
            if (A.final_t && inside) A.final_t[(size_t)py * A.W + px] = T;
            const bool any = __any_sync(0xffffffffu, ncontrib > 0);
            if (lane == 0) progress(A, 1 + cw, (uint32_t)it, 0x10000u | (uint32_t)bs);
            bar_wait(&S.w_full[slot], (it >> 1) & 1);
            if (lane == 0) progress(A, 1 + cw, (uint32_t)it, 0x20000u | (uint32_t)bs);
            // published only now: the W slot's previous tile (it - 2) has been
            // fully decoded (its slot_free preceded this tile's E V products),
            // so the MMA issuer has read that tile's flag
            if (lane == 0) {
                if (any) atomicOr(&S.contrib[slot], 1u << cw);
                else atomicAnd(&S.contrib[slot], ~(1u << cw));
            }
            tc_after();
            const uint32_t wcol = tm + lane_off + (uint32_t)(slot * kSlotCols);
            const size_t pix = (size_t)py * A.W + px;
            for (int b = 0; b < n_levels; ++b) {
                double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0, f0 = 0.0, f1 = 0.0, f2 = 0.0, f3 = 0.0;
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    uint32_t v[32];
                    const uint32_t col = wcol + (uint32_t)(64 * b + 32 * h);
                    if (nbatches) {
                        tmem_ld32(col, v);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = 0u;
                    }
                    float w[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) w[i] = __uint_as_float(v[i]) * kInvW;
                    if (rel) {
                        const double* P = S.pd + (size_t)(64 * b + 32 * h) * 4;
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const double2 a01 = *reinterpret_cast<const double2*>(P + 4 * i);
                            const double2 a23 = *reinterpret_cast<const double2*>(P + 4 * i + 2);
                            const double2 b01 = *reinterpret_cast<const double2*>(P + 4 * i + 4);
                            const double2 b23 = *reinterpret_cast<const double2*>(P + 4 * i + 6);
                            const double x = (double)w[i], y = (double)w[i + 1];
                            d0 = fma(x, a01.x, d0), d1 = fma(x, a01.y, d1), d2 = fma(x, a23.x, d2), d3 = fma(x, a23.y, d3);
                            f0 = fma(y, b01.x, f0), f1 = fma(y, b01.y, f1), f2 = fma(y, b23.x, f2), f3 = fma(y, b23.y, f3);
                        }
                    }
                    if (A.coeff_map && inside) {
                        float4* dst = reinterpret_cast<float4*>(A.coeff_map + pix * n_ch + 64 * b + 32 * h);
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            __stcs(dst + i, make_float4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]));
                    }
                    if (DEC) {
                        uint32_t hi[16], lo[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) split2(w[2 * i] * kScale, w[2 * i + 1] * kScale, hi[i], lo[i]);
                        tmem_st16(col, hi);
                        tmem_st16(col + 16, lo);
                    }
                }
                if (rel && inside) {
                    d0 += f0, d1 += f1, d2 += f2, d3 += f3;
                    // sigmoid is monotone: min_j sigmoid(d_j) = sigmoid(min_j d_j)
                    A.relevancy_raw[(size_t)b * A.W * A.H + pix] =
                        sigmoid2(np_minimum(np_minimum(d0, d1), np_minimum(d2, d3)));
                }
            }
            if (DEC) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_before();
            __syncwarp();
            if (lane == 0) bar_arrive(DEC ? &S.a_ready[slot] : &S.slot_free[slot]);
        }
    } else if (warp < kDrainWarp0 + 4) {
        // ---------------- drain warps: accumulators -> swizzled boxes -> TMA stores ----------------
        if (DEC) {
            const int q = warp - kDrainWarp0;  // TMEM lane quarter = pixel patch
            const uint32_t lane_off = (uint32_t)(32 * q) << 16;
            unsigned char* wbox = S.box[q][0];
            float scl[kMaxLevels];
#pragma unroll
            for (int b = 0; b < kMaxLevels; ++b) scl[b] = (b < n_levels ? A.dec_scale[b] : 1.f) / kScale;
            int Gd = 0;
            bool box_zero = false;
            for (int it = 0; it < n_my; ++it) {
                const int ht = (int)blockIdx.x + it * (int)gridDim.x;
                const int slot = it & 1;
                const int tile = A.tile0 + (ht >> 1), half = ht & 1;
                const int w8 = half * 4 + q;
                const int bx = (tile % A.tiles_x) * SF_TILE + (w8 & 1) * 8, by = (tile / A.tiles_x) * SF_TILE + (w8 >> 1) * 4;
                if (lane == 0) progress(A, 5 + q, (uint32_t)it, 0x10000u | (uint32_t)Gd);
                bar_wait(&S.dq_full[slot], (it >> 1) & 1);
                if (lane == 0) progress(A, 5 + q, (uint32_t)it, 0x20000u | (uint32_t)Gd);
                const bool contrib = *reinterpret_cast<volatile uint32_t*>(&S.dq_info[slot]) != 0u;
                __syncwarp();
                if (lane == 0) bar_arrive(&S.dq_empty[slot]);
                if (!contrib) {
                    // no contribution anywhere in the half tile: its features are zero
                    if (!box_zero) {
                        if (lane == 0) bulk_wait_read<0>();
                        __syncwarp();
                        for (int i = lane; i < 2 * kBoxBytes / 16; i += 32) sts128(smem_addr(wbox) + 16 * i, 0u, 0u, 0u, 0u);
                        proxy_fence();
                        __syncwarp();
                        box_zero = true;
                    }
                    if (lane == 0) {
                        for (int g = 0; g < nchunk; ++g) {
                            const int b = g / dchunks, c = g - b * dchunks;
                            tma_store_4d(&fmap, wbox, c * kDecN, bx, by, b);
                            tma_store_4d(&fmap, wbox + kBoxBytes, c * kDecN + kBoxCols, bx, by, b);
                        }
                        bulk_commit();
                    }
                    continue;
                }
                for (int g = 0; g < nchunk; ++g, ++Gd) {
                    const int t = Gd & 1, b = g / dchunks, c = g - b * dchunks;
                    if (lane == 0) progress(A, 5 + q, (uint32_t)it, 0x30000u | (uint32_t)Gd);
                    bar_wait(&S.acc_full[t], (Gd >> 1) & 1);
                    if (q == 0 && lane == 0) {
                        // chunk Gd's MMAs are complete: its codebook stage takes chunk Gd + 2
                        const int sg = Gd % kBStages;
                        bar_expect_tx(&S.b_full[sg], kChunkBytes);
                        bulk_g2s(S.bring[sg],
                                 reinterpret_cast<const unsigned char*>(A.dec_b) + (size_t)((Gd + kBStages) % nchunk) * kChunkBytes,
                                 kChunkBytes, &S.b_full[sg]);
                    }
                    tc_after();
                    uint32_t v[64];
                    tmem_ld32(tm + lane_off + (uint32_t)(kAccCol0 + t * kDecN), *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                    tmem_ld32(tm + lane_off + (uint32_t)(kAccCol0 + t * kDecN + 32), *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    tc_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(&S.acc_empty[t]);
                    const float sc = b == 0 ? scl[0] : (b == 1 ? scl[1] : scl[2]);
#pragma unroll
                    for (int i = 0; i < 64; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * sc);
                    if (lane == 0) bulk_wait_read<0>();  // the previous chunk's stores have left the boxes
                    __syncwarp();
#pragma unroll
                    for (int qq = 0; qq < 2; ++qq) {
                        const uint32_t row = smem_addr(wbox + qq * kBoxBytes) + lane * (kBoxCols * 4);
#pragma unroll
                        for (int u = 0; u < kBoxCols / 4; ++u) {
                            const int pu = u ^ (lane & 7);  // 128-byte swizzle
                            sts128(row + (pu << 4), v[32 * qq + 4 * u], v[32 * qq + 4 * u + 1], v[32 * qq + 4 * u + 2],
                                   v[32 * qq + 4 * u + 3]);
                        }
                    }
                    box_zero = false;
                    proxy_fence();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_4d(&fmap, wbox, c * kDecN, bx, by, b);
                        tma_store_4d(&fmap, wbox + kBoxBytes, c * kDecN + kBoxCols, bx, by, b);
                        bulk_commit();
                    }
                }
            }
            if (lane == 0) bulk_wait_read<0>();
            if (q == 0 && lane == 0) {
                // the two codebook loads still in flight (chunks Gd, Gd + 1) land before exit
                for (int G = Gd; G < Gd + kBStages; ++G) bar_wait(&S.b_full[G % kBStages], (G / kBStages) & 1);
            }
        }
    } else if (warp == kMmaWarp && lane == 0) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc_ev = (1u << 4) | ((uint32_t)(n_ch >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t idesc_dec = (1u << 4) | ((uint32_t)(kDecN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const unsigned char* img = reinterpret_cast<const unsigned char*>(A.dec_b);
        if (DEC) {
            for (int g = 0; g < kBStages; ++g) {
                bar_expect_tx(&S.b_full[g], kChunkBytes);
                bulk_g2s(S.bring[g], img + (size_t)(g % nchunk) * kChunkBytes, kChunkBytes, &S.b_full[g]);
            }
        }
        const uint32_t eh0 = smem_addr(&S.ehi[0][0]), el0 = smem_addr(&S.elo[0][0]);
        const uint32_t vh0 = smem_addr(&S.vhi[0][0]), vl0 = smem_addr(&S.vlo[0][0]);
        const uint64_t bdesc0 = sw128_desc(smem_addr(S.bring[0]));
        int te = 0, be = 0;
        bool first = true;
        int td = 0, cd = 0, Gd = 0;
        bool dactive = false;
        while (te < n_my || (DEC && td < n_my)) {
            bool prog = false;
            if (DEC && td < te) {
                if (!dactive && bar_test(&S.a_ready[td & 1], (td >> 1) & 1) &&
                    (td < 2 || bar_test(&S.dq_empty[td & 1], ((td >> 1) - 1) & 1))) {
                    tc_after();
                    // the drains learn the tile's kind in order, through their own ring
                    const uint32_t c = *reinterpret_cast<volatile uint32_t*>(&S.contrib[td & 1]);
                    S.dq_info[td & 1] = c;
                    bar_arrive(&S.dq_full[td & 1]);
                    if (c != 0u) {
                        dactive = true;
                        cd = 0;
                    } else {
                        bar_arrive(&S.slot_free[td & 1]);  // nothing to multiply: the slot is free now
                        ++td;
                    }
                    prog = true;
                }
                if (dactive) {
                    const int s = Gd % kBStages, t = Gd & 1;
                    if (bar_test(&S.b_full[s], (Gd / kBStages) & 1) &&
                        (Gd < 2 || bar_test(&S.acc_empty[t], ((Gd >> 1) - 1) & 1))) {
                        tc_after();
                        const int b = cd / dchunks;
                        const uint32_t d = tm + (uint32_t)(kAccCol0 + t * kDecN);
                        const uint64_t bd = bdesc0 + (uint64_t)((s * kChunkBytes) >> 4);
                        const uint32_t a0 = tm + (uint32_t)((td & 1) * kSlotCols + 64 * b);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {  // K steps of 16: Al Bh + Ah Bl + Ah Bh
                            const uint64_t bh = bd + 2 * k, bl = bh + ((kChunkBytes / 2) >> 4);
                            const uint32_t ah = a0 + (uint32_t)(32 * (k >> 1) + 8 * (k & 1)), al = ah + 16;
                            mma_f16_tmem_a(d, al, bh, idesc_dec, k > 0 ? 1u : 0u);
                            mma_f16_tmem_a(d, ah, bl, idesc_dec, 1u);
                            mma_f16_tmem_a(d, ah, bh, idesc_dec, 1u);
                        }
                        mma_commit(&S.acc_full[t]);
                        ++Gd;
                        if (++cd == nchunk) {
                            mma_commit(&S.slot_free[td & 1]);
                            ++td;
                            dactive = false;
                        }
                        prog = true;
                    }
                }
            }
            if (te < n_my) {
                const int s = be % kStages;
                const bool slot_ok = !first || te < 2 || bar_test(&S.slot_free[te & 1], ((te >> 1) - 1) & 1);
                if (slot_ok && bar_test(&S.ev_full[s], (be / kStages) & 1)) {
                    tc_after();
                    const int nb = *reinterpret_cast<volatile int*>(&S.nb[s]);
                    if (nb) {
                        const uint32_t d = tm + (uint32_t)((te & 1) * kSlotCols);
#pragma unroll
                        for (int k = 0; k < 2; ++k) {
                            const uint32_t o = 256u * k;
                            const uint64_t ah = ns_desc(eh0 + s * kEBytes + o), al = ns_desc(el0 + s * kEBytes + o);
                            const uint64_t bh = ns_desc(vh0 + s * kVBytes + o), bl = ns_desc(vl0 + s * kVBytes + o);
                            mma_f16_ss(d, ah, bh, idesc_ev, (first && k == 0) ? 0u : 1u);
                            mma_f16_ss(d, ah, bl, idesc_ev, 1u);
                            mma_f16_ss(d, al, bh, idesc_ev, 1u);
                        }
                        mma_commit(&S.ev_empty[s]);
                        first = false;
                    } else {
                        // end of the tile's stream: W complete once the issued MMAs are
                        if (!first) mma_commit(&S.w_full[te & 1]);
                        else bar_arrive(&S.w_full[te & 1]);
                        bar_arrive(&S.ev_empty[s]);
                        ++te;
                        first = true;
                    }
                    ++be;
                    prog = true;
                }
            }
            if (!prog) __nanosleep(20);
            else progress(A, 9, ((uint32_t)te << 16) | (uint32_t)td, ((uint32_t)be << 16) | (uint32_t)Gd);
        }
    }
    __syncwarp();
    tc_before();
    __syncthreads();
    if (warp == 0) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

}  // namespace tcs

size_t splat_tc_smem_bytes() { return sizeof(tcs::Smem) + 1024; }

bool splat_tc_supported(const BlendArgs& a) {
    if (a.L != 64 || a.n_levels < 1 || a.n_levels > tcs::kMaxLevels || a.n_ch != 64 * a.n_levels) return false;
    if (a.C < 1 || a.C > (int)tcs::kMaxC) return false;
    if (a.proj_cb && a.n_canon != 4) return false;
    if (a.features && (a.D % tcs::kDecN != 0 || !a.dec_b || (uintptr_t)a.features % 16)) return false;
    return true;
}

int make_feature_map(CUtensorMap* map, float* f, int D, int W, int H, int n_levels);
int ensure_smem_attr(const void* func, size_t bytes);
int device_sm_count();

int launch_splat_tc(const BlendArgs& a, cudaStream_t st) {
    if (!splat_tc_supported(a)) return -1;
    const bool dec = a.features != nullptr;
    CUtensorMap fmap;
    memset(&fmap, 0, sizeof(fmap));
    if (dec && make_feature_map(&fmap, a.features, a.D, a.W, a.H, a.n_levels)) return -5;
    const bool rel = a.proj_cb != nullptr;
    void (*kern)(BlendArgs, const CUtensorMap);
    if (dec) kern = rel ? tcs::k_splat_tc<4, true> : tcs::k_splat_tc<0, true>;
    else kern = rel ? tcs::k_splat_tc<4, false> : tcs::k_splat_tc<0, false>;
    const size_t smem = splat_tc_smem_bytes();
    if (ensure_smem_attr((const void*)kern, smem)) return -6;
    const int n_half = 2 * a.n_band_tiles;
    if (n_half <= 0) return 0;
    const int grid = std::min(n_half, device_sm_count());
    BlendArgs a2 = a;
    static const unsigned long long prog = [] {
        const char* e = getenv("SF_TC_PROGRESS");
        return e ? strtoull(e, nullptr, 10) : 0ull;
    }();
    a2.timeline = prog ? reinterpret_cast<uint64_t*>(prog) : nullptr;
    kern<<<grid, tcs::kThreads, smem, st>>>(a2, fmap);
    return 0;
}

}  // namespace sf
