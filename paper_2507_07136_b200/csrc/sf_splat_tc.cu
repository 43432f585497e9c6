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
// CTA = one SM (persistent; half tiles claimed dynamically through A.sched),
// 16 warps:
//   warps 0-7  blend: two per TMEM lane quarter (an 8x4 pixel patch); warp
//              hb = w >> 2 takes entries [16 hb, 16 hb + 16) of each batch.
//              Per batch: conservative patch test (ballot), fp32 alpha with
//              the fp64 guard band, the transmittance walk handed between the
//              pair, e -> E rows (fp16 hi/lo).  Per tile: W from TMEM (each
//              warp its own 32 columns per level), fused relevancy (fp64; the
//              pair's partial dots meet in E stage memory), final T, the
//              early-exit ambiguity list, and the in-place conversion of W
//              into the decode's A operand.
//   warps 8-11 drains (fused decode): accumulator -> registers -> 128B-swizzled
//              boxes -> TMA stores of features[level][y][x][col].
//   warp 12    producer: claims half tiles; tile lists -> record ring
//              (cp.async), sparse codes -> dense V^T stage (the previous
//              batch's 12 positions are cleared, not the whole stage).
//   warp 13    E V issuer (one thread): each batch's products into the W
//              slot of the blending tile.
//   warp 14    decode issuer (one thread): the 3-term fp16 decode chunks
//              (A = W from TMEM, B = codebook chunk) of the previous tile.
//   warp 15    codebook chunk loader (one thread, sleeps on its mbarrier).
//   Issuers block on mbarriers; each tcgen05.commit tracks only its own products.
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

constexpr int kThreads = 512;
constexpr int kBlendWarps = 8;   // warps 0-7: two per TMEM lane quarter
constexpr int kDrainWarp0 = 8;   // warps 8-11
constexpr int kProdWarp = 12;
constexpr int kMmaWarp = 13;   // E V issuer (one thread)
constexpr int kDecWarp = 14;   // decode issuer (one thread)
constexpr int kLoadWarp = 15;  // codebook chunk loader (one thread)
constexpr int kStages = 3;
constexpr int kBatch = 32;
#ifndef SF_AG
#define SF_AG 2
#endif
constexpr int kAG = SF_AG;  // alphas evaluated per group (the last group of a batch may run short)
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
constexpr float kScale = 4096.f;                  // 2^12 on E and V (keeps their fp16 lo parts normal)
constexpr float kInvW = 1.f / 16777216.f;         // W = W' 2^-24
constexpr uint32_t kMaxC = 12;  // channels per Gaussian (levels x K); more: legacy k_blend

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
    uint32_t ering[8][kBatch];          // producer: the half tile's filtered entries, 3 batches ahead
    unsigned char cring[3][kBatch][96]; // producer: the entries' sparse codes (plan records), 2 batches ahead
    float guard[kBlendWarps][kBatch];   // per blend warp: its batch entries' patch guard bands
    float alpha[4][2][16 * 32];         // per blend warp (quarter, hb): alphas of its <= 16 candidates x 32 pixels
    float4 hand[4][2][32];              // pair hand-off: (T, T before last, error bound, count | done)
    int nb[kStages];
    int sched[8];    // producer -> blend warps / E V issuer: half tile of iteration it (-1: no more)
    int a_ht[2];     // blend warps -> decode issuer, per W slot: the converted tile's half tile
    int dq_ht[2];    // decode issuer -> drains, per tile in order: half tile (-1: no more)
    int done_count;
    uint32_t contrib[2];   // per W slot: bit w = blend warp w's pixels got a contribution
    uint32_t dq_info[2];   // MMA -> drains, per tile in order: contrib of the tile
    uint32_t ev_tag[kStages];  // batch sequence number + 1 when some blend warp had a candidate in it
    uint32_t ev_union[kStages];  // profiling variant: entries of the batch that are some warp's candidate
    uint32_t tile_tag[2];      // per W slot: tile iteration + 1 when some batch of the tile had a candidate
    uint64_t rec_full[kStages], ev_full[kStages], ev_empty[kStages];
    uint64_t w_full[2], a_ready[2], slot_free[2];
    uint64_t dq_full[2], dq_empty[2];
    uint64_t b_full[kBStages], b_empty[kBStages], acc_full[2], acc_empty[2];
    uint64_t dec_done;  // the decode issuer's products have all completed
    int dec_total;  // decode issuer -> loader: chunks decoded in all (-1 while running)
    int loader_g;   // loader -> decode issuer: the chunk whose stage it waits for
    uint32_t tmem_base;
};

static_assert(sizeof(Smem) + 1024 <= 232448, "shared memory exceeds the 227 KB opt-in limit");

// wait for the phase up to about `ns` nanoseconds (the thread sleeps in
// hardware until the phase completes or the hint expires): true if it completed
__device__ __forceinline__ bool bar_wait_for(uint64_t* b, uint32_t parity, uint32_t ns) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_addr(b)), "r"(parity), "r"(ns)
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
        *reinterpret_cast<volatile uint64_t*>(A.timeline + (size_t)blockIdx.x * 128 + role) =
            ((uint64_t)a << 32) | (uint64_t)b | (1ull << 63);
}

// per-tile event timeline of CTA 0 (same aid): stamp[tile][event] at [148 * 128 + 16 * tile + event]
__device__ __forceinline__ void tl_stamp(const BlendArgs& A, int tile_it, int ev) {
    if (A.timeline && blockIdx.x == 0 && tile_it < 256)
        A.timeline[148 * 128 + 16 * tile_it + ev] = clock64();
}
// per-chunk decode timeline of CTA 0 (same aid): stamp[chunk][event] at [148 * 128 + 16 * 256 + 8 * Gd + event]
__device__ __forceinline__ void ch_stamp(const BlendArgs& A, int gd, int ev) {
    if (A.timeline && blockIdx.x == 0 && gd < 2048)
        A.timeline[148 * 128 + 16 * 256 + 8 * gd + ev] = clock64();
}
// cycle accounting (same aid): slot i of the CTA's 64 counters at [16, 80) of its 128
__device__ __forceinline__ void prof_add(const BlendArgs& A, int i, uint64_t v) {
    if (A.timeline) A.timeline[(size_t)blockIdx.x * 128 + 16 + i] += v;
}
#define SF_PROG(...)                       \
    do {                                   \
        if constexpr (prof) progress(__VA_ARGS__); \
    } while (0)
#define SF_STAMP(...)                      \
    do {                                   \
        if constexpr (prof) tl_stamp(__VA_ARGS__); \
    } while (0)
#define SF_CSTAMP(...)                     \
    do {                                   \
        if constexpr (prof) ch_stamp(__VA_ARGS__); \
    } while (0)
#define SF_TIMED(acc, stmt)                     \
    do {                                        \
        const uint64_t t0_ = prof ? clock64() : 0; \
        stmt;                                   \
        if (prof) acc += clock64() - t0_;       \
    } while (0)

template <int NC, bool DEC, bool PROF>
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
    // Half tiles are claimed dynamically (A.sched[0], zeroed per frame): a CTA
    // takes the next one when its producer starts streaming a tile, so SMs
    // that drew light tiles take more (tile cost varies ~100x across a frame).

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
        for (int i = 0; i < kBStages; ++i) {
            bar_init(&S.b_full[i], 1);
            bar_init(&S.b_empty[i], 1);
        }
        bar_init(&S.dec_done, 1);
        S.dec_total = -1;
        S.loader_g = -1;
        S.done_count = 0;
        S.contrib[0] = S.contrib[1] = 0u;
        for (int i = 0; i < kStages; ++i) S.ev_tag[i] = S.ev_union[i] = 0u;
        S.tile_tag[0] = S.tile_tag[1] = 0u;
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
    constexpr bool prof = PROF;  // the SF_TC_PROGRESS development variant: progress, cycle counters, timeline
    const uint64_t t_start = prof ? clock64() : 0;
    uint64_t w0 = 0, w1 = 0, w2 = 0;  // per-role wait counters (SF_TC_PROGRESS only)

    if (warp == kProdWarp) {
        // ---------------- producer: records -> ring, sparse codes -> V^T ----------------
        // The half tile's entries: the tile list filtered by the half-tile
        // flags (launch_binning: an entry without its half's flag has alpha = 0
        // at every pixel of the half) and compacted into ering, kept 3 batches
        // ahead; raw chunks of 32 entries are loaded two chunks ahead in
        // registers.  A cp.async pipeline for the rest: the entries' sparse
        // codes 2 batches ahead (cring), the geometry records of batch bi with
        // the stage's rec_full barrier.  Commit group G_bi = everything issued
        // in iteration bi; wait_group 2 at its end lands G_{bi-2}: batch bi's
        // codes.
        const int C = A.C;
        const int cs = chan_rec_bytes(C), voff = chan_val_offset(C);
        const int cq = cs / 16;
        const uint32_t vh0 = smem_addr(&S.vhi[0][0]), vl0 = smem_addr(&S.vlo[0][0]);
        // channel ids (u8) this lane wrote into the stage used 1, 2, 3 batches ago
        uint32_t old0[3] = {~0u, ~0u, ~0u}, old1[3] = {~0u, ~0u, ~0u}, old2[3] = {~0u, ~0u, ~0u};
        auto load_codes = [&](int slot3, uint32_t row) {
            const unsigned char* src = A.chan + (size_t)row * cs;
            unsigned char* dst = &S.cring[slot3][lane][0];
            for (int q = 0; q < cq; ++q) cp_async16(dst + 16 * q, src + 16 * q);
        };
        int bs = 0;
        auto claim = [&]() -> int {
            uint32_t x = 0;
            if (lane == 0) x = atomicAdd(A.sched, 1u);
            x = __shfl_sync(0xffffffffu, x, 0);
            return x < (uint32_t)n_half ? (int)x : -1;
        };
        int ht_next = claim();
        for (int it = 0;; ++it) {
            // the tile after this one is claimed now, so its first entries can be warmed in L2
            const int ht = ht_next;
            ht_next = ht >= 0 ? claim() : -1;
            if (lane == 0) S.sched[it & 7] = ht;  // published by the tile's first rec_full arrive
            // ht < 0: no more tiles -- one empty batch (nb = 0) tells every role
            const int tile = ht >= 0 ? A.tile0 + (ht >> 1) : 0;
            const uint32_t beg = ht >= 0 ? A.tile_offsets[tile] : 0u, end = ht >= 0 ? A.tile_offsets[tile + 1] : 0u;
            if (lane == 0) SF_STAMP(A, it, 9);
            if (ht_next >= 0 && lane < 4) {
                const int t2 = A.tile0 + (ht_next >> 1);
                const uint32_t b2 = A.tile_offsets[t2] + 32u * lane;
                if (b2 < A.tile_offsets[t2 + 1]) asm volatile("prefetch.global.L2 [%0];" ::"l"(A.entries + b2));
            }
            // filtered entry stream of this half tile
            const uint32_t hbit = 1u << (ht & 1);
            uint32_t rp = beg, nf = 0;  // next raw index, filtered entries so far
            uint32_t r0, f0, r1, f1;    // raw chunks at rp and rp + 32 (row, flags)
            auto load_raw = [&](uint32_t i, uint32_t& row, uint32_t& fl) {
                row = 0u;
                fl = 0u;
                if (i < end) {
                    row = __ldg(A.entries + i);
                    fl = A.entry_flags ? (uint32_t)__ldg(A.entry_flags + i) : 3u;
                }
            };
            load_raw(beg + lane, r0, f0);
            load_raw(beg + 32u + lane, r1, f1);
            auto fill = [&](uint32_t target) {
                while (nf < target && rp < end) {
                    uint32_t r2, f2;
                    load_raw(rp + 64u + lane, r2, f2);
                    if (lane == 0 && rp + 256u < end) {
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(A.entries + rp + 256u));
                        if (A.entry_flags) asm volatile("prefetch.global.L2 [%0];" ::"l"(A.entry_flags + rp + 256u));
                    }
                    const bool keep = rp + lane < end && (f0 & hbit) != 0u;
                    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                    if (keep) {
                        const uint32_t q = nf + (uint32_t)__popc(bal & ((1u << lane) - 1u));
                        S.ering[(q >> 5) & 7][q & 31] = r0;
                    }
                    nf += (uint32_t)__popc(bal);
                    rp += 32u;
                    r0 = r1, f0 = f1, r1 = r2, f1 = f2;
                }
                __syncwarp();
            };
            // prologue: filtered entries of batches 0..2, then the codes of batches 0, 1
            fill(3u * kBatch);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (32u * k + lane < nf) {
                    const uint32_t r = S.ering[k][lane];
                    load_codes(k, r);
                    prefetch_records(A, r, cs);
                }
                cp_async_commit();
            }
            for (int bi = 0;; ++bi) {
                const int s = bs % kStages;
                const uint32_t base = (uint32_t)bi * kBatch;  // in the filtered stream
                if (bs >= kStages) SF_TIMED(w0, bar_wait(&S.ev_empty[s], ((bs / kStages) - 1) & 1));
                const bool all_done = *reinterpret_cast<volatile int*>(&S.done_count) == kBlendWarps * (it + 1);
                if (!all_done) fill(base + 3u * kBatch);  // batches bi .. bi + 2 (fewer at the list's end)
                const int nb = (base < nf && !all_done) ? (int)min((uint32_t)kBatch, nf - base) : 0;
                const uint32_t row = S.ering[bi & 7][lane];
                if (lane < nb) {
                    cp_async16(&S.g[s][lane], A.geom + row);
                    cp_async16(reinterpret_cast<char*>(&S.g[s][lane]) + 16, reinterpret_cast<const char*>(A.geom + row) + 16);
                    S.row[s][lane] = row;
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(&S.rec_full[s]))
                             : "memory");
                if (lane == 0) S.nb[s] = nb;
                if (prof && nb) ++w1;
                if (prof) w2 += (uint64_t)nb;  // entries streamed
                __syncwarp();
                if (lane == 0) bar_arrive(&S.rec_full[s]);
                if (nb == kBatch) {
                    // codes of batch bi + 2
                    if (base + 2u * kBatch + lane < nf) {
                        const uint32_t r2 = S.ering[(bi + 2) & 7][lane];
                        load_codes((bi + 2) % 3, r2);
                        prefetch_records(A, r2, cs);
                    }
                }
                cp_async_commit();
                cp_async_wait<2>();  // G_{bi-2}: this batch's codes
                const uint32_t vh = vh0 + s * kVBytes, vl = vl0 + s * kVBytes;
                // clear what this lane wrote into the stage last time (column k = lane)
#pragma unroll
                for (int q = 0; q < 3; ++q) {
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
                uint32_t nw[3] = {~0u, ~0u, ~0u};
                if (lane < nb) {
                    const unsigned char* rec = &S.cring[bi % 3][lane][0];
                    uint32_t wv[12];
                    float fv[12];
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const uint4 w4 = q * 4 < C ? *reinterpret_cast<const uint4*>(rec + 16 * q) : make_uint4(0, 0, 0, 0);
                        const float4 v4 =
                            q * 4 < C ? *reinterpret_cast<const float4*>(rec + voff + 16 * q) : make_float4(0, 0, 0, 0);
                        wv[4 * q] = w4.x, wv[4 * q + 1] = w4.y, wv[4 * q + 2] = w4.z, wv[4 * q + 3] = w4.w;
                        fv[4 * q] = v4.x, fv[4 * q + 1] = v4.y, fv[4 * q + 2] = v4.z, fv[4 * q + 3] = v4.w;
                    }
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
                for (int q = 0; q < 3; ++q) {
                    old0[q] = old1[q];
                    old1[q] = old2[q];
                    old2[q] = nw[q];
                }
                proxy_fence();
                __syncwarp();
                if (lane == 0) bar_arrive(&S.ev_full[s]);
                ++bs;
                if (lane == 0) SF_PROG(A, 0, (uint32_t)it, (uint32_t)bs);
                if (nb == 0) {
                    if (lane == 0) SF_STAMP(A, it, 10);
                    break;
                }
            }
            cp_async_wait<0>();
            if (ht < 0) break;
        }
    } else if (warp < kBlendWarps) {
        // ---------------- blend warps: E rows per batch, W epilogue per tile ----------------
        // Warps w and w + 4 share TMEM lane quarter w & 3 (32 pixels, an 8x4
        // patch).  Warp hb = w >> 2 owns entries [16 hb, 16 hb + 16) of every
        // batch: both evaluate their alphas at once, then walk the
        // transmittance in depth order -- hb 0, hand the pixel state (T, T
        // before the last contribution, error bound, count / done) to hb 1
        // through shared memory and a named barrier, hb 1 walks, hands back.
        const int cw = warp & 3, hb = warp >> 2;
        const int m = 32 * cw + lane;  // MMA row = TMEM lane = pixel slot in the half tile
        const uint32_t lane_off = (uint32_t)(32 * cw) << 16;
        const uint32_t eh0 = smem_addr(&S.ehi[0][0]) + (uint32_t)((m >> 3) * 512 + (m & 7) * 16);
        const uint32_t el0 = smem_addr(&S.elo[0][0]) + (uint32_t)((m >> 3) * 512 + (m & 7) * 16);
        const bool rel = NC == 4 && A.proj_cb != nullptr;
        const bool early_exit = A.early_exit != 0;
        float* gsm = S.guard[warp];
        float* asc = S.alpha[cw][hb];          // [16][32] alphas of this warp's candidates
        float4* hand_out = S.hand[cw][hb];     // state this warp posts
        const float4* hand_in = S.hand[cw][hb ^ 1];
        const int bar_ab = 1 + cw, bar_ba = 5 + cw;  // named barriers of the pair (64 threads)
        const int bar_rd = 9 + cw;                    // hb 0 has read hb 1's partial relevancy dots
        const int e0 = 16 * hb;                       // first batch entry of this warp
        int bs = 0;
        uint32_t zero_mask = 0;  // stages whose E half-rows of this warp are all zero
        for (int it = 0;; ++it) {
            const int slot = it & 1;
            // the tile's first batch carries its half-tile index (S.sched)
            SF_TIMED(w0, bar_wait(&S.rec_full[bs % kStages], (bs / kStages) & 1));
            const int ht = *reinterpret_cast<volatile int*>(&S.sched[it & 7]);
            if (ht < 0) {
                // no more tiles: pass the empty batch on; once the E V issuer has
                // released this W slot (as for any tile), tell the decode issuer
                __syncwarp();
                if (lane == 0) bar_arrive(&S.ev_full[bs % kStages]);
                ++bs;
                SF_TIMED(w0, bar_wait(&S.w_full[slot], (it >> 1) & 1));
                if (lane == 0) {
                    S.a_ht[slot] = -1;
                    bar_arrive(DEC ? &S.a_ready[slot] : &S.slot_free[slot]);
                }
                break;
            }
            const int tile = A.tile0 + (ht >> 1), half = ht & 1;
            const int x0 = (tile % A.tiles_x) * SF_TILE, y0 = (tile / A.tiles_x) * SF_TILE;
            const int w8 = half * 4 + cw;
            const int px = x0 + (w8 & 1) * 8 + (lane & 7), py = y0 + (w8 >> 1) * 4 + (lane >> 3);
            const bool inside = px < A.W && py < A.H;
            const float pxf = (float)px, pyf = (float)py;
            const double pxd = (double)px, pyd = (double)py;
            const float pdx0 = (float)(x0 + (w8 & 1) * 8), pdy0 = (float)(y0 + (w8 >> 1) * 4);
            // this warp's entries only: T after / before its last counted entry,
            // error bound, count, batch of that entry + 1 (merged at the tile end)
            float Tw = 1.f, Tpw = 1.f, ebw = 0.f;
            int nw = 0, lastw = 0, nbatches = 0;
            float Trun = 1.f;  // hb 0: the running transmittance entering the batch
            bool tile_hit = false;  // some batch of this tile had a candidate for this warp
            bool done = !inside;
            if (warp == 0 && lane == 0) SF_STAMP(A, it, 0);
            bool all_done = __all_sync(0xffffffffu, done);
            bool counted = all_done;
            if (all_done && lane == 0) atomicAdd(&S.done_count, 1);
            // the pair's hand-off carries only the running transmittance: each warp
            // folds prod (1 - a) over its candidates into its alpha phase and passes
            // T_in prod on at once, before its own walk (the walk is off the chain)
            auto recv = [&](int id) -> float {
                named_bar_sync(id, 64);
                return hand_in[lane].x;
            };
            auto post = [&](int id, float t) {
                hand_out[lane].x = t;
                asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory");
            };
            for (;;) {
                const int s = bs % kStages;
                SF_TIMED(w0, bar_wait(&S.rec_full[s], (bs / kStages) & 1));
                const int nb = *reinterpret_cast<volatile int*>(&S.nb[s]);
                if (nb == 0) {
                    if (hb == 0 && nbatches > 0) Trun = recv(bar_ba);  // the running T after the tile
                    __syncwarp();
                    if (lane == 0) bar_arrive(&S.ev_full[s]);
                    ++bs;
                    break;
                }
                const uint32_t eh = eh0 + s * kEBytes + 256 * hb, el = el0 + s * kEBytes + 256 * hb;
                const GeomF32* G = S.g[s];
                // ---- alphas of this warp's candidates (before the hand-off) ----
                const uint64_t ta0 = prof ? clock64() : 0;
                uint32_t wmask = 0;
                float P = 1.f;  // prod (1 - a) over this warp's candidates, in depth order
                if (!all_done) {
                    bool hit = false;
                    if (lane < 16 && e0 + lane < nb) {
                        hit = patch_may_hit(G[e0 + lane], pdx0, pdy0);
                        gsm[lane] = patch_guard(G[e0 + lane], pdx0, pdy0);
                    }
                    wmask = __ballot_sync(0xffffffffu, hit);
                    __syncwarp();
                    int c0 = 0;
#pragma unroll 1
                    for (uint32_t wm = wmask; wm; c0 += kAG) {
                        int jj[kAG];
#pragma unroll
                        for (int u = 0; u < kAG; ++u) {
                            jj[u] = wm ? __ffs(wm) - 1 : -1;
                            wm &= wm - 1;
                        }
                        float alv[kAG];
                        bool anyamb = false;
                        uint32_t amb = 0;
#pragma unroll
                        for (int u = 0; u < kAG; ++u) {
                            const int j = jj[u] & 15;
                            bool gb = false;
                            alv[u] = blend_alpha_guarded(G[e0 + j], pxf, pyf, gsm[j], gb);
                            gb = gb && jj[u] >= 0;
                            amb |= (gb ? 1u : 0u) << u;
                            anyamb |= gb;
                        }
                        if (__any_sync(0xffffffffu, anyamb)) {
                            // rare; unrolled so alv stays in registers (a rolled loop
                            // indexes it dynamically and spills it on the common path)
#pragma unroll
                            for (int u = 0; u < kAG; ++u)
                                if (amb & (1u << u))
                                    alv[u] = blend_alpha_exact(G[e0 + jj[u]], A.geom + S.row[s][e0 + jj[u]], pxd, pyd);
                        }
#pragma unroll
                        for (int u = 0; u < kAG; ++u) {
                            if (c0 + u < 16) asc[(c0 + u) * 32 + lane] = alv[u];
                            if (jj[u] >= 0) P = fmaf(-alv[u], P, P);
                        }
                    }
                }
                // ---- E half-row: zero, then the candidates' e (hi, lo) ----
                if (wmask || !((zero_mask >> s) & 1u)) {
                    sts128(eh, 0u, 0u, 0u, 0u);
                    sts128(eh + 128, 0u, 0u, 0u, 0u);
                    sts128(el, 0u, 0u, 0u, 0u);
                    sts128(el + 128, 0u, 0u, 0u, 0u);
                }
                zero_mask = wmask ? (zero_mask & ~(1u << s)) : (zero_mask | (1u << s));
                // ---- hand-off in, transmittance walk in depth order, hand-off out ----
                if (prof) w1 += clock64() - ta0;
                float Tr;  // running transmittance before this warp's entries of the batch
                if (hb == 1) {
                    SF_TIMED(w0, Tr = recv(bar_ab));
                } else {
                    if (nbatches > 0) SF_TIMED(w0, Trun = recv(bar_ba));
                    Tr = Trun;
                }
                post(hb == 0 ? bar_ab : bar_ba, Tr * P);
                const uint64_t tw0 = prof ? clock64() : 0;
                {
                    int c = 0;
#pragma unroll 4
                    for (uint32_t wm = wmask; wm; ++c) {
                        const int j = __ffs(wm) - 1;
                        wm &= wm - 1;
                        // Tr runs through every entry (one FMA per entry carries the
                        // loop); an entry counts iff alpha > 0 and Tr before it >= 1e-4
                        // (T only falls, so that is the reference's early exit, and the
                        // counted entries see exactly the transmittance they saw before)
                        const float al = asc[c * 32 + lane];
                        const bool live = al > 0.f && inside && (!early_exit || Tr >= (float)SF_EARLY_EXIT_T);
                        const float alive = live ? al : 0.f;
                        const float e = alive * Tr;
                        Tpw = live ? Tr : Tpw;
                        Tr = fmaf(-al, Tr, Tr);
                        Tw = live ? Tr : Tw;
                        ebw = fmaf(alive, rcp_approx(1.f - alive), ebw);  // 1 - alive in [0.01, 1]
                        nw += live ? 1 : 0;
                        lastw = live ? nbatches + 1 : lastw;
                        const float x = e * kScale;
                        const __half h = __float2half_rn(x);
                        const __half l = __float2half_rn(x - __half2float(h));
                        const uint32_t o = (uint32_t)(2 * j + (j >> 3) * 112);  // (j >> 3) 128 + (j & 7) 2
                        sts16(eh + o, __half_as_ushort(h));
                        sts16(el + o, __half_as_ushort(l));
                    }
                }
                done = !inside || (early_exit && Tr < (float)SF_EARLY_EXIT_T);
                if (prof) w2 += clock64() - tw0;
                ++nbatches;
                // batches without a candidate in any warp have E = 0: the issuer skips them
                if (wmask && lane == 0) S.ev_tag[s] = (uint32_t)bs + 1u;
                if (prof && wmask && lane == 0) atomicOr(&S.ev_union[s], wmask << (16 * hb));
                tile_hit |= wmask != 0u;
                proxy_fence();
                __syncwarp();
                if (lane == 0) bar_arrive(&S.ev_full[s]);
                ++bs;
                if (!all_done && __all_sync(0xffffffffu, done)) {
                    all_done = true;
                    if (!counted && lane == 0) atomicAdd(&S.done_count, 1);
                    counted = true;
                }
            }
            if (!counted && lane == 0) atomicAdd(&S.done_count, 1);
            if (warp == 0 && lane == 0) SF_STAMP(A, it, 1);
            // W holds products iff some warp had a candidate in some batch (else
            // the issuer skipped every batch and the slot is stale): the 8 blend
            // warps agree on that through the tile tag
            if (tile_hit && lane == 0) S.tile_tag[slot] = (uint32_t)it + 1u;
            named_bar_sync(13, 32 * kBlendWarps);
            if (warp == 0 && lane == 0) SF_STAMP(A, it, 11);
            const bool wvalid = *reinterpret_cast<volatile uint32_t*>(&S.tile_tag[slot]) == (uint32_t)it + 1u;

            // ---- per-tile epilogue: hb 0 takes columns [0, 32) of each level, hb 1 [32, 64) ----
            const bool any = __any_sync(0xffffffffu, nw > 0);  // this warp's entries contributed somewhere
            if (lane == 0 && hb == 0) SF_PROG(A, 1 + cw, (uint32_t)it, 0x10000u | (uint32_t)bs);
            SF_TIMED(w0, bar_wait(&S.w_full[slot], (it >> 1) & 1));
            if (warp == 0 && lane == 0) SF_STAMP(A, it, 12);
            if (lane == 0 && hb == 0) SF_PROG(A, 1 + cw, (uint32_t)it, 0x20000u | (uint32_t)bs);
            // published only now: the W slot's previous tile (it - 2) has been
            // fully decoded (its slot_free preceded this tile's E V products),
            // so the decode issuer has read that tile's flag
            if (lane == 0) {
                if (any) atomicOr(&S.contrib[slot], 1u << warp);
                else atomicAnd(&S.contrib[slot], ~(1u << warp));
            }
            tc_after();
            const uint32_t wslot = tm + lane_off + (uint32_t)(slot * kSlotCols);
            const size_t pix = (size_t)py * A.W + px;
            // Compact code: this part runs once per tile per warp, so its
            // instructions are fetched cold -- loops stay rolled.
            // Each warp works on its own 32 columns of each level only (no
            // cross-warp TMEM dependency): its half of the fused relevancy dot
            // products (fp64, W (P_q - P_cj)), the coefficient map (if
            // requested) and, fused decode, the in-place A operand.  The pair's
            // partial dots meet in the quarter's rows of E stages 0-1 (no MMA
            // reads E between w_full and the next tile's batches).
            auto xslot = [&](int h, int b) -> double* {
                const int g = 3 * h + b;  // 6 groups of 32 px x 4 doubles: ehi[0], elo[0], ehi[1] quarter rows
                unsigned char* base = (g >> 1) == 0 ? (unsigned char*)&S.ehi[0][0]
                                                    : ((g >> 1) == 1 ? (unsigned char*)&S.elo[0][0] : (unsigned char*)&S.ehi[1][0]);
                return reinterpret_cast<double*>(base + cw * 2048 + (g & 1) * 1024) + 4 * lane;
            };
            // (1) the warp's partial relevancy dots over its own 32 columns of
            //     each level, 8 columns per step (compact code)
            if (rel) {
#pragma unroll 1
                for (int b = 0; b < n_levels; ++b) {
                    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0, f0 = 0.0, f1 = 0.0, f2 = 0.0, f3 = 0.0;
                    if (wvalid) {
#pragma unroll 1
                        for (int c = 32 * hb; c < 32 * hb + 32; c += 8) {
                            uint32_t v[8];
                            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                                           "=r"(v[7])
                                         : "r"(wslot + (uint32_t)(64 * b + c)));
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                            const double* P = S.pd + (size_t)(64 * b + c) * 4;
#pragma unroll
                            for (int i = 0; i < 8; i += 2) {
                                const double2 a01 = *reinterpret_cast<const double2*>(P + 4 * i);
                                const double2 a23 = *reinterpret_cast<const double2*>(P + 4 * i + 2);
                                const double2 b01 = *reinterpret_cast<const double2*>(P + 4 * i + 4);
                                const double2 b23 = *reinterpret_cast<const double2*>(P + 4 * i + 6);
                                const double x = (double)(__uint_as_float(v[i]) * kInvW);
                                const double y = (double)(__uint_as_float(v[i + 1]) * kInvW);
                                d0 = fma(x, a01.x, d0), d1 = fma(x, a01.y, d1), d2 = fma(x, a23.x, d2), d3 = fma(x, a23.y, d3);
                                f0 = fma(y, b01.x, f0), f1 = fma(y, b01.y, f1), f2 = fma(y, b23.x, f2), f3 = fma(y, b23.y, f3);
                            }
                        }
                    }
                    double2* o = reinterpret_cast<double2*>(xslot(hb, b));
                    o[0] = make_double2(d0 + f0, d1 + f1);
                    o[1] = make_double2(d2 + f2, d3 + f3);
                }
            }
            if (warp == 0 && lane == 0) SF_STAMP(A, it, 13);
            // (2) its 32 columns of each level -> coefficient map (if requested)
            //     and, fused decode, the A operand (fp16 hi/lo pairs of W 2^12) in place
            if (DEC || A.coeff_map) {
#pragma unroll 1
                for (int b = 0; b < n_levels; ++b) {
                    const uint32_t col = wslot + (uint32_t)(64 * b + 32 * hb);
                    uint32_t v[32];
                    if (wvalid) {
                        tmem_ld32(col, v);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = 0u;
                    }
                    if (A.coeff_map && inside) {
                        float4* dst = reinterpret_cast<float4*>(A.coeff_map + pix * n_ch + 64 * b + 32 * hb);
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            __stcs(dst + i, make_float4(__uint_as_float(v[4 * i]) * kInvW, __uint_as_float(v[4 * i + 1]) * kInvW,
                                                        __uint_as_float(v[4 * i + 2]) * kInvW,
                                                        __uint_as_float(v[4 * i + 3]) * kInvW));
                    }
                    if (DEC) {
                        // W = W' 2^-24: hi / lo of W itself (F = A B needs no rescale in the
                        // drains; a subnormal fp16 part costs < 3e-8 absolute per coefficient)
                        uint32_t hi[16], lo[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            split2(__uint_as_float(v[2 * i]) * kInvW, __uint_as_float(v[2 * i + 1]) * kInvW,
                                   hi[i], lo[i]);
                        tmem_st16(col, hi);
                        tmem_st16(col + 16, lo);
                    }
                }
            }
            if (DEC) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_before();
            __syncwarp();
            if (lane == 0) {
                S.a_ht[slot] = ht;
                bar_arrive(DEC ? &S.a_ready[slot] : &S.slot_free[slot]);
            }
            if (warp == 0 && lane == 0) SF_STAMP(A, it, 14);
            // hb 1 -> hb 0 (bar_ba, as after a batch): its per-pixel state and,
            // fused relevancy, its partial dots; hb 0 -> hb 1 (bar_rd): read,
            // hb 1 may write E / post again
            if (hb == 1) {
                hand_out[lane] = make_float4(Tw, Tpw, ebw, __int_as_float((nw << 12) | lastw));
                asm volatile("bar.arrive %0, 64;" ::"r"(bar_ba) : "memory");
                named_bar_sync(bar_rd, 64);
            } else {
                named_bar_sync(bar_ba, 64);
                const float4 st1 = hand_in[lane];
                double dm[kMaxLevels] = {0.0, 0.0, 0.0};
                if (rel) {
#pragma unroll
                    for (int b = 0; b < kMaxLevels; ++b) {
                        if (b < n_levels) {
                            const double2* p0 = reinterpret_cast<const double2*>(xslot(0, b));
                            const double2* p1 = reinterpret_cast<const double2*>(xslot(1, b));
                            const double2 a01 = p0[0], a23 = p0[1], b01 = p1[0], b23 = p1[1];
                            dm[b] = np_minimum(np_minimum(a01.x + b01.x, a01.y + b01.y), np_minimum(a23.x + b23.x, a23.y + b23.y));
                        }
                    }
                }
                asm volatile("bar.arrive %0, 64;" ::"r"(bar_rd) : "memory");  // hb 1 may go on while hb 0 finishes
                if (rel && inside) {
                    // sigmoid is monotone: min_j sigmoid(d_j) = sigmoid(min_j d_j)
#pragma unroll 1
                    for (int b = 0; b < n_levels; ++b) {
                        const double d = b == 0 ? dm[0] : (b == 1 ? dm[1] : dm[2]);
                        A.relevancy_raw[(size_t)b * A.W * A.H + pix] = sigmoid2(d);
                    }
                }
                // the pixel's state: the later of the two warps' last counted entries
                // (same batch: hb 1's entries come after hb 0's)
                const int c1 = __float_as_int(st1.w), n1 = c1 >> 12, last1 = c1 & 0xFFF;
                const bool one = n1 > 0 && last1 >= lastw;
                const float T = one ? st1.x : Tw, Tprev = one ? st1.y : Tpw;
                const float eb = ebw + st1.z;
                const int ncontrib = nw + n1;
                const float thr = (float)SF_EARLY_EXIT_T;
                const bool pdone = !inside || (early_exit && Trun < thr);
                if (inside && early_exit && A.fixup_list) {
                    // early-exit decisions fp32 cannot certify: replayed in fp64 by k_blend_fixup_cta
                    const float tol = fmaf(4e-6f, eb, fmaf(3e-7f, (float)ncontrib, 2e-6f));
                    const bool amb = pdone ? (Tprev < thr * (1.f + tol) || T > thr * (1.f - tol)) : (T < thr * (1.f + tol));
                    if (amb) {
                        const uint32_t k = atomicAdd(A.fixup_count, 1u);
                        if (k < A.fixup_capacity) A.fixup_list[k] = ((uint32_t)tile << 8) | (uint32_t)(half * 128 + m);
                    }
                }
                if (A.final_t && inside) A.final_t[pix] = T;
            }
            if (rel) zero_mask &= ~3u;  // the partials overwrote E rows of stages 0 and 1
            if (warp == 0 && lane == 0) SF_STAMP(A, it, 2);
        }
    } else if (warp < kDrainWarp0 + 4) {
        // ---------------- drain warps: accumulators -> swizzled boxes -> TMA stores ----------------
        if (DEC) {
            const int q = warp - kDrainWarp0;  // TMEM lane quarter = pixel patch
            const uint32_t lane_off = (uint32_t)(32 * q) << 16;
            unsigned char* wbox = S.box[q][0];
            float scl[kMaxLevels];
#pragma unroll
            for (int b = 0; b < kMaxLevels; ++b) scl[b] = b < n_levels ? A.dec_scale[b] : 1.f;  // 1 unless the atoms needed scaling
            int Gd = 0;
            bool box_zero = false;
            for (int it = 0;; ++it) {
                const int slot = it & 1;
                if (lane == 0) SF_PROG(A, 5 + q, (uint32_t)it, 0x10000u | (uint32_t)Gd);
                SF_TIMED(w0, bar_wait(&S.dq_full[slot], (it >> 1) & 1));
                if (lane == 0) SF_PROG(A, 5 + q, (uint32_t)it, 0x20000u | (uint32_t)Gd);
                if (q == 0 && lane == 0) SF_STAMP(A, it, 6);
                const int ht = *reinterpret_cast<volatile int*>(&S.dq_ht[slot]);
                const bool contrib = *reinterpret_cast<volatile uint32_t*>(&S.dq_info[slot]) != 0u;
                __syncwarp();
                if (lane == 0) bar_arrive(&S.dq_empty[slot]);
                if (ht < 0) break;
                const int tile = A.tile0 + (ht >> 1), half = ht & 1;
                const int w8 = half * 4 + q;
                const int bx = (tile % A.tiles_x) * SF_TILE + (w8 & 1) * 8, by = (tile / A.tiles_x) * SF_TILE + (w8 >> 1) * 4;
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
                        for (int g = 0, b = 0, c = 0; g < nchunk; ++g, c = (c + 1 == dchunks) ? (++b, 0) : c + 1) {
#ifndef SF_NOSTORE  // experiment only: no feature stores
                            tma_store_4d(&fmap, wbox, c * kDecN, bx, by, b);
                            tma_store_4d(&fmap, wbox + kBoxBytes, c * kDecN + kBoxCols, bx, by, b);
#endif
                        }
                        bulk_commit();
                    }
                    continue;
                }
                for (int g = 0, b = 0, c = 0; g < nchunk; ++g, ++Gd, c = (c + 1 == dchunks) ? (++b, 0) : c + 1) {
                    const int t = Gd & 1;  // (b, c) = (level, chunk in level) of g, stepped without a division
                    if (lane == 0) SF_PROG(A, 5 + q, (uint32_t)it, 0x30000u | (uint32_t)Gd);
                    SF_TIMED(w1, bar_wait(&S.acc_full[t], (Gd >> 1) & 1));
                    if (q == 0 && lane == 0) SF_CSTAMP(A, Gd, 0);
                    tc_after();
                    uint32_t v[64];
                    tmem_ld32(tm + lane_off + (uint32_t)(kAccCol0 + t * kDecN), *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                    tmem_ld32(tm + lane_off + (uint32_t)(kAccCol0 + t * kDecN + 32), *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    tc_before();
                    __syncwarp();
                    if (lane == 0) bar_arrive(&S.acc_empty[t]);
                    if (q == 0 && lane == 0) SF_CSTAMP(A, Gd, 1);
                    const float sc = b == 0 ? scl[0] : (b == 1 ? scl[1] : scl[2]);
                    if (sc != 1.f) {  // warp-uniform; only for atoms outside the fp16-friendly range
#pragma unroll
                        for (int i = 0; i < 64; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * sc);
                    }
                    if (lane == 0) SF_TIMED(w2, bulk_wait_read<0>());  // the previous chunk's stores have left the boxes
                    if (q == 0 && lane == 0) SF_CSTAMP(A, Gd, 2);
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
#ifndef SF_NOSTORE
                        tma_store_4d(&fmap, wbox, c * kDecN, bx, by, b);
                        tma_store_4d(&fmap, wbox + kBoxBytes, c * kDecN + kBoxCols, bx, by, b);
#endif
                        bulk_commit();
                        if (q == 0) SF_CSTAMP(A, Gd, 3);
                        if (q == 0 && g == nchunk - 1) SF_STAMP(A, it, 7);
                        if (q == 0 && g == 0) SF_STAMP(A, it, 8);
                    }
                }
            }
            if (lane == 0) bulk_wait_read<0>();
        }
    } else if (warp == kMmaWarp && lane == 0) {
        // ---------------- E V issuer: the blend products, batch by batch ----------------
        const uint32_t idesc_ev = (1u << 4) | ((uint32_t)(n_ch >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t eh0 = smem_addr(&S.ehi[0][0]), el0 = smem_addr(&S.elo[0][0]);
        const uint32_t vh0 = smem_addr(&S.vhi[0][0]), vl0 = smem_addr(&S.vlo[0][0]);
        int be = 0;
        for (int te = 0;; ++te) {
            bool first = true;
            int ht = 0;
            for (;;) {
                const int s = be % kStages;
                SF_TIMED(w0, bar_wait(&S.ev_full[s], (be / kStages) & 1));
                const int nb = *reinterpret_cast<volatile int*>(&S.nb[s]);
                if (first) ht = *reinterpret_cast<volatile int*>(&S.sched[te & 7]);
                ++be;
                // The slot's previous tile (te - 2) must be fully decoded before
                // this tile writes it -- also when the tile has no batch at all:
                // w_full(te) lets the blend warps convert into the slot and
                // publish a_ready(te), which must not complete a second phase of
                // a_ready[slot] before the decode issuer consumed a_ready(te - 2).
                if (first && te >= 2) SF_TIMED(w1, bar_wait(&S.slot_free[te & 1], ((te >> 1) - 1) & 1));
                if (nb == 0) {
                    // end of the tile's stream: W complete once the issued products are
                    if (!first) mma_commit(&S.w_full[te & 1]);
                    else bar_arrive(&S.w_full[te & 1]);
                    SF_STAMP(A, te, 3);
                    bar_arrive(&S.ev_empty[s]);
                    break;
                }
                if (prof) {
                    w2 += (uint64_t)__popc(*reinterpret_cast<volatile uint32_t*>(&S.ev_union[s]));
                    S.ev_union[s] = 0u;
                }
                if (*reinterpret_cast<volatile uint32_t*>(&S.ev_tag[s]) != (uint32_t)(be - 1) + 1u) {
                    // no blend warp had a candidate: E = 0, nothing to add
                    bar_arrive(&S.ev_empty[s]);
                    continue;
                }
                tc_after();
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
            }
            SF_PROG(A, 9, (uint32_t)te, (uint32_t)be);
            if (ht < 0) break;  // the terminal empty tile
        }
    } else if (DEC && warp == kDecWarp && lane == 0) {
        // ---------------- decode issuer: 3-term fp16 chunks of each converted tile ----------------
        const uint32_t idesc_dec = (1u << 4) | ((uint32_t)(kDecN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t bdesc0 = sw128_desc(smem_addr(S.bring[0]));
        int Gd = 0;
        for (int td = 0;; ++td) {
            SF_TIMED(w0, bar_wait(&S.a_ready[td & 1], (td >> 1) & 1));
            if (td >= 2) SF_TIMED(w0, bar_wait(&S.dq_empty[td & 1], ((td >> 1) - 1) & 1));
            tc_after();
            SF_STAMP(A, td, 4);
            // the drains learn the tile (and its kind) in order, through their own ring
            const int ht = *reinterpret_cast<volatile int*>(&S.a_ht[td & 1]);
            const uint32_t c = ht >= 0 ? *reinterpret_cast<volatile uint32_t*>(&S.contrib[td & 1]) : 0u;
            S.dq_info[td & 1] = c;
            S.dq_ht[td & 1] = ht;
            bar_arrive(&S.dq_full[td & 1]);
            if (ht < 0) break;
            if (c == 0u) {
                bar_arrive(&S.slot_free[td & 1]);  // nothing to multiply: the slot is free now
                continue;
            }
            for (int cd = 0, b = 0, cl = 0; cd < nchunk; ++cd, ++Gd, cl = (cl + 1 == dchunks) ? (++b, 0) : cl + 1) {
                const int s = Gd % kBStages, t = Gd & 1;
                SF_TIMED(w1, bar_wait(&S.b_full[s], (Gd / kBStages) & 1));
                if (Gd >= 2) SF_TIMED(w2, bar_wait(&S.acc_empty[t], ((Gd >> 1) - 1) & 1));
                tc_after();
                SF_CSTAMP(A, Gd, 4);
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
                mma_commit(&S.b_empty[s]);  // the chunk's codebook stage is free once its MMAs are
                SF_CSTAMP(A, Gd, 5);
            }
            mma_commit(&S.slot_free[td & 1]);
            SF_STAMP(A, td, 5);
            SF_PROG(A, 10, (uint32_t)td, (uint32_t)Gd);
        }
        // wake the loader: once every product has completed (no stage is read any
        // more), publish the chunk count and complete one more phase of each stage
        mma_commit(&S.dec_done);
        bar_wait(&S.dec_done, 0);
        // the loader has consumed every real phase once it waits for chunk Gd's
        // (only then may one more completion land without skipping a phase it
        // has not seen)
        while (*reinterpret_cast<volatile int*>(&S.loader_g) != Gd) __nanosleep(64);
        *reinterpret_cast<volatile int*>(&S.dec_total) = Gd;
        bar_arrive(&S.b_empty[Gd % kBStages]);
    } else if (DEC && warp == kLoadWarp && lane == 0) {
        // ---------------- codebook loader: chunk g + kBStages into the stage chunk g frees ----------------
        // (decoupled from the drains, which read the accumulators later; every
        // non-empty tile decodes chunks 0 .. nchunk - 1 in order, so global
        // chunk G needs image chunk G % nchunk)
        const unsigned char* img = reinterpret_cast<const unsigned char*>(A.dec_b);
        for (int g = 0; g < kBStages; ++g) {
            bar_expect_tx(&S.b_full[g], kChunkBytes);
            bulk_g2s(S.bring[g], img + (size_t)(g % nchunk) * kChunkBytes, kChunkBytes, &S.b_full[g]);
        }
        int G = 0;
        for (;;) {
            const int sg = G % kBStages;
            // blocks until the stage frees (this warp shares an SMSP with a blend
            // pair: no polling); after the last chunk the decode issuer completes
            // this phase itself, with dec_total set
            *reinterpret_cast<volatile int*>(&S.loader_g) = G;
            bar_wait(&S.b_empty[sg], (G / kBStages) & 1);
            const int total = *reinterpret_cast<volatile int*>(&S.dec_total);
            if (total >= 0 && G >= total) break;
            bar_expect_tx(&S.b_full[sg], kChunkBytes);
            bulk_g2s(S.bring[sg], img + (size_t)((G + kBStages) % nchunk) * kChunkBytes, kChunkBytes, &S.b_full[sg]);
            ++G;
        }
        // the loads of chunks G .. G + kBStages - 1 were never consumed: they land before exit
        for (int g = G; g < G + kBStages; ++g) bar_wait(&S.b_full[g % kBStages], (g / kBStages) & 1);
    }
    if (prof && lane == 0) {
        // 4 counters per warp: blend 0..31, drain 32..47, producer 48, E V issuer 52, decode issuer 56
        const int slot = 4 * warp;
        prof_add(A, slot + 0, clock64() - t_start);
        prof_add(A, slot + 1, w0);
        prof_add(A, slot + 2, w1);
        prof_add(A, slot + 3, w2);
    }
    __syncwarp();
    tc_before();
    __syncthreads();
    if (warp == 0) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
        if (lane == 0) SF_PROG(A, 11, 1u, 1u);
    }
}

}  // namespace tcs

size_t splat_tc_smem_bytes() { return sizeof(tcs::Smem) + 1024; }

bool splat_tc_supported(const BlendArgs& a) {
    if (!a.sched) return false;
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
    static const unsigned long long prog = [] {
        const char* e = getenv("SF_TC_PROGRESS");
        return e ? strtoull(e, nullptr, 10) : 0ull;
    }();
    void (*kern)(BlendArgs, const CUtensorMap);
    if (prog) {
        if (dec) kern = rel ? tcs::k_splat_tc<4, true, true> : tcs::k_splat_tc<0, true, true>;
        else kern = rel ? tcs::k_splat_tc<4, false, true> : tcs::k_splat_tc<0, false, true>;
    } else {
        if (dec) kern = rel ? tcs::k_splat_tc<4, true, false> : tcs::k_splat_tc<0, true, false>;
        else kern = rel ? tcs::k_splat_tc<4, false, false> : tcs::k_splat_tc<0, false, false>;
    }
    const size_t smem = splat_tc_smem_bytes();
    if (ensure_smem_attr((const void*)kern, smem)) return -6;
    const int n_half = 2 * a.n_band_tiles;
    if (n_half <= 0) return 0;
    static const int grid_env = [] {  // development aid: fewer CTAs than SMs (SF_TC_GRID)
        const char* e = getenv("SF_TC_GRID");
        return e ? atoi(e) : 0;
    }();
    const int grid = std::min(n_half, grid_env > 0 ? grid_env : device_sm_count());
    BlendArgs a2 = a;
    a2.timeline = prog ? reinterpret_cast<uint64_t*>(prog) : nullptr;
    kern<<<grid, tcs::kThreads, smem, st>>>(a2, fmap);
    return 0;
}

}  // namespace sf
