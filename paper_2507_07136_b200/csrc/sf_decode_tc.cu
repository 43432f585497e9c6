// sf_decode_tc.cu -- K7: codebook decode on tcgen05 tensor cores, 3xTF32.
//
// Reference: decode, sparse_splat.py:183-199 -- per level F = W @ atoms with
// W (P, L) the coefficient map block and atoms (L, D), fp64 BLAS.
//
// Precision.  TF32 keeps 10 mantissa bits; one TF32 product would miss the
// 1e-4 feature tolerance (hard part 3).  Split both operands
// x = hi + lo with hi = rna_tf32(x) and lo = x - hi (exact in fp32), then
//     F ~= A_lo B_hi + A_hi B_lo + A_hi B_hi        (error ~2^-22 |A||B|)
// accumulated in fp32 in TMEM.  B (the codebook) is split once per call by
// a prep kernel; A is split in shared memory by converter warps right after
// its TMA lands.
//
// Mapping.  Persistent grid of 148 CTAs (one per SM).  CTA c owns output
// columns [128 (c % 4), +128) of D = 512 and M tiles m = c / 4 + k * 37, so
// the four CTAs of a group walk the same W tiles together (L2 hits).  The
// codebook slice (hi + lo, K-major, 128B swizzle, 64 KB) stays resident in
// SMEM; W tiles (128 pixels x L) stream in through a 2-stage TMA ring.  One
// elected thread issues 3 x (L / 8) MMAs of 128 x 128 x 8 per tile into one
// of four TMEM accumulators (4 x 128 columns), so epilogues of earlier tiles
// overlap the MMAs of later ones.  Eight epilogue warps drain TMEM with
// tcgen05.ld.32x32b into 128B-swizzled SMEM boxes (128 rows x 32 columns)
// that TMA bulk-stores to HBM (out-of-range rows are clipped by the TMA
// unit).  The kernel is HBM-store bound: 4 B per output element (D = 512,
// 3 levels: 9.56 GB per 1440x1080 frame).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "sf_common.cuh"

namespace sf {

namespace tc {

constexpr int BM = 128;           // pixels per tile (TMEM lanes)
constexpr int BN = 128;           // output columns per CTA (MMA N)
constexpr int KBOX = 32;          // fp32 per 128-byte swizzle row
constexpr int kThreads = 576;     // 18 warps
constexpr int kEpiWarp0 = 2;      // warps 2..9 epilogue: 2 column halves x 4 lane quarters
constexpr int kEpiWarps = 8;
constexpr int kCvtWarp0 = 10;     // warps 10..17 A splitters
constexpr int kCvtThreads = 256;
constexpr int kStages = 2;        // W tile ring; A_lo is double-buffered with it
constexpr int kAcc = 4;           // TMEM accumulators (4 x 128 columns)
constexpr int kBoxes = BN / 32;   // output boxes per tile
constexpr int kStageBuf = 2;      // output staging boxes in flight (TMA store ring)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"((uint64_t)map), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"((uint64_t)map),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major, 128B-swizzled operand: rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
    d |= (uint64_t)(1) << 16;                      // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;              // stride byte offset: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                        // layout: SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

struct Smem {
    // operand tiles (1024-byte aligned, SW128 atoms)
    float b_hi[64 / KBOX][BN * KBOX];        // 2 x 16 KB
    float b_lo[64 / KBOX][BN * KBOX];        // 2 x 16 KB
    float a[kStages][64 / KBOX][BM * KBOX];     // 2 x 2 x 16 KB (hi after split)
    float a_lo[kStages][64 / KBOX][BM * KBOX];  // 2 x 2 x 16 KB
    float out[kStageBuf][BM * 32];           // 2 x 16 KB output staging (SW128)
    uint64_t full[kStages];      // TMA landed
    uint64_t ready[kStages];     // A split done
    uint64_t empty[kStages];     // MMAs finished reading the stage
    uint64_t acc_full[kAcc];     // accumulator complete
    uint64_t acc_empty[kAcc];    // accumulator drained
    uint64_t b_full;             // codebook slice landed
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(kThreads, 1)
k_decode_tc(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
            const __grid_constant__ CUtensorMap map_out, int64_t P, int L, int D, int nsplit) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkb = L / KBOX;              // 1 or 2 K boxes
    const int split = blockIdx.x % nsplit;
    const int groups = gridDim.x / nsplit;
    const int group = blockIdx.x / nsplit;
    const int n0 = split * BN;
    const int n_mtiles = (int)((P + BM - 1) / BM);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.ready[s], kCvtThreads);
            mbar_init(&S.empty[s], 1);
        }
        for (int s = 0; s < kAcc; ++s) {
            mbar_init(&S.acc_full[s], 1);
            mbar_init(&S.acc_empty[s], kEpiWarps * 32);
        }
        mbar_init(&S.b_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&S.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    // idesc: D f32, A/B tf32, K-major both, N = 128, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    const uint32_t a_tile_bytes = (uint32_t)(BM * KBOX * 4) * nkb;
    const int my_tiles = (group < n_mtiles) ? (n_mtiles - group + groups - 1) / groups : 0;

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        mbar_expect_tx(&S.b_full, (uint32_t)(2 * nkb * BN * KBOX * 4));
        for (int kb = 0; kb < nkb; ++kb) {
            tma_load_2d(S.b_hi[kb], &map_b, &S.b_full, kb * KBOX, n0);
            tma_load_2d(S.b_lo[kb], &map_b, &S.b_full, kb * KBOX, D + n0);
        }
        constexpr int kPrefetch = 4;  // W tiles warmed into L2 ahead of their TMA load
        if (split == 0)
            for (int i = 0; i < kPrefetch && i < my_tiles; ++i)
                for (int kb = 0; kb < nkb; ++kb) tma_prefetch_2d(&map_a, kb * KBOX, (group + i * groups) * BM);
        for (int i = 0; i < my_tiles; ++i) {
            const int s = i % kStages;
            if (split == 0 && i + kPrefetch < my_tiles)
                for (int kb = 0; kb < nkb; ++kb)
                    tma_prefetch_2d(&map_a, kb * KBOX, (group + (i + kPrefetch) * groups) * BM);
            if (i >= kStages) mbar_wait(&S.empty[s], ((i / kStages) - 1) & 1);
            const int m = group + i * groups;
            mbar_expect_tx(&S.full[s], a_tile_bytes);
            for (int kb = 0; kb < nkb; ++kb) tma_load_2d(S.a[s][kb], &map_a, &S.full[s], kb * KBOX, m * BM);
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        mbar_wait(&S.b_full, 0);
        tc_fence_after();
        for (int i = 0; i < my_tiles; ++i) {
            const int s = i % kStages, as = i % kAcc;
            mbar_wait(&S.ready[s], (i / kStages) & 1);
            if (i >= kAcc) mbar_wait(&S.acc_empty[as], ((i / kAcc) - 1) & 1);
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)(as * BN);
            uint32_t acc = 0;
            for (int kb = 0; kb < nkb; ++kb) {
                const uint32_t ahi = smem_u32(S.a[s][kb]);
                const uint32_t alo = smem_u32(S.a_lo[s][kb]);
                const uint32_t bhi = smem_u32(S.b_hi[kb]);
                const uint32_t blo = smem_u32(S.b_lo[kb]);
#pragma unroll
                for (int k = 0; k < KBOX / 8; ++k) {
                    const uint32_t off = k * 32;  // 8 tf32 = 32 B along the swizzled row
                    mma_tf32(d, sw128_desc(alo + off), sw128_desc(bhi + off), idesc, acc);
                    acc = 1;
                    mma_tf32(d, sw128_desc(ahi + off), sw128_desc(blo + off), idesc, 1);
                    mma_tf32(d, sw128_desc(ahi + off), sw128_desc(bhi + off), idesc, 1);
                }
            }
            mma_commit(&S.empty[s]);
            mma_commit(&S.acc_full[as]);
        }
    } else if (warp >= kCvtWarp0) {
        // ---------------- A splitters: hi = rna(x) in place, lo = x - hi ----------------
        // A_lo[s] is free whenever stage s has refilled: the producer only
        // reloads stage s after the MMAs of the tile two back completed
        const int t = threadIdx.x - kCvtWarp0 * 32;  // 0..255
        for (int i = 0; i < my_tiles; ++i) {
            const int s = i % kStages;
            mbar_wait(&S.full[s], (i / kStages) & 1);
            for (int kb = 0; kb < nkb; ++kb) {
                const uint32_t av = smem_u32(S.a[s][kb]);
                const uint32_t lv = smem_u32(S.a_lo[s][kb]);
#pragma unroll 4
                for (int j = t; j < BM * KBOX / 4; j += kCvtThreads) {
                    float4 x;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                                 : "r"(av + 16 * j));
                    float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(av + 16 * j), "f"(h.x), "f"(h.y),
                                 "f"(h.z), "f"(h.w)
                                 : "memory");
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(lv + 16 * j), "f"(x.x - h.x),
                                 "f"(x.y - h.y), "f"(x.z - h.z), "f"(x.w - h.w)
                                 : "memory");
                }
            }
            fence_proxy_async();
            mbar_arrive(&S.ready[s]);
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
        // ---------------- epilogue: TMEM -> swizzled SMEM box -> TMA store ----------------
        // warp (quarter, half) drains rows 32*quarter.. and columns 16*half.. of each 32-column box
        const int quarter = warp & 3;                     // TMEM lane quarter this warp may access
        const int half = (warp - kEpiWarp0) >> 2;
        const int r = quarter * 32 + lane;                // row within the tile
        const bool issuer = (warp == kEpiWarp0 && lane == 0);
        const int bar_id = 1;
        const int nthr = kEpiWarps * 32;
        int nstore = 0;
        for (int i = 0; i < my_tiles; ++i) {
            const int as = i % kAcc;
            const int m = group + i * groups;
            mbar_wait(&S.acc_full[as], (i / kAcc) & 1);
            tc_fence_after();
            for (int box = 0; box < kBoxes; ++box) {
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(as * BN + box * 32 + half * 16);
                uint32_t v[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                    "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (box == kBoxes - 1) {  // accumulator fully read: hand it back to the MMA warp
                    tc_fence_before();
                    mbar_arrive(&S.acc_empty[as]);
                }
                // staging slot must be drained by the TMA store issued two boxes ago
                const int slot = nstore % kStageBuf;
                if (issuer) bulk_wait_read<kStageBuf - 1>();
                named_bar(bar_id, nthr);
                const uint32_t rowp = smem_u32(S.out[slot]) + r * 128;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int pc = (half * 4 + c) ^ (r & 7);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowp + pc * 16), "r"(v[4 * c]),
                                 "r"(v[4 * c + 1]), "r"(v[4 * c + 2]), "r"(v[4 * c + 3])
                                 : "memory");
                }
                fence_proxy_async();
                named_bar(bar_id, nthr);
                if (issuer) {
                    tma_store_2d(&map_out, S.out[slot], n0 + box * 32, m * BM);
                    bulk_commit();
                }
                ++nstore;
            }
        }
        if (issuer) bulk_wait<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// B (L x D, row-major) -> [hi; lo] as (2D x L) K-major rows (row n = column n of B).
__global__ void k_split_codebook(const float* __restrict__ cb, int L, int D, float* __restrict__ out) {
    int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= L * D) return;
    int n = idx / L, k = idx % L;
    float x = cb[(size_t)k * D + n];
    float h = tf32_rna(x);
    out[(size_t)n * L + k] = h;
    out[(size_t)(D + n) * L + k] = x - h;
}

}  // namespace tc

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

static int make_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                       uint32_t box_inner, uint32_t box_outer) {
    auto enc = get_encode();
    if (!enc) return -1;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

size_t decode_ws_bytes(int L, int D) { return (size_t)2 * L * D * sizeof(float); }

static bool decode_tc_supported(int64_t P, int L, int D, const float* w, int64_t w_stride, const float* out) {
    return (L == 32 || L == 64) && D % tc::BN == 0 && ((uintptr_t)w % 16) == 0 && (w_stride * 4) % 16 == 0 &&
           ((uintptr_t)out % 16) == 0 && P > 0 && P < (int64_t)1 << 31;
}

int launch_decode(int64_t P, int L, int D, const float* w, int64_t w_stride, const float* cb, float* out,
                  void* ws, cudaStream_t st) {
    if (P == 0) return 0;
    if (!decode_tc_supported(P, L, D, w, w_stride, out) || ws == nullptr)
        return launch_decode_simt(P, L, D, w, w_stride, cb, out, st);
    float* bsplit = (float*)ws;
    tc::k_split_codebook<<<ceil_div((int64_t)L * D, 256), 256, 0, st>>>(cb, L, D, bsplit);
    CUtensorMap ma, mb, mo;
    if (make_map_2d(&ma, w, (uint64_t)L, (uint64_t)P, (uint64_t)w_stride * 4, tc::KBOX, tc::BM)) return -3;
    if (make_map_2d(&mb, bsplit, (uint64_t)L, (uint64_t)2 * D, (uint64_t)L * 4, tc::KBOX, tc::BN)) return -3;
    if (make_map_2d(&mo, out, (uint64_t)D, (uint64_t)P, (uint64_t)D * 4, 32, tc::BM)) return -3;
    static int num_sms = 0;
    if (!num_sms) {
        int dev;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int nsplit = D / tc::BN;
    int groups = num_sms / nsplit;
    if (groups < 1) groups = 1;
    const int n_mtiles = (int)((P + tc::BM - 1) / tc::BM);
    if (groups > n_mtiles) groups = n_mtiles;
    const size_t smem = sizeof(tc::Smem) + 1024;
    ensure_smem_attr((const void*)tc::k_decode_tc, smem);
    tc::k_decode_tc<<<groups * nsplit, tc::kThreads, smem, st>>>(ma, mb, mo, P, L, D, nsplit);
    return 0;
}

}  // namespace sf
