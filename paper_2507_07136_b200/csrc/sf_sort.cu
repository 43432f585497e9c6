// sf_sort.cu -- K2: stable LSD radix sort of (u64 key, u32 value) pairs,
// hand-written for sm_100a (one-sweep passes with decoupled look-back).
//
// Reference: the canonical order lexsort((ids, depths)) (projection.py:396).
// The frame's rows are id-ordered and positive fp64 depths order like their
// bit patterns, so a STABLE sort of the depth bits gives the (depth, id)
// order exactly (culled rows carry key ~0 and land last).
//
// Algorithm (per 8-bit digit, least significant first):
//   k_sort_hist    one read of all keys: the 8 digit histograms at once
//   k_sort_plan    per pass: exclusive digit bases, and whether the pass is
//                  trivial (every key in one digit -- e.g. the exponent byte
//                  of depths within a factor 2^16) and skipped
//   k_sort_pass    CTA = 3072 consecutive keys (12 per thread, striped per
//                  warp so (item, lane) order is input order).  Warp-level
//                  stable ranks with __match_any_sync, per-warp digit counts,
//                  the tile's digit counts published to a status word per
//                  (tile, digit) and summed over earlier tiles by decoupled
//                  look-back (tile ids are taken in launch order, so every
//                  earlier tile is already resident), a local reorder in
//                  shared memory, then coalesced runs to global memory.
//   k_sort_copy    if the number of executed passes is even, the result is
//                  in the input buffers: copy it to the output buffers.
// Stability: within a tile equal digits keep input order (ranks are taken
// in input order); tiles are ordered by the look-back.  So each pass is a
// stable counting sort and the LSD sequence sorts by the full key.
#include <stdint.h>

#include <algorithm>

#include "sf_common.cuh"

namespace sf {
namespace rsort {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 12;
constexpr int kTile = kThreads * kItems;  // 3072 keys per CTA (46 KB of static shared memory)
constexpr int kPasses = 8;
constexpr int kBins = 256;
// status word per (tile, digit): [63:60] pass tag (1 + pass), [59] inclusive
// flag, [58:0] count.  The buffer is cleared once per sort; a word written by
// an earlier pass carries an older tag and reads as "not yet published".
constexpr uint64_t kIncl = 1ull << 59;
constexpr uint64_t kCountMask = kIncl - 1;

struct Plan {
    uint32_t hist[kPasses][kBins];   // global digit histograms
    uint32_t base[kPasses][kBins];   // exclusive digit bases
    uint32_t active;                 // bit p: pass p moves keys
    uint32_t tile_ctr[kPasses];      // dynamic tile ids per pass
};

__device__ __forceinline__ uint32_t digit(uint64_t k, int p) { return (uint32_t)(k >> (8 * p)) & 0xFFu; }

__global__ void __launch_bounds__(kThreads) k_sort_hist(const uint64_t* __restrict__ keys, int64_t n, Plan* plan) {
    __shared__ uint32_t h[kPasses][kBins];
    for (int i = threadIdx.x; i < kPasses * kBins; i += kThreads) (&h[0][0])[i] = 0u;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
        const uint64_t k = __ldg(keys + i);
#pragma unroll
        for (int p = 0; p < kPasses; ++p) atomicAdd(&h[p][digit(k, p)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kPasses * kBins; i += kThreads) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(&plan->hist[0][0] + i, v);
    }
}

// one CTA of kBins threads: pass p's exclusive bases; the active-pass mask
__global__ void __launch_bounds__(kBins) k_sort_plan(int64_t n, Plan* plan) {
    __shared__ uint32_t s[kBins];
    __shared__ uint32_t trivial[kPasses];
    const int d = threadIdx.x;
    if (d < kPasses) trivial[d] = 0u;
    __syncthreads();
    for (int p = 0; p < kPasses; ++p) {
        const uint32_t c = plan->hist[p][d];
        if ((int64_t)c == n) trivial[p] = 1u;
        // inclusive Hillis-Steele scan over the 256 bins
        s[d] = c;
        __syncthreads();
        for (int o = 1; o < kBins; o <<= 1) {
            const uint32_t v = d >= o ? s[d - o] : 0u;
            __syncthreads();
            s[d] += v;
            __syncthreads();
        }
        plan->base[p][d] = s[d] - c;
        __syncthreads();
    }
    if (d == 0) {
        uint32_t m = 0;
        for (int p = 0; p < kPasses; ++p)
            if (!trivial[p]) m |= 1u << p;
        plan->active = m;
        for (int p = 0; p < kPasses; ++p) plan->tile_ctr[p] = 0u;
    }
}

__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One pass (digit p).  Keys / values ping-pong between (k0, v0) and (k1, v1):
// the source is k0 iff an even number of passes before p were executed.
__global__ void __launch_bounds__(kThreads) k_sort_pass(int p, int64_t n, uint64_t* k0, uint32_t* v0, uint64_t* k1,
                                                        uint32_t* v1, Plan* plan, uint64_t* status) {
    __shared__ uint64_t sk[kTile];
    __shared__ uint32_t sv[kTile];
    __shared__ uint32_t whist[kWarps][kBins];  // per-warp digit counts -> per-warp exclusive offsets
    __shared__ uint32_t loc[kBins];            // exclusive digit offsets inside the tile
    __shared__ uint32_t gofs[kBins];           // global start of the tile's run of each digit
    __shared__ uint32_t s_tile;
    const uint32_t active = plan->active;
    if (!((active >> p) & 1u)) return;
    const bool from0 = (__popc(active & ((1u << p) - 1u)) & 1) == 0;
    const uint64_t* ksrc = from0 ? k0 : k1;
    const uint32_t* vsrc = from0 ? v0 : v1;
    uint64_t* kdst = from0 ? k1 : k0;
    uint32_t* vdst = from0 ? v1 : v0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) s_tile = atomicAdd(&plan->tile_ctr[p], 1u);
    for (int i = threadIdx.x; i < kWarps * kBins; i += kThreads) (&whist[0][0])[i] = 0u;
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t base = (int64_t)tile * kTile + warp * (kTile / kWarps);

    // load (striped inside the warp: item j of lane l is position 32 j + l)
    uint64_t key[kItems];
    uint32_t val[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const int64_t i = base + 32 * j + lane;
        key[j] = i < n ? ksrc[i] : ~0ull;
        val[j] = i < n ? vsrc[i] : 0u;
    }
    // stable warp ranks: items in (j, lane) order = input order
    uint32_t rank[kItems];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const bool ok = base + 32 * j + lane < n;
        const uint32_t d = ok ? digit(key[j], p) : kBins + lane;  // out-of-range items match nobody
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t before = 0;
        if (ok) before = whist[warp][d];
        __syncwarp();
        rank[j] = before + __popc(peers & lt);
        if (ok && (peers & lt) == 0u) whist[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit (thread d): warp offsets, tile count, look-back
    {
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = whist[w][d];
            whist[w][d] = run;
            run += c;
        }
        const uint32_t cnt = run;
        const uint64_t tag = (uint64_t)(p + 1) << 60;
        uint64_t* my = status + (size_t)tile * kBins + d;
        if (tile == 0) {
            st_status(my, tag | kIncl | cnt);
            gofs[d] = plan->base[p][d];
        } else {
            st_status(my, tag | cnt);
            uint64_t excl = 0;
            for (int64_t t = (int64_t)tile - 1; t >= 0; --t) {
                const uint64_t* ps = status + (size_t)t * kBins + d;
                uint64_t v;
                do {
                    v = ld_status(ps);
                } while ((v & (0xFull << 60)) != tag);
                excl += v & kCountMask;
                if (v & kIncl) break;
            }
            st_status(my, tag | kIncl | (excl + cnt));
            gofs[d] = plan->base[p][d] + (uint32_t)excl;
        }
        // exclusive scan of the tile's digit counts (local reorder offsets)
        loc[d] = cnt;
    }
    __syncthreads();
    {
        // inclusive Hillis-Steele scan of loc (256 entries, one per thread)
        const int d = threadIdx.x;
        const uint32_t c = loc[d];
        uint32_t acc = c;
        for (int o = 1; o < kBins; o <<= 1) {
            const uint32_t v = d >= o ? loc[d - o] : 0u;
            __syncthreads();
            acc += v;
            loc[d] = acc;
            __syncthreads();
        }
        loc[d] = acc - c;
    }
    __syncthreads();
    // local reorder: digit-sorted, stable
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        if (base + 32 * j + lane < n) {
            const uint32_t d = digit(key[j], p);
            const uint32_t pos = loc[d] + whist[warp][d] + rank[j];
            sk[pos] = key[j];
            sv[pos] = val[j];
        }
    }
    __syncthreads();
    // coalesced write-out: slot i holds the (i - loc[d])-th key of digit d in this tile
    const int64_t t0 = (int64_t)tile * kTile;
    const int cnt_tile = (int)min((int64_t)kTile, n - t0);
    for (int i = threadIdx.x; i < cnt_tile; i += kThreads) {
        const uint64_t k = sk[i];
        const uint32_t d = digit(k, p);
        const uint32_t o = gofs[d] + (uint32_t)i - loc[d];
        kdst[o] = k;
        vdst[o] = sv[i];
    }
}

__global__ void __launch_bounds__(kThreads) k_sort_copy(int64_t n, const uint64_t* __restrict__ k0,
                                                        const uint32_t* __restrict__ v0, uint64_t* __restrict__ k1,
                                                        uint32_t* __restrict__ v1, const Plan* plan) {
    if (__popc(plan->active) & 1) return;  // odd: the last pass wrote (k1, v1)
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
        k1[i] = k0[i];
        v1[i] = v0[i];
    }
}

}  // namespace rsort

size_t depth_sort_tmp_bytes(int64_t n) {
    const int64_t tiles = (n + rsort::kTile - 1) / rsort::kTile;
    return ((sizeof(rsort::Plan) + 255) & ~(size_t)255) + (size_t)(tiles > 0 ? tiles : 1) * rsort::kBins * 8;
}

// Stable sort of (keys, vals) by the full 64-bit key into (keys_out, vals_out).
// keys_in / vals_in are scratch (overwritten by the ping-pong passes).
int depth_sort(uint64_t* keys_in, uint64_t* keys_out, uint32_t* vals_in, uint32_t* vals_out, int64_t n, void* tmp,
               size_t tmp_bytes, cudaStream_t st) {
    if (n == 0) return 0;
    if (tmp_bytes < depth_sort_tmp_bytes(n) || n >= ((int64_t)1 << 32)) return -1;
    using namespace rsort;
    Plan* plan = reinterpret_cast<Plan*>(tmp);
    uint64_t* status = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(tmp) + ((sizeof(Plan) + 255) & ~(size_t)255));
    const int64_t tiles = (n + kTile - 1) / kTile;
    cudaMemsetAsync(plan, 0, sizeof(Plan), st);
    cudaMemsetAsync(status, 0, (size_t)tiles * kBins * 8, st);
    const int hb = (int)std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 4);
    k_sort_hist<<<hb, kThreads, 0, st>>>(keys_in, n, plan);
    k_sort_plan<<<1, kBins, 0, st>>>(n, plan);
    for (int p = 0; p < kPasses; ++p)
        k_sort_pass<<<(unsigned)tiles, kThreads, 0, st>>>(p, n, keys_in, vals_in, keys_out, vals_out, plan, status);
    k_sort_copy<<<hb, kThreads, 0, st>>>(n, keys_in, vals_in, keys_out, vals_out, plan);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace sf
