// sf_binning.cu -- K2-K4: depth-rank sort, tile-key duplication, per-tile lists.
//
// Reference: bin_projected, projection.py:379-450.
//  (1) canonical order lexsort((ids, depths))            projection.py:396
//  (2) candidate tile rectangle from the +-3 sigma extent projection.py:406-418
//  (3) exact ellipse/rectangle test q_min <= 9            projection.py:429-441
//  (4) stable argsort by tile + searchsorted bounds       projection.py:443-449
//
// B200 design.  (1) is a device radix sort (sf_sort.cu) of the fp64 depth bits (positive
// doubles order like their bit patterns) over rows already stored in id
// order, so a stable sort gives the (depth, id) order exactly; the position
// in that order is the Gaussian's depth rank r.  (2)+(3) run per rank with
// the reference's fp64 arithmetic (this file is compiled with -fmad=false)
// and emit (tile, r) pairs; a per-tile counting pass plus an atomic bucket
// fill replaces the global pair sort, and a CTA-local sort of each tile's
// ranks restores the canonical order.  The resulting key order is exactly
// (tile id | depth rank), i.e. the reference's per-tile lists, bit for bit.
#include <cub/cub.cuh>

#include <algorithm>

#include "sf_blend_dev.cuh"
#include "sf_common.cuh"

namespace sf {

constexpr int kCountCTAs = 296;      // CTAs of the aggregated count pass (2 per SM)
constexpr int kAggMaxTiles = 16384;  // shared-memory tile histogram limit (64 KB)

size_t bin_cta_base_elems(int W, int H) {
    const int n_tiles = ((W + SF_TILE - 1) / SF_TILE) * ((H + SF_TILE - 1) / SF_TILE);
    return (size_t)kCountCTAs * (size_t)n_tiles;
}


// ---------------------------------------------------------------------------
// per-row scatter plan (sparse_splat.py:126-132 cat_idx / cat_vals)

__global__ void __launch_bounds__(256) k_pack_channels(int64_t G, const uint16_t* __restrict__ cidx,
                                                       const float* __restrict__ cval, int K, int L,
                                                       LevelSelDev levels, unsigned char* __restrict__ chan) {
    int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= G) return;
    const int C = levels.n * K;
    const int cs = chan_rec_bytes(C);
    if (C <= 16) {
        // build the record in registers, write it with 16-byte stores
        uint32_t rec[32];  // <= 128 bytes
#pragma unroll
        for (int i = 0; i < 32; ++i) rec[i] = 0;
        uint32_t* ch = rec;
        float* val = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(rec) + chan_val_offset(C));
        for (int b = 0; b < levels.n; ++b) {
            const int lv = levels.lv[b];
            const uint16_t* ip = cidx + ((int64_t)lv * G + row) * K;
            const float* vp = cval + ((int64_t)lv * G + row) * K;
            for (int k = 0; k < K; ++k) {
                ch[b * K + k] = (uint32_t)(__ldg(ip + k) + b * L) * kChanWord;
                val[b * K + k] = __ldg(vp + k);
            }
        }
        uint4* dst = reinterpret_cast<uint4*>(chan + (size_t)row * cs);
        for (int q = 0; q < cs / 16; ++q) dst[q] = make_uint4(rec[4 * q], rec[4 * q + 1], rec[4 * q + 2], rec[4 * q + 3]);
        return;
    }
    unsigned char* rp = chan + (size_t)row * cs;
    uint32_t* ch = reinterpret_cast<uint32_t*>(rp);
    float* val = reinterpret_cast<float*>(rp + chan_val_offset(C));
    for (int b = 0; b < levels.n; ++b) {
        const int lv = levels.lv[b];
        for (int k = 0; k < K; ++k) {
            ch[b * K + k] = (uint32_t)(cidx[((int64_t)lv * G + row) * K + k] + b * L) * kChanWord;
            val[b * K + k] = cval[((int64_t)lv * G + row) * K + k];
        }
    }
}

void launch_pack_channels(const SfScene& s, const LevelSelDev& levels, unsigned char* chan, cudaStream_t st) {
    if (s.num_gaussians)
        k_pack_channels<<<ceil_div(s.num_gaussians, 256), 256, 0, st>>>(s.num_gaussians, s.coeff_indices,
                                                                        s.coeff_values, s.K, s.L, levels, chan);
}

// ---------------------------------------------------------------------------
// candidate rectangle + exact tile test (reference fp64 order)

struct TileGrid {
    int W, H, tiles_x, tiles_y;
    int ty_lo, ty_hi;  // tile rows binned: [ty_lo, ty_hi] (band mode; else 0 .. tiles_y - 1)
};

__device__ __forceinline__ void cand_rect(const Proj64& p, const TileGrid& g, int& tx0, int& tx1,
                                          int& ty0, int& ty1) {
    double den = p.a * p.c - p.b * p.b;  // inv00*inv11 - inv01**2
    double cov_xx = p.c / den;
    double cov_yy = p.a / den;
    double rx = 3.0 * sqrt(np_maximum(cov_xx, 0.0));
    double ry = 3.0 * sqrt(np_maximum(cov_yy, 0.0));
    static_assert((SF_TILE & (SF_TILE - 1)) == 0, "tile size must be a power of two");
    const double inv_ts = 1.0 / (double)SF_TILE;
    int64_t v;
    v = np_to_i64(np_floor_divide_pow2(p.mx - rx, inv_ts));
    tx0 = (int)(v < 0 ? 0 : (v > g.tiles_x - 1 ? g.tiles_x - 1 : v));
    v = np_to_i64(np_floor_divide_pow2(p.mx + rx, inv_ts));
    tx1 = (int)(v < 0 ? 0 : (v > g.tiles_x - 1 ? g.tiles_x - 1 : v));
    v = np_to_i64(np_floor_divide_pow2(p.my - ry, inv_ts));
    ty0 = (int)(v < 0 ? 0 : (v > g.tiles_y - 1 ? g.tiles_y - 1 : v));
    v = np_to_i64(np_floor_divide_pow2(p.my + ry, inv_ts));
    ty1 = (int)(v < 0 ? 0 : (v > g.tiles_y - 1 ? g.tiles_y - 1 : v));
    // band mode: only the band's tile rows (each tile's test is independent)
    ty0 = max(ty0, g.ty_lo);
    ty1 = min(ty1, g.ty_hi);
}

__device__ __forceinline__ bool tile_hit(const MahalPre& p, int tx, int ty, const TileGrid& g) {
    double lx = (double)(tx * SF_TILE), ly = (double)(ty * SF_TILE);
    double hx = np_minimum(lx + (double)SF_TILE, (double)g.W) - 1;
    double hy = np_minimum(ly + (double)SF_TILE, (double)g.H) - 1;
    return min_mahal_sq_to_rect_pre(p, lx, ly, hx, hy) <= SF_CUTOFF;
}

// tile_hit with an fp32 pre-test.  The rectangle is taken relative to the
// mean with exact fp64 differences; the four edge minima of the reference's
// quadratic (the same clipped points) are evaluated in fp32, and the result
// decides when it clears 9 by more than 1e-5 of the largest term magnitude
// met (+1e-6) -- fp32 rounding of these few operations stays below 1e-6 of
// it.  Otherwise (and for the mean inside the rectangle) the decision is the
// exact fp64 one, so the lists stay byte-identical.
struct MahalPre32 {
    float a, c, boc, boa, twob;
};
__device__ __forceinline__ MahalPre32 mahal_pre32(const MahalPre& p) {
    return MahalPre32{(float)p.a, (float)p.c, (float)p.boc, (float)p.boa, (float)p.twob};
}
__device__ __forceinline__ bool tile_hit_fast(const MahalPre& p, const MahalPre32& f, int tx, int ty,
                                              const TileGrid& g) {
    const double lx = (double)(tx * SF_TILE), ly = (double)(ty * SF_TILE);
    const double hx = np_minimum(lx + (double)SF_TILE, (double)g.W) - 1;
    const double hy = np_minimum(ly + (double)SF_TILE, (double)g.H) - 1;
    if ((p.mx >= lx) && (p.mx <= hx) && (p.my >= ly) && (p.my <= hy)) return true;  // q = 0 <= 9
    const float x0 = (float)(lx - p.mx), x1 = (float)(hx - p.mx);
    const float y0 = (float)(ly - p.my), y1 = (float)(hy - p.my);
    float best = INFINITY, mag = 0.f;
    auto ev = [&](float dx, float dy) {
        const float t1 = f.a * dx * dx, t2 = f.twob * dx * dy, t3 = f.c * dy * dy;
        best = fminf(best, t1 + t2 + t3);
        mag = fmaxf(mag, t1 + fabsf(t2) + t3);
    };
    ev(x0, fminf(fmaxf(-f.boc * x0, y0), y1));
    ev(x1, fminf(fmaxf(-f.boc * x1, y0), y1));
    ev(fminf(fmaxf(-f.boa * y0, x0), x1), y0);
    ev(fminf(fmaxf(-f.boa * y1, x0), x1), y1);
    const float tol = 1e-5f * mag + 1e-6f;
    if (best + tol < (float)SF_CUTOFF) return true;
    if (best - tol > (float)SF_CUTOFF) return false;
    return min_mahal_sq_to_rect_pre(p, lx, ly, hx, hy) <= SF_CUTOFF;
}

// The item an entry names: frame mode (row_keys != null) -- item i is scene
// row i, visible iff its depth key is not the culled sentinel, and the entry
// is the row (put in (depth, row) order by k_tile_sort_depth); sf_bin mode --
// item i has canonical rank i (i < stats[VISIBLE]) and the entry is i.
__device__ __forceinline__ bool item_rank(int64_t i, const int64_t* stats, const uint64_t* row_keys, uint32_t& r) {
    r = (uint32_t)i;
    if (row_keys) return __ldg(row_keys + i) != ~0ull;
    return i < stats[SF_STAT_VISIBLE];
}

// Count pass: exact tests of every candidate tile.  The first kBinSlots hits
// of an item take their in-tile position from the counter (atomic with
// return) and remember it, so the emit pass stores without atomics; later
// hits count in a second counter bank and claim positions in the emit pass.
// The hit pattern over the candidate rectangle (row-major, <= 64 tiles) is
// kept too, so the emit pass repeats no fp64 arithmetic.
__global__ void __launch_bounds__(256, 4) k_count_pairs(int64_t N, const int64_t* __restrict__ stats,
                                                     const GeomRec* __restrict__ geom,
                                                     const uint64_t* __restrict__ row_keys,
                                                     TileGrid g, uint32_t* __restrict__ tile_counts,
                                                     BinAux* __restrict__ aux) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t r;
    if (i >= N || !item_rank(i, stats, row_keys, r)) return;
    Proj64 p = geom_proj(geom[i]);
    int tx0, tx1, ty0, ty1;
    cand_rect(p, g, tx0, tx1, ty0, ty1);
    const MahalPre mp = mahal_pre(p.mx, p.my, p.a, p.b, p.c);
    const MahalPre32 mf = mahal_pre32(mp);
    const int n_tiles = g.tiles_x * g.tiles_y;
    BinAux a;
    a.mask = 0;
    a.tx0 = (uint16_t)tx0;
    a.ty0 = (uint16_t)ty0;
    a.w = (uint16_t)(tx1 - tx0 + 1);
    a.h = (uint16_t)max(0, ty1 - ty0 + 1);
#pragma unroll
    for (int k = 0; k < kBinSlots; ++k) a.pos[k] = 0;
    int bit = 0, nh = 0;
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx, ++bit)
            if (tile_hit_fast(mp, mf, tx, ty, g)) {
                const int t = ty * g.tiles_x + tx;
                if (nh < kBinSlots) {
                    const uint32_t pos = atomicAdd(&tile_counts[t], 1u);
#pragma unroll
                    for (int k = 0; k < kBinSlots; ++k)
                        if (k == nh) a.pos[k] = pos;
                } else {
                    atomicAdd(&tile_counts[n_tiles + t], 1u);
                }
                ++nh;
                if (bit < 64) a.mask |= 1ull << bit;
            }
    const uint4* src = reinterpret_cast<const uint4*>(&a);
    uint4* dst = reinterpret_cast<uint4*>(aux + i);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(BinAux) / 16); ++k) dst[k] = src[k];
}

// Aggregated count pass (n_tiles <= kAggMaxTiles): CTA c owns items
// [c * per, (c + 1) * per) and counts its slot hits in a shared-memory tile
// histogram (the in-CTA position comes from the shared atomic); one global
// atomic per (CTA, tile) then reserves the CTA's range inside the tile and
// its base is kept in cta_base[c][tile].  4x fewer global atomics than one
// per pair, with the same emit-time arithmetic.
__global__ void __launch_bounds__(512, 2) k_count_pairs_agg(int64_t N, int64_t per, const int64_t* __restrict__ stats,
                                                         const GeomRec* __restrict__ geom,
                                                         const uint64_t* __restrict__ row_keys, TileGrid g,
                                                         uint32_t* __restrict__ tile_counts, BinAux* __restrict__ aux,
                                                         uint32_t* __restrict__ cta_base) {
    extern __shared__ uint32_t hist[];
    const int n_tiles = g.tiles_x * g.tiles_y;
    // the in-tile slots of the thread's current item (shared memory, not registers:
    // the fp64 tile test already needs most of the register budget)
    __shared__ uint32_t spos[512][kBinSlots];
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) hist[t] = 0;
    __syncthreads();
    const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(N, i0 + per);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        uint32_t r;
        if (!item_rank(i, stats, row_keys, r)) continue;
        Proj64 p = geom_proj(geom[i]);
        int tx0, tx1, ty0, ty1;
        cand_rect(p, g, tx0, tx1, ty0, ty1);
        const MahalPre mp = mahal_pre(p.mx, p.my, p.a, p.b, p.c);
        const MahalPre32 mf = mahal_pre32(mp);
        unsigned long long mask = 0;
        uint32_t* pos_k = spos[threadIdx.x];
        int bit = 0, nh = 0;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx, ++bit) {
                if (tile_hit_fast(mp, mf, tx, ty, g)) {
                    const int t = ty * g.tiles_x + tx;
                    if (nh < kBinSlots) pos_k[nh] = atomicAdd(&hist[t], 1u);
                    else atomicAdd(&tile_counts[n_tiles + t], 1u);
                    ++nh;
                    if (bit < 64) mask |= 1ull << bit;
                }
            }
        BinAux a;
        a.mask = mask;
        a.tx0 = (uint16_t)tx0;
        a.ty0 = (uint16_t)ty0;
        a.w = (uint16_t)(tx1 - tx0 + 1);
        a.h = (uint16_t)max(0, ty1 - ty0 + 1);
#pragma unroll
        for (int k = 0; k < kBinSlots; ++k) a.pos[k] = k < nh ? pos_k[k] : 0u;
        const uint4* src = reinterpret_cast<const uint4*>(&a);
        uint4* dst = reinterpret_cast<uint4*>(aux + i);
#pragma unroll
        for (int k = 0; k < (int)(sizeof(BinAux) / 16); ++k) dst[k] = src[k];
    }
    __syncthreads();
    uint32_t* base = cta_base + (size_t)blockIdx.x * n_tiles;
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
        const uint32_t c = hist[t];
        base[t] = c ? atomicAdd(&tile_counts[t], c) : 0u;
    }
}

// Exclusive scan over tiles (single CTA): offsets, emit cursors (past the
// slot-positioned entries), pair total.
// Also lists the tiles whose lists exceed kShortList entries (big[0] = count,
// big[1..] = tile ids) for the long-list sorts, and those with kTinyList <
// n <= kMidList in mid, kMidList < n <= kShortList in mid4 (same layout) for
// the mid-size sorts.
constexpr int kShortList = 4096;
constexpr int kTinyList = 2048;
constexpr int kMidList = 3072;  // mid-size lists split at 3072 (into mid / mid4)
// warp-aggregated append of t to list (list[0] = count, list[1..] = items);
// called by all 32 lanes of the warp
__device__ __forceinline__ void list_append(uint32_t* list, bool take, uint32_t t) {
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(&list[0], (uint32_t)__popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (take) list[1 + base + __popc(m & ((1u << lane) - 1u))] = t;
}

__global__ void __launch_bounds__(1024) k_tile_scan(int n_tiles, const uint32_t* __restrict__ counts,
                                                    uint32_t* __restrict__ offsets,
                                                    uint32_t* __restrict__ cursor,
                                                    int64_t pair_capacity, int64_t* stats,
                                                    uint32_t* __restrict__ big, uint32_t* __restrict__ mid,
                                                    uint32_t* __restrict__ mid4) {
    typedef cub::BlockScan<unsigned long long, 1024> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) {
        carry = 0;
        big[0] = 0u;
        mid[0] = 0u;
        mid4[0] = 0u;
    }
    __syncthreads();
    // 8 consecutive tiles per thread and pass: one block scan covers 8192 tiles
    constexpr int kPer = 8;
    for (int base = 0; base < n_tiles; base += 1024 * kPer) {
        const int t0 = base + threadIdx.x * kPer;
        uint32_t c0[kPer], c[kPer];  // per-tile counts fit 32 bits (the pair total may not)
        unsigned long long sum = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int t = t0 + k;
            c0[k] = (t < n_tiles) ? counts[t] : 0u;
            c[k] = (t < n_tiles) ? c0[k] + counts[n_tiles + t] : 0u;
            sum += c[k];
        }
        unsigned long long ex, tot;
        Scan(tmp).ExclusiveSum(sum, ex, tot);
        ex += carry;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int t = t0 + k;
            if (t < n_tiles) {
                offsets[t] = (uint32_t)ex;
                cursor[t] = (uint32_t)(ex + c0[k]);
            }
            // class lists: one atomic per warp and class (thousands of same-address
            // atomics serialised in the L2 otherwise); list order is irrelevant
            const unsigned long long n = t < n_tiles ? c[k] : 0ull;
            list_append(big, n > (unsigned long long)kShortList, (uint32_t)t);
            list_append(mid4, n > (unsigned long long)kMidList && n <= (unsigned long long)kShortList, (uint32_t)t);
            list_append(mid, n > (unsigned long long)kTinyList && n <= (unsigned long long)kMidList, (uint32_t)t);
            ex += c[k];
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        offsets[n_tiles] = (uint32_t)carry;
        stats[SF_STAT_PAIRS] = (int64_t)carry;
        stats[SF_STAT_OVERFLOW] = ((int64_t)carry > pair_capacity) ? 1 : 0;
    }
}

// Half-tile flags of a tile hit (frame mode): bit h is set when the 16 x 8
// pixel half h (rows 8h .. 8h + 7) may see the Gaussian.  With the conic
// written q = a (dx + k dy)^2 + d dy^2 (GeomF32), every point with q <= 9 has
// |dy| <= 3 / sqrt(d): the flag tests the half's pixel rows against that
// y-extent (widened by 1e-3 relative + 1e-3 px for the fp32 evaluation), so
// an entry without its half's flag has alpha = 0 at every pixel there.
struct HalfTest {
    float my, ry;
};
__device__ __forceinline__ HalfTest half_test_of(const GeomF32& g) {
    const float ry = 3.f * rsqrtf(g.d);
    return HalfTest{g.my_hi + g.my_lo, fmaf(ry, 1e-3f, ry) + 1e-3f};
}
__device__ __forceinline__ uint32_t half_tile_flags(const HalfTest& g, int x0, int y0) {
    (void)x0;
    const float lo = g.my - g.ry, hi = g.my + g.ry;
    const float y = (float)y0;
    return ((hi >= y && lo <= y + 7.f) ? 1u : 0u) | ((hi >= y + 8.f && lo <= y + 15.f) ? 2u : 0u);
}

__device__ __forceinline__ void emit_one(int j, int t, uint32_t r, const BinAux& a,
                                         const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ base,
                                         uint32_t* __restrict__ cursor, uint32_t* __restrict__ entries) {
    uint32_t pos;
    if (j < kBinSlots) {
        uint32_t slot = a.pos[0];
#pragma unroll
        for (int k = 1; k < kBinSlots; ++k)
            if (k == j) slot = a.pos[k];
        pos = __ldg(offsets + t) + (base ? __ldg(base + t) : 0u) + slot;
    } else {
        pos = atomicAdd(&cursor[t], 1u);
    }
    entries[pos] = r;
}

#ifndef SF_EMIT_MINB
#define SF_EMIT_MINB 4
#endif
__global__ void __launch_bounds__(256, SF_EMIT_MINB) k_emit_pairs(int64_t N, const int64_t* __restrict__ stats,
                                                    const GeomRec* __restrict__ geom,
                                                    const uint64_t* __restrict__ row_keys, TileGrid g,
                                                    const BinAux* __restrict__ aux,
                                                    const uint32_t* __restrict__ offsets,
                                                    uint32_t* __restrict__ cursor,
                                                    uint32_t* __restrict__ entries,
                                                    const uint32_t* __restrict__ cta_base, int64_t per) {
    if (stats[SF_STAT_OVERFLOW]) return;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t r;
    if (i >= N || !item_rank(i, stats, row_keys, r)) return;
    BinAux a;
    {
        const uint4* src = reinterpret_cast<const uint4*>(aux + i);
        uint4* dst = reinterpret_cast<uint4*>(&a);
#pragma unroll
        for (int k = 0; k < (int)(sizeof(BinAux) / 16); ++k) dst[k] = src[k];
    }
    const int w = a.w;
    int j = 0;
    const uint32_t* base = cta_base ? cta_base + (size_t)(i / per) * (g.tiles_x * g.tiles_y) : nullptr;
    // frame mode: which half tiles of the hit tile the splat's patch tests may
    // see the Gaussian in (entry bits 31 / 30; moved to the flag array by the sort)
    HalfTest ht;
    if (row_keys) ht = half_test_of(*reinterpret_cast<const GeomF32*>(geom + i));
    auto tagged = [&](int tx, int ty) -> uint32_t {
        return row_keys ? r | (half_tile_flags(ht, tx * SF_TILE, ty * SF_TILE) << kEntryFlagShift) : r;
    };
    if (w * (int)a.h <= 64) {
        // row by row over the hit mask (row-major bits, w per row): no division per hit
        unsigned long long mask = a.mask;
        const unsigned long long row_bits = w >= 64 ? ~0ull : (1ull << w) - 1ull;
        for (int ty = a.ty0; mask; ++ty) {
            unsigned long long rm = mask & row_bits;
            mask = w >= 64 ? 0ull : mask >> w;
            while (rm) {
                const int tx = a.tx0 + __ffsll((long long)rm) - 1;
                rm &= rm - 1;
                emit_one(j++, ty * g.tiles_x + tx, tagged(tx, ty), a, offsets, base, cursor, entries);
            }
        }
        return;
    }
    // rectangles over 64 tiles: repeat the exact tests (same row-major hit order)
    Proj64 p = geom_proj(geom[i]);
    const MahalPre mp = mahal_pre(p.mx, p.my, p.a, p.b, p.c);
    for (int ty = a.ty0; ty < a.ty0 + (int)a.h; ++ty)
        for (int tx = a.tx0; tx < a.tx0 + w; ++tx)
            if (tile_hit(mp, tx, ty, g))
                emit_one(j++, ty * g.tiles_x + tx, tagged(tx, ty), a, offsets, base, cursor, entries);
}

// ---------------------------------------------------------------------------
// per-tile sort of depth ranks (restores canonical order inside each bucket)

constexpr int kSortSmemElems = 8192;

__device__ void block_bitonic_sort(uint32_t* s, int N) {
    // N is a power of two; ascending.
    for (int k = 2; k <= N; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int p = threadIdx.x; p < (N >> 1); p += blockDim.x) {
                int i = 2 * j * (p / j) + (p % j);
                int ixj = i + j;
                bool up = ((i & k) == 0);
                uint32_t a = s[i], b = s[ixj];
                if ((a > b) == up) {
                    s[i] = b;
                    s[ixj] = a;
                }
            }
            __syncthreads();
        }
    }
}

// LSD 1-bit stable split sort through global scratch (rare, very long lists).
__device__ void block_radix_split_global(uint32_t* a, uint32_t* b, int n, int nbits) {
    typedef cub::BlockScan<int, 256> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int s_zero;
    uint32_t* src = a;
    uint32_t* dst = b;
    for (int bit = 0; bit < nbits; ++bit) {
        int z = 0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) z += !((src[i] >> bit) & 1u);
        int zsum;
        Scan(tmp).ExclusiveSum(z, z, zsum);
        if (threadIdx.x == 0) s_zero = zsum;
        __syncthreads();
        int base0 = 0, base1 = s_zero;
        for (int start = 0; start < n; start += blockDim.x) {
            int i = start + threadIdx.x;
            bool valid = i < n;
            uint32_t v = valid ? src[i] : 0u;
            int isz = (valid && !((v >> bit) & 1u)) ? 1 : 0;
            int ex, tot;
            Scan(tmp).ExclusiveSum(isz, ex, tot);
            if (valid) dst[isz ? base0 + ex : base1 + ((int)threadIdx.x - ex)] = v;
            int chunk = min((int)blockDim.x, n - start);
            base0 += tot;
            base1 += chunk - tot;
            __syncthreads();
        }
        uint32_t* t = src;
        src = dst;
        dst = t;
        __syncthreads();
    }
    if (src != a) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = src[i];
        __syncthreads();
    }
}

__device__ __forceinline__ int rank_bits(const int64_t* stats) {
    int64_t nvis = stats[SF_STAT_VISIBLE];
    int nbits = 1;
    while (nbits < 32 && ((int64_t)1 << nbits) < nvis) ++nbits;
    return nbits;
}

// Per-tile sort of unique depth ranks, n <= CAP: MSD bucket sort in shared
// memory.  Keys are distinct, so placement may use atomics (no stability is
// needed): bucket ~ (key - min) * NB / (max - min + 1), histogram, scan,
// scatter, then an insertion sort inside each bucket (a few keys on average).
// A tile whose largest bucket exceeds kMaxBucket (strongly clustered ranks)
// is bitonic-sorted instead.  The sorted ranks are written back as rows.
#ifndef SF_TS_CAP
#define SF_TS_CAP 4096
#endif
#ifndef SF_TS_NB
#define SF_TS_NB 1024
#endif
#ifndef SF_TS_MAXB
#define SF_TS_MAXB 48
#endif
constexpr int kMaxBucket = SF_TS_MAXB;
template <int CAP, int NB>
__global__ void __launch_bounds__(256) k_tile_sort_bucket(const uint32_t* __restrict__ offsets,
                                                          uint32_t* __restrict__ entries, int lo_exclusive,
                                                          const int64_t* __restrict__ stats,
                                                          const uint32_t* __restrict__ rank_to_row) {
    if (stats[SF_STAT_OVERFLOW]) return;
    extern __shared__ __align__(16) uint32_t sort_smem[];
    uint32_t* keys = sort_smem;         // CAP
    uint32_t* outk = sort_smem + CAP;   // CAP
    __shared__ uint32_t start[NB + 1];
    __shared__ uint32_t cursor[NB];
    __shared__ uint32_t s_min, s_max, s_big;
    const int t = blockIdx.x;
    const uint32_t beg = offsets[t], end = offsets[t + 1];
    const int n = (int)(end - beg);
    if (n <= lo_exclusive || n > CAP) return;
    uint32_t* e = entries + beg;
    if (threadIdx.x == 0) {
        s_min = 0xffffffffu;
        s_max = 0;
        s_big = 0;
    }
    for (int b = threadIdx.x; b < NB; b += blockDim.x) cursor[b] = 0;
    __syncthreads();
    uint32_t mn = 0xffffffffu, mx = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t k = e[i];
        keys[i] = k;
        mn = min(mn, k);
        mx = max(mx, k);
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&s_min, mn);
        atomicMax(&s_max, mx);
    }
    __syncthreads();
    const uint32_t kmin = s_min;
    // bucket = floor((key - min) * NB / span) in fp32: rounding is monotone, so
    // the buckets stay in key order (the sorted output does not depend on where
    // exactly the boundaries fall) -- no 64-bit integer division per key
    const float bscale = (float)NB / ((float)(s_max - kmin) + 1.0f);
    auto bucket_of = [&](uint32_t k) { return min(NB - 1, (int)((float)(k - kmin) * bscale)); };
    // histogram
    for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&cursor[bucket_of(keys[i])], 1u);
    __syncthreads();
    // exclusive scan of the NB bucket counts (NB / 256 per thread)
    {
        typedef cub::BlockScan<uint32_t, 256> Scan;
        __shared__ typename Scan::TempStorage tmp;
        constexpr int PER = NB / 256;
        uint32_t c[PER], sum = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            c[j] = cursor[threadIdx.x * PER + j];
            sum += c[j];
        }
        uint32_t ex;
        Scan(tmp).ExclusiveSum(sum, ex);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int b = threadIdx.x * PER + j;
            start[b] = ex;
            cursor[b] = ex;
            if (c[j] > (uint32_t)kMaxBucket) s_big = 1;
            ex += c[j];
        }
        if (threadIdx.x == 255) start[NB] = ex;
    }
    __syncthreads();
    if (s_big) {
        // clustered ranks: bitonic sort of the whole list
        int N = 2;
        while (N < n) N <<= 1;
        for (int i = n + threadIdx.x; i < N; i += blockDim.x) keys[i] = 0xffffffffu;
        __syncthreads();
        block_bitonic_sort(keys, N);
        for (int i = threadIdx.x; i < n; i += blockDim.x) e[i] = rank_to_row ? __ldg(rank_to_row + keys[i]) : keys[i];
        return;
    }
    // scatter into buckets
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t k = keys[i];
        outk[atomicAdd(&cursor[bucket_of(k)], 1u)] = k;
    }
    __syncthreads();
    // insertion sort inside each bucket
    for (int b = threadIdx.x; b < NB; b += blockDim.x) {
        const int b0 = (int)start[b], b1 = (int)start[b + 1];
        for (int i = b0 + 1; i < b1; ++i) {
            const uint32_t k = outk[i];
            int j = i - 1;
            while (j >= b0 && outk[j] > k) {
                outk[j + 1] = outk[j];
                --j;
            }
            outk[j + 1] = k;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) e[i] = rank_to_row ? __ldg(rank_to_row + outk[i]) : outk[i];
}

// Longer lists: bitonic sort in shared memory up to 8192 entries, else a
// stable 1-bit LSD split through global scratch.
__global__ void __launch_bounds__(256) k_tile_sort_large(const uint32_t* __restrict__ offsets,
                                                         uint32_t* __restrict__ entries,
                                                         uint32_t* __restrict__ scratch, int lo_exclusive,
                                                         const int64_t* __restrict__ stats,
                                                         const uint32_t* __restrict__ rank_to_row) {
    if (stats[SF_STAT_OVERFLOW]) return;
    __shared__ uint32_t s[kSortSmemElems];
    int t = blockIdx.x;
    uint32_t beg = offsets[t], end = offsets[t + 1];
    int n = (int)(end - beg);
    if (n <= lo_exclusive) return;
    uint32_t* e = entries + beg;
    if (n <= kSortSmemElems) {
        int N = 2;
        while (N < n) N <<= 1;
        for (int i = threadIdx.x; i < N; i += blockDim.x) s[i] = (i < n) ? e[i] : 0xffffffffu;
        __syncthreads();
        block_bitonic_sort(s, N);
        for (int i = threadIdx.x; i < n; i += blockDim.x) e[i] = rank_to_row ? rank_to_row[s[i]] : s[i];
    } else {
        block_radix_split_global(e, scratch + beg, n, rank_bits(stats));
        if (rank_to_row)
            for (int i = threadIdx.x; i < n; i += blockDim.x) e[i] = rank_to_row[e[i]];
    }
}

// ---------------------------------------------------------------------------
// Frame mode: per-tile sort of ROWS by (depth key, row).  Reference order
// lexsort((ids, depths)) (projection.py:396) restricted to one tile, then the
// stable argsort by tile (projection.py:443-449) keeps it inside each list:
// so sorting each tile's rows by (fp64 depth, id) gives the reference's lists
// without ranking all Gaussians globally.  Depth keys are the fp64 depth bits
// (positive doubles order like their bits; sf_preprocess.cu) and rows are in
// id order, so (key, row) compares exactly like (depth, id).  The keys of a
// tile are gathered from the L2-resident key array (8 B per entry).
//
// Sort: MSD bucket pass in shared memory -- as many buckets as list slots,
// bucket = (key - min) >> shift (monotone, so buckets stay in key order),
// histogram, scan, scatter of entry indices into their buckets; then every
// entry's final position is its bucket's start plus the number of bucket
// members ordering before it on (key, row) -- each entry independently, so
// there is no serial insertion chain (keys are unique as (key, row) pairs).
template <int CAP>
struct TileSortDepth {
    // keys, rows, bucket order (CAP each), bucket starts and cursors (NB = CAP)
    static constexpr size_t kSmem = (size_t)CAP * (8 + 4 + 2) + (size_t)(2 * CAP + 1) * 4;
};


template <int CAP, int NB, int NT>
__device__ __forceinline__ void tile_sort_depth_one(int t, const uint32_t* __restrict__ offsets,
                                                    uint32_t* __restrict__ entries, int lo_exclusive,
                                                    const uint64_t* __restrict__ row_keys,
                                                    uint8_t* __restrict__ flags);

// NT threads per CTA: the mid-size and long lists use 384 / 512 (shared memory caps
// the CTAs per SM, so more warps per CTA hide the key-gather latency); MINB
// CTAs per SM bounds the registers so that the shared memory sets residency
template <int CAP, int NB, int NT, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) k_tile_sort_depth(const uint32_t* __restrict__ offsets,
                                                         uint32_t* __restrict__ entries, int lo_exclusive,
                                                         const int64_t* __restrict__ stats,
                                                         const uint64_t* __restrict__ row_keys,
                                                         const uint32_t* __restrict__ big,
                                                         uint8_t* __restrict__ flags) {
    static_assert(CAP <= 65536 && NB % NT == 0, "index width / scan split");
    if (stats[SF_STAT_OVERFLOW]) return;
    if (!big) {
        tile_sort_depth_one<CAP, NB, NT>(blockIdx.x, offsets, entries, lo_exclusive, row_keys, flags);
        return;
    }
    // long lists only: the tiles k_tile_scan listed
    const int nb = (int)big[0];
    for (int i = blockIdx.x; i < nb; i += gridDim.x) {
        tile_sort_depth_one<CAP, NB, NT>((int)big[1 + i], offsets, entries, lo_exclusive, row_keys, flags);
        __syncthreads();
    }
}

template <int CAP, int NB, int NT>
__device__ __forceinline__ void tile_sort_depth_one(int t, const uint32_t* __restrict__ offsets,
                                                    uint32_t* __restrict__ entries, int lo_exclusive,
                                                    const uint64_t* __restrict__ row_keys,
                                                    uint8_t* __restrict__ flags) {
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) unsigned char ts_smem[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(ts_smem);           // CAP
    uint32_t* rows = reinterpret_cast<uint32_t*>(keys + CAP);       // CAP
    uint16_t* order = reinterpret_cast<uint16_t*>(rows + CAP);      // CAP: entry indices grouped by bucket
    uint32_t* start = reinterpret_cast<uint32_t*>(order + CAP);     // NB + 1
    uint32_t* cursor = start + NB + 1;                              // NB
    static_assert(NB == CAP && CAP % 4 == 0, "one bucket per entry slot; 4-byte aligned bucket arrays");
    __shared__ unsigned long long w_min[NW], w_max[NW];  // per warp
    const uint32_t beg = offsets[t], end = offsets[t + 1];
    const int n = (int)(end - beg);
    if (n <= lo_exclusive || n > CAP) return;
    uint32_t* e = entries + beg;
    for (int b = threadIdx.x; b < NB; b += blockDim.x) cursor[b] = 0;
    // rows (coalesced) and their keys (L2 gathers), 8 in flight per thread
    unsigned long long mn = ~0ull, mx = 0ull;
    for (int i0 = threadIdx.x; i0 < n; i0 += 8 * blockDim.x) {
        uint32_t r[8];
        uint64_t k[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x;
            r[u] = i < n ? e[i] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x;
            k[u] = i < n ? __ldg(row_keys + (r[u] & kEntryRowMask)) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x;
            if (i < n) {
                rows[i] = r[u];
                keys[i] = k[u];
                mn = min(mn, (unsigned long long)k[u]);
                mx = max(mx, (unsigned long long)k[u]);
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        w_min[threadIdx.x >> 5] = mn;
        w_max[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        mn = min(mn, w_min[w]);
        mx = max(mx, w_max[w]);
    }
    const uint64_t kmin = mn;
    // bucket = (key - min) >> shift, the smallest shift that maps the span
    // below NB: monotone in the key, between NB / 2 and NB buckets used
    const uint64_t span = mx - kmin;
    constexpr int kLogNB = 31 - __builtin_clz((unsigned)NB);  // floor(log2 NB): NB need not be a power of two
    const int shift = max(0, 64 - __clzll((long long)span) - kLogNB);
    auto bucket_of = [&](uint64_t k) { return (int)((k - kmin) >> shift); };
    for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&cursor[bucket_of(keys[i])], 1u);
    __syncthreads();
    {
        typedef cub::BlockScan<uint32_t, NT> Scan;
        __shared__ typename Scan::TempStorage tmp;
        constexpr int PER = NB / NT;
        uint32_t c[PER], sum = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            c[j] = cursor[threadIdx.x * PER + j];
            sum += c[j];
        }
        uint32_t ex;
        Scan(tmp).ExclusiveSum(sum, ex);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int b = threadIdx.x * PER + j;
            start[b] = ex;
            cursor[b] = ex;
            ex += c[j];
        }
        if (threadIdx.x == NT - 1) start[NB] = ex;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) order[atomicAdd(&cursor[bucket_of(keys[i])], 1u)] = (uint16_t)i;
    __syncthreads();
    // final position = bucket start + the members of the bucket that order
    // before the entry on (key, row): independent per entry (no serial chain);
    // the rows are in shared memory, so the list is overwritten in place
    // (rows compare without their half-tile flags; the flags go to their own array)
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        const int i = order[p];
        const uint64_t ki = keys[i];
        const uint32_t ri = rows[i] & kEntryRowMask;
        const int b = bucket_of(ki);
        const int q0 = (int)start[b], q1 = (int)start[b + 1];
        int r = q0;
        // not unrolled, compare without branches: buckets hold ~2 entries, and
        // nvcc's 8-way unroll with a fully unrolled remainder cost every warp
        // ~330 instructions per pass whatever the trip count (ncu, config C)
#pragma unroll 1
        for (int q = q0; q < q1; ++q) {
            const int j = order[q];
            const uint64_t kj = keys[j];
            const uint32_t rj = rows[j] & kEntryRowMask;
            r += (int)((kj < ki) | ((kj == ki) & (rj < ri)));
        }
        e[r] = ri;
        flags[beg + r] = (uint8_t)(rows[i] >> kEntryFlagShift);
    }
}

// Lists over 8192 entries (pathological overlap): a stable LSD split sort in
// global scratch, first on the row bits, then on the 64 key bits.
__device__ __noinline__ void tile_sort_depth_split(int t, const uint32_t* __restrict__ offsets,
                                                   uint32_t* __restrict__ entries, uint32_t* __restrict__ scratch,
                                                   int lo_exclusive, const uint64_t* __restrict__ row_keys,
                                                   uint8_t* __restrict__ flags);
__global__ void __launch_bounds__(256) k_tile_sort_depth_large(const uint32_t* __restrict__ offsets,
                                                               uint32_t* __restrict__ entries,
                                                               uint32_t* __restrict__ scratch, int lo_exclusive,
                                                               const int64_t* __restrict__ stats,
                                                               const uint64_t* __restrict__ row_keys,
                                                               const uint32_t* __restrict__ big,
                                                               uint8_t* __restrict__ flags) {
    if (stats[SF_STAT_OVERFLOW]) return;
    const int nb = (int)big[0];
    for (int i = blockIdx.x; i < nb; i += gridDim.x) {
        tile_sort_depth_split((int)big[1 + i], offsets, entries, scratch, lo_exclusive, row_keys, flags);
        __syncthreads();
    }
}

__device__ __noinline__ void tile_sort_depth_split(int t, const uint32_t* __restrict__ offsets,
                                                   uint32_t* __restrict__ entries, uint32_t* __restrict__ scratch,
                                                   int lo_exclusive, const uint64_t* __restrict__ row_keys,
                                                   uint8_t* __restrict__ flags) {
    typedef cub::BlockScan<int, 256> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int s_zero;
    const uint32_t beg = offsets[t], end = offsets[t + 1];
    const int n = (int)(end - beg);
    if (n <= lo_exclusive) return;
    uint32_t* src = entries + beg;
    uint32_t* dst = scratch + beg;
    uint32_t rmax = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) rmax = max(rmax, src[i] & kEntryRowMask);
    rmax = __reduce_max_sync(0xffffffffu, rmax);
    __shared__ uint32_t s_rmax;
    if (threadIdx.x == 0) s_rmax = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicMax(&s_rmax, rmax);
    __syncthreads();
    int row_bits = 1;
    while (row_bits < 32 && (s_rmax >> row_bits)) ++row_bits;
    for (int pass = 0; pass < row_bits + 64; ++pass) {
        auto bit_of = [&](uint32_t r) -> uint32_t {
            r &= kEntryRowMask;
            return pass < row_bits ? (r >> pass) & 1u : (uint32_t)(__ldg(row_keys + r) >> (pass - row_bits)) & 1u;
        };
        int z = 0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) z += !bit_of(src[i]);
        int zsum;
        Scan(tmp).ExclusiveSum(z, z, zsum);
        if (threadIdx.x == 0) s_zero = zsum;
        __syncthreads();
        int base0 = 0, base1 = s_zero;
        for (int s0 = 0; s0 < n; s0 += blockDim.x) {
            const int i = s0 + threadIdx.x;
            const bool valid = i < n;
            const uint32_t v = valid ? src[i] : 0u;
            const int isz = (valid && !bit_of(v)) ? 1 : 0;
            int ex, tot;
            Scan(tmp).ExclusiveSum(isz, ex, tot);
            if (valid) dst[isz ? base0 + ex : base1 + ((int)threadIdx.x - ex)] = v;
            base0 += tot;
            base1 += min((int)blockDim.x, n - s0) - tot;
            __syncthreads();
        }
        uint32_t* tt = src;
        src = dst;
        dst = tt;
        __syncthreads();
    }
    // plain rows to the entries, half-tile flags to their array
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t v = src[i];
        flags[beg + i] = (uint8_t)(v >> kEntryFlagShift);
        entries[beg + i] = v & kEntryRowMask;
    }
}

void launch_binning(int64_t n_items, const int64_t* stats, const GeomRec* geom, const uint64_t* row_keys,
                    uint8_t* entry_flags, int W, int H, int64_t pair_capacity, uint32_t* tile_counts,
                    uint32_t* tile_offsets, uint32_t* tile_cursor,
                    uint32_t* entries, uint32_t* sort_scratch, BinAux* aux, uint32_t* cta_base, int tile_row0,
                    int tile_row1, cudaStream_t st) {
    TileGrid g{W, H, (W + SF_TILE - 1) / SF_TILE, (H + SF_TILE - 1) / SF_TILE, 0, 0};
    g.ty_lo = tile_row0;
    g.ty_hi = (tile_row1 > tile_row0 ? tile_row1 : g.tiles_y) - 1;
    int n_tiles = g.tiles_x * g.tiles_y;
    cudaMemsetAsync(tile_counts, 0, sizeof(uint32_t) * 2 * n_tiles, st);
    int blocks = n_items > 0 ? ceil_div(n_items, 256) : 0;
    const bool agg = cta_base && n_tiles <= kAggMaxTiles && n_items > 0;
    const int64_t per = agg ? (n_items + kCountCTAs - 1) / kCountCTAs : 1;
    if (agg) {
        const size_t smem = sizeof(uint32_t) * n_tiles;
        ensure_smem_attr((const void*)k_count_pairs_agg, smem);
        k_count_pairs_agg<<<kCountCTAs, 512, smem, st>>>(n_items, per, stats, geom, row_keys, g, tile_counts, aux,
                                                         cta_base);
    } else if (blocks) {
        k_count_pairs<<<blocks, 256, 0, st>>>(n_items, stats, geom, row_keys, g, tile_counts, aux);
    }
    uint32_t* big = tile_cursor + n_tiles;  // long-list tiles (tile_cursor holds 4 n_tiles + 3)
    uint32_t* mid = big + n_tiles + 1;      // mid-size lists (2048, 3072]
    uint32_t* mid4 = mid + n_tiles + 1;     // (3072, 4096]
    k_tile_scan<<<1, 1024, 0, st>>>(n_tiles, tile_counts, tile_offsets, tile_cursor, pair_capacity,
                                    const_cast<int64_t*>(stats), big, mid, mid4);
    if (blocks)
        k_emit_pairs<<<blocks, 256, 0, st>>>(n_items, stats, geom, row_keys, g, aux, tile_offsets, tile_cursor,
                                             entries, agg ? cta_base : nullptr, per);
    if (row_keys) {
        // frame mode: each tile's rows into (depth, row) order -- the canonical
        // order, since scene rows are id-ordered; no global depth sort
        constexpr size_t s0 = TileSortDepth<2048>::kSmem, s1 = TileSortDepth<4096>::kSmem,
                         s2 = TileSortDepth<8192>::kSmem, s15 = TileSortDepth<3072>::kSmem;
        ensure_smem_attr((const void*)k_tile_sort_depth<2048, 2048, 256, 4>, s0);
        ensure_smem_attr((const void*)k_tile_sort_depth<3072, 3072, 384, 3>, s15);
        ensure_smem_attr((const void*)k_tile_sort_depth<4096, 4096, 512>, s1);
        ensure_smem_attr((const void*)k_tile_sort_depth<8192, 8192, 512>, s2);
        const int sms = device_sm_count();
        static_assert(kShortList == 4096 && kMidList == 3072 && kTinyList == 2048, "list-size classes");
        // the classes touch disjoint tiles: the mid-size lists (2048, 4096] -- the bulk
        // of the entries in dense views -- go first on a side stream, the <= 2048 lists
        // on the frame's stream fill the SMs as the mid-size CTAs drain
        SideStream* ss = side_stream(st);
        cudaStream_t sm = st;
        if (ss && cudaEventRecord(ss->fork, st) == cudaSuccess && cudaStreamWaitEvent(ss->s, ss->fork, 0) == cudaSuccess)
            sm = ss->s;
        // (2048, 3072]: 3 CTAs per SM (71 KB each), the rest 2 per SM; each grid is
        // exactly one resident wave striding over k_tile_scan's list (a second
        // partial wave would double the slowest CTAs' tile count)
        k_tile_sort_depth<3072, 3072, 384, 3><<<std::min(n_tiles, 3 * sms), 384, s15, sm>>>(tile_offsets, entries, 2048,
                                                                                      stats, row_keys, mid, entry_flags);
        k_tile_sort_depth<4096, 4096, 512><<<std::min(n_tiles, 2 * sms), 512, s1, sm>>>(tile_offsets, entries, 3072, stats,
                                                                                  row_keys, mid4, entry_flags);
        // one CTA per tile for the common lists (<= 2048 entries: 28 KB of
        // shared memory, 4 CTAs per SM); the long ones by grids striding over
        // the tiles k_tile_scan listed
        k_tile_sort_depth<2048, 2048, 256, 4><<<n_tiles, 256, s0, st>>>(tile_offsets, entries, 0, stats, row_keys, nullptr,
                                                                entry_flags);
        k_tile_sort_depth<8192, 8192, 512><<<std::min(n_tiles, sms), 512, s2, st>>>(tile_offsets, entries, 4096, stats,
                                                                              row_keys, big, entry_flags);
        k_tile_sort_depth_large<<<std::min(n_tiles, sms), 256, 0, st>>>(tile_offsets, entries, sort_scratch, 8192,
                                                                        stats, row_keys, big, entry_flags);
        if (sm != st) {
            cudaEventRecord(ss->join, sm);
            cudaStreamWaitEvent(st, ss->join, 0);
        }
        return;
    }
    // sf_bin mode: unique ranks; most lists fit the shared-memory bucket sort
    // (<= 4096), the rest go to the larger-capacity kernels (each CTA skips
    // other sizes)
    ensure_smem_attr((const void*)k_tile_sort_bucket<8192, 1024>, 2 * 8192 * 4);
    k_tile_sort_bucket<SF_TS_CAP, SF_TS_NB><<<n_tiles, 256, 2 * SF_TS_CAP * 4, st>>>(tile_offsets, entries, 0, stats,
                                                                                   nullptr);
    k_tile_sort_bucket<8192, 1024><<<n_tiles, 256, 2 * 8192 * 4, st>>>(tile_offsets, entries, SF_TS_CAP, stats,
                                                                       nullptr);
    k_tile_sort_large<<<n_tiles, 256, 0, st>>>(tile_offsets, entries, sort_scratch, 8192, stats, nullptr);
}

}  // namespace sf
