// sf_capi.cu -- extern "C" entry points (include/splatfield_b200.h).
//
// Validation happens on the host before any launch, mirroring where the
// reference raises (sparse_splat.py:114-122, query.py:73-90).  All scratch
// is carved from the caller's workspace; nothing allocates.
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <cub/cub.cuh>

#include "sf_common.cuh"

using namespace sf;

static thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

static int check_cuda(const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SF_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
    return SF_OK;
}

extern "C" const char* sf_last_error(void) { return g_err; }

namespace sf {
void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
}  // namespace sf

extern "C" void* sf_event_create(void) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return (void*)e;
}
extern "C" void sf_event_destroy(void* e) {
    if (e) cudaEventDestroy((cudaEvent_t)e);
}
extern "C" float sf_event_elapsed_ms(void* a, void* b) {
    float ms = -1.f;
    if (cudaEventSynchronize((cudaEvent_t)b) != cudaSuccess) return -1.f;
    if (cudaEventElapsedTime(&ms, (cudaEvent_t)a, (cudaEvent_t)b) != cudaSuccess) return -1.f;
    return ms;
}
extern "C" int sf_abi_version(void) { return 4; }

extern "C" int sf_decode_fused(int32_t n_levels, int32_t L, int32_t K, int32_t D) {
    return blend_dec_supported(n_levels, L, K, D) ? 1 : 0;
}

// Relevancy is fused into the blend epilogue while the coefficient tile is on
// chip.  It is computed from the map in HBM instead (so the frame needs a
// coefficient map buffer) when the channels span several blend CTAs, or when
// the tensor-core splat (L = 64, <= 3 levels, <= 12 channels per Gaussian)
// renders the frame and the canonical count is not its fused 4: every query
// frame of a shape then uses the same splat kernel, hence the same W.
static bool relevancy_fused(int n_levels, int L, int K, int n_canon) {
    const int n_ch = n_levels * L;
    if (n_ch > 192) return false;
    const bool tc = L == 64 && n_levels <= 3 && n_levels * K <= 12;
    return !tc || n_canon == 4;
}

extern "C" int sf_relevancy_fused(int32_t n_levels, int32_t L, int32_t K, int32_t n_canon) {
    return relevancy_fused(n_levels, L, K, n_canon) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// frame workspace layout

struct FrameWs {
    BinAux* aux;
    uint32_t* cta_base;
    uint64_t* keys_in;  // per row: fp64 depth bits, ~0 = culled
    uint32_t* vals_in;
    int64_t* stats;
    double* stats_f;
    GeomRec* geom;
    unsigned char* chan;
    uint32_t* tile_counts;
    uint32_t* tile_offsets;
    uint32_t* tile_cursor;
    uint32_t* entries;
    uint8_t* entry_flags;  // per entry: half-tile flags (bit 0 top, bit 1 bottom half)
    uint32_t* scratch;
    double* proj_cb;
    double* filter_tmp;
    void* sel_ws;
    float* dec_ws;
    float* dec_img;   // fused decode: pre-swizzled tf32 hi/lo codebook chunks
    float* fixw;      // exact coefficients of replayed pixels for k_fixup_decode (kFixWPixels x channels)
    uint32_t* fixup;  // [0] = count, [1] = the splat's half-tile claim counter, [2, 4) pad, then the list
};

// Exact-replay list capacity: every pixel can be listed at most once, so
// W * H can never overflow.  SF_FIXUP_CAPACITY (tests only) lowers it to
// exercise the overflow report: the blend still counts every ambiguous pixel
// (SF_STAT_FIXUPS), the host raises when the count exceeds the capacity.
static uint32_t fixup_capacity(int W, int H) {
    static const long forced = [] {
        const char* e = getenv("SF_FIXUP_CAPACITY");
        return e ? atol(e) : -1L;
    }();
    const int64_t px = (int64_t)(W > 0 ? W : 1) * (H > 0 ? H : 1);
    if (forced >= 0 && forced < px) return (uint32_t)forced;
    return (uint32_t)px;
}
extern "C" int64_t sf_fixup_capacity(int32_t W, int32_t H) { return (int64_t)fixup_capacity(W, H); }

static constexpr int kMaxCanon = 64;
// replayed pixels whose features k_fixup_decode redoes in one batch (more: the
// replay kernel redoes them itself)
static constexpr uint32_t kFixWPixels = 16384;

static size_t carve_frame(void* base, size_t cap, int64_t G, int W, int H, int n_levels, int L,
                          int K, int D, int64_t pair_cap, FrameWs* ws) {
    Carver c(base, cap);
    int64_t Gp = G > 0 ? G : 1;
    int n_tiles = ((W + SF_TILE - 1) / SF_TILE) * ((H + SF_TILE - 1) / SF_TILE);
    int C = n_levels * K;
    ws->aux = c.take<BinAux>(Gp);
    ws->cta_base = c.take<uint32_t>(bin_cta_base_elems(W, H));
    ws->keys_in = c.take<uint64_t>(Gp);
    ws->vals_in = c.take<uint32_t>(Gp);
    ws->stats = c.take<int64_t>(16);
    ws->stats_f = c.take<double>(8 + 2 * kMaxLevels);
    ws->geom = c.take<GeomRec>(Gp);
    ws->chan = c.take<unsigned char>((size_t)Gp * chan_rec_bytes(C));
    ws->tile_counts = c.take<uint32_t>(2 * n_tiles);
    ws->tile_offsets = c.take<uint32_t>(n_tiles + 1);
    ws->tile_cursor = c.take<uint32_t>(4 * n_tiles + 3);  // + the long / two mid-size list tile lists (launch_binning)
    ws->entries = c.take<uint32_t>(pair_cap > 0 ? pair_cap : 1);
    ws->entry_flags = c.take<uint8_t>(pair_cap > 0 ? pair_cap : 1);
    ws->scratch = c.take<uint32_t>(pair_cap > 0 ? pair_cap : 1);
    ws->proj_cb = c.take<double>((size_t)n_levels * L * (1 + kMaxCanon));
    ws->filter_tmp = c.take<double>((size_t)n_levels * W * H);
    ws->sel_ws = c.take<char>(select_segment_ws_bytes(n_levels, H, W));
    ws->dec_ws = c.take<float>(decode_ws_bytes(L, D) / sizeof(float));
    ws->dec_img = c.take<float>(blend_dec_image_bytes(n_levels, D) / sizeof(float));
    ws->fixup = c.take<uint32_t>((size_t)fixup_capacity(W, H) + 4);
    ws->fixw = c.take<float>(D > 0 ? (size_t)kFixWPixels * n_levels * L : 1);
    return c.off;
}

extern "C" int sf_frame_workspace_bytes(int64_t G, int32_t W, int32_t H, int32_t n_levels,
                                        int32_t L, int32_t K, int32_t D, int64_t pair_cap, size_t* bytes) {
    FrameWs ws;
    *bytes = carve_frame(nullptr, 0, G, W, H, n_levels, L, K, D, pair_cap, &ws) + 256;
    return SF_OK;
}

static int validate_scene_cam(const SfScene* s, const SfCamera* cam) {
    if (!s || !cam) return fail(SF_ERR_VALIDATION, "null scene or camera");
    if (cam->width < 1 || cam->height < 1) return fail(SF_ERR_VALIDATION, "image size must be >= 1 pixel");
    if (!(cam->fx > 0) || !(cam->fy > 0)) return fail(SF_ERR_VALIDATION, "focal lengths must be > 0");
    if (!(cam->near_plane > 0)) return fail(SF_ERR_VALIDATION, "near plane must be > 0");
    if (s->num_gaussians < 0 || s->num_gaussians >= (int64_t)1 << kEntryFlagShift)
        return fail(SF_ERR_VALIDATION, "num_gaussians out of range");
    return SF_OK;
}

// One frame.  Projection, sort, binning and the per-frame codebook products
// go to st_prep; blend (+ decode), filter and selection to st.  When the two
// differ, `handoff` (a cudaEvent_t) orders them.
static int render_frame(const SfScene* s, const SfCamera* cam, const SfQuery* q, const SfFrame* f,
                        void* workspace, size_t workspace_bytes, cudaStream_t st_prep, cudaStream_t st,
                        cudaEvent_t handoff, int band_halo = -1) {
    int rc = validate_scene_cam(s, cam);
    if (rc) return rc;
    if (!f || f->n_levels < 1 || f->n_levels > kMaxLevels)
        return fail(SF_ERR_VALIDATION, "1..%d levels must be selected", kMaxLevels);
    LevelSelDev lv;
    lv.n = f->n_levels;
    for (int b = 0; b < f->n_levels; ++b) {
        int l = f->host_levels[b];
        if (l < 0 || l >= s->num_levels)
            return fail(SF_ERR_VALIDATION, "level %d out of range for %d levels", l, s->num_levels);
        lv.lv[b] = l;
    }
    const int W = cam->width, H = cam->height;
    const int L = s->L, K = s->K, D = s->D;
    const int C = f->n_levels * K;
    const int n_ch = f->n_levels * L;
    if (C > 16) return fail(SF_ERR_VALIDATION, "levels*K = %d exceeds 16 channels per Gaussian", C);
    if (n_ch > 65535) return fail(SF_ERR_VALIDATION, "too many channels");
    if (q) {
        if (q->n_canonicals < 1) return fail(SF_ERR_VALIDATION, "at least one canonical D-vector is required");
        if (q->n_canonicals > kMaxCanon) return fail(SF_ERR_VALIDATION, "at most %d canonicals", kMaxCanon);
        if (q->window < 1 || q->window % 2 == 0)
            return fail(SF_ERR_VALIDATION, "filter window must be odd and >= 1, got %d", q->window);
        if (q->fixed_level >= f->n_levels) return fail(SF_ERR_VALIDATION, "fixed level was not rendered");
        if (!f->relevancy_raw || !f->relevancy_filtered)
            return fail(SF_ERR_VALIDATION, "query frames need relevancy buffers");
    }
    // decode fused into the blend CTAs whenever the shape allows (features
    // then never need the coefficient map in HBM)
    const bool fused_dec = f->features && blend_dec_supported(f->n_levels, L, K, D);
    const bool rel_from_map = q && !relevancy_fused(f->n_levels, L, K, q->n_canonicals);
    bool need_cmap = (f->features != nullptr && !fused_dec) || rel_from_map;
    if (need_cmap && !f->coeff_map) return fail(SF_ERR_VALIDATION, "coefficient map buffer required");
    // band mode: owned rows [y0, y1), rendered rows = tile rows covering the
    // owned rows +- the mean-filter halo
    const bool band = f->band_y1 > f->band_y0;
    if (band && (f->band_y0 < 0 || f->band_y1 > H))
        return fail(SF_ERR_VALIDATION, "band rows [%d, %d) outside the %d-row image", f->band_y0, f->band_y1, H);
    if (!band && (f->band_y0 != 0 || f->band_y1 != 0))
        return fail(SF_ERR_VALIDATION, "empty band [%d, %d)", f->band_y0, f->band_y1);
    const int oy0 = band ? f->band_y0 : 0, oy1 = band ? f->band_y1 : H;
    // band mode renders the owned rows +- the mean-filter halo (a sweep passes
    // its window's halo, having no SfQuery)
    const int halo = band ? (q ? q->window / 2 : (band_halo > 0 ? band_halo : 0)) : 0;
    const int tiles_x = (W + SF_TILE - 1) / SF_TILE, tiles_y = (H + SF_TILE - 1) / SF_TILE;
    const int tr0 = band ? max(0, oy0 - halo) / SF_TILE : 0;
    const int tr1 = band ? (min(H, oy1 + halo) + SF_TILE - 1) / SF_TILE : tiles_y;
    const int ry0 = tr0 * SF_TILE, ry1 = min(H, tr1 * SF_TILE);  // rendered pixel rows

    FrameWs ws;
    size_t need = carve_frame(workspace, workspace_bytes, s->num_gaussians, W, H, f->n_levels, L, K, D,
                              f->pair_capacity, &ws);
    if (need > workspace_bytes) return fail(SF_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, need);

    const int64_t G = s->num_gaussians;
    if (f->events[0]) cudaEventRecord((cudaEvent_t)f->events[0], st_prep);
    if (f->reuse_lists && q) return fail(SF_ERR_VALIDATION, "reuse_lists is for frames without a query");
    if (!f->reuse_lists) {
        cudaMemsetAsync(ws.stats, 0, 16 * sizeof(int64_t), st_prep);
        cudaMemsetAsync(ws.stats_f, 0, (8 + 2 * kMaxLevels) * sizeof(double), st_prep);
    }
    cudaMemsetAsync(ws.fixup, 0, 4 * sizeof(uint32_t), st_prep);
    const unsigned char* chan = f->chan_by_row;
    if (!chan && f->reuse_lists) return fail(SF_ERR_VALIDATION, "reuse_lists needs a scatter plan (chan_by_row)");
    if (!f->reuse_lists) {
        // K1
        launch_preprocess(*s, *cam, ws.geom, ws.keys_in, ws.vals_in, ws.stats, st_prep);
        // per-row scatter plan: a scene constant for a level selection, so callers
        // may pass a cached copy (sf_pack_channels)
        if (!chan) {
            launch_pack_channels(*s, lv, ws.chan, st_prep);
            chan = ws.chan;
        }
        // K2-K4: per-tile lists of scene rows in (depth, id) order -- the depth
        // order is established per tile (k_tile_sort_depth), not globally
        launch_binning(G, ws.stats, ws.geom, ws.keys_in, ws.entry_flags, W, H, f->pair_capacity, ws.tile_counts,
                       ws.tile_offsets, ws.tile_cursor, ws.entries, ws.scratch, ws.aux, ws.cta_base, tr0, tr1,
                       st_prep);
    }
    if (q) launch_project_codebook(s->codebooks, lv, L, D, q->vector, q->canonicals, q->n_canonicals,
                                   ws.proj_cb, st_prep);
    if (f->grad_coeff_map) {
        // training backward: transpose of the splat over the same tile lists
        if (!f->grad_values) return fail(SF_ERR_VALIDATION, "grad_values buffer required");
        if (st_prep != st) {
            cudaEventRecord(handoff, st_prep);
            cudaStreamWaitEvent(st, handoff, 0);
        }
        BlendArgs t;
        memset(&t, 0, sizeof(t));
        t.W = W, t.H = H, t.tiles_x = tiles_x, t.tiles_y = tiles_y;
        t.tile0 = tr0 * tiles_x, t.n_band_tiles = (tr1 - tr0) * tiles_x;
        t.n_ch = n_ch, t.C = C, t.early_exit = f->early_exit;
        t.tile_offsets = ws.tile_offsets, t.entries = ws.entries, t.geom = ws.geom, t.chan = chan;
        t.stats = ws.stats;
        if (launch_splat_transpose(t, f->grad_coeff_map, f->grad_values, K, G, st))
            return fail(SF_ERR_VALIDATION, "transpose splat needs levels*L <= 192 channels");
        if (f->stats_i64) cudaMemcpyAsync(f->stats_i64, ws.stats, 16 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
        return check_cuda("sf_render_frame (transpose)");
    }
    // K5/K6 (+ fused relevancy)
    BlendArgs a;
    memset(&a, 0, sizeof(a));
    a.W = W;
    a.H = H;
    a.tiles_x = tiles_x;
    a.tiles_y = tiles_y;
    a.tile0 = tr0 * tiles_x;
    a.n_band_tiles = (tr1 - tr0) * tiles_x;
    a.n_ch = n_ch;
    a.C = C;
    a.early_exit = f->early_exit;
    a.tile_offsets = ws.tile_offsets;
    a.entries = ws.entries;
    a.entry_flags = ws.entry_flags;
    a.geom = ws.geom;
    a.chan = chan;
    a.fixup_count = ws.fixup;
    a.sched = ws.fixup + 1;
    a.fixup_list = ws.fixup + 4;
    a.fixup_capacity = fixup_capacity(W, H);
    a.stats = ws.stats;
    a.coeff_map = f->coeff_map;
    a.final_t = f->final_t;
    // relevancy: fused into the blend epilogue while the coefficient tile is
    // in shared memory; from the map in HBM only when the channels span
    // several blend CTAs
    a.proj_cb = (q && !rel_from_map) ? ws.proj_cb : nullptr;
    a.n_levels = f->n_levels;
    a.L = L;
    a.n_canon = q ? q->n_canonicals : 0;
    a.relevancy_raw = q ? f->relevancy_raw : nullptr;
    const void* dec_img = f->dec_image ? f->dec_image : ws.dec_img;
    if (fused_dec && !f->dec_image) launch_dec_codebook_image(s->codebooks, lv, L, D, ws.dec_img, st_prep);
    if (st_prep != st) {
        cudaEventRecord(handoff, st_prep);
        cudaStreamWaitEvent(st, handoff, 0);
    }
    if (fused_dec) {
        a.features = f->features;
        a.D = D;
        a.feat_level_stride = (int64_t)W * H * D;
        a.dec_b = dec_img;
        a.dec_scale = (const float*)((const char*)dec_img + blend_dec_image_bytes(f->n_levels, D) - 64);
        a.codebooks = s->codebooks;
        a.lv = lv;
        if (L <= 64 && D % 64 == 0) {
            a.fixup_w = ws.fixw;
            a.fixup_w_capacity = kFixWPixels;
        }
    }
    if (f->events[4]) cudaEventRecord((cudaEvent_t)f->events[4], st);
    if (launch_blend(a, st)) return fail(SF_ERR_VALIDATION, "blend configuration unsupported");
    if (rel_from_map)
        launch_relevancy_from_cmap((int64_t)W * (ry1 - ry0), n_ch, f->coeff_map + (size_t)ry0 * W * n_ch,
                                   ws.proj_cb, f->n_levels, L, q->n_canonicals, f->relevancy_raw + (size_t)ry0 * W,
                                   (int64_t)W * H, st);
    if (f->events[1]) cudaEventRecord((cudaEvent_t)f->events[1], st);
    // K7
    if (f->features && !fused_dec) {
        const int64_t HW = (int64_t)W * H;
        const int64_t P = (int64_t)W * (ry1 - ry0);  // rendered rows only
        for (int b = 0; b < f->n_levels; ++b) {
            if (launch_decode(P, L, D, f->coeff_map + (size_t)ry0 * W * n_ch + (size_t)b * L, n_ch,
                              s->codebooks + (size_t)lv.lv[b] * L * D,
                              f->features + (size_t)b * HW * D + (size_t)ry0 * W * D, ws.dec_ws, st))
                return fail(SF_ERR_VALIDATION, "decode configuration unsupported (L=%d, D=%d)", L, D);
        }
    }
    if (f->events[2]) cudaEventRecord((cudaEvent_t)f->events[2], st);
    // K8-K10
    if (q && filter_select_fusable(q->window)) {
        launch_filter_select(f->n_levels, H, W, f->relevancy_raw, q->window, f->relevancy_filtered,
                             q->fixed_level, q->threshold, f->mask, ws.stats, ws.stats_f, ws.sel_ws, st, oy0, oy1);
    } else if (q) {
        launch_mean_filter(f->n_levels, H, W, f->relevancy_raw, q->window, ws.filter_tmp,
                           f->relevancy_filtered, st, oy0, oy1);
        launch_select_segment(f->n_levels, H, W, f->relevancy_filtered, q->fixed_level, q->threshold,
                              f->mask, ws.stats, ws.stats_f, ws.sel_ws, st, oy0, oy1);
    }
    if (f->events[3]) cudaEventRecord((cudaEvent_t)f->events[3], st);
    if (f->stats_i64) cudaMemcpyAsync(f->stats_i64, ws.stats, 16 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
    if (f->stats_f64)
        cudaMemcpyAsync(f->stats_f64, ws.stats_f, (8 + 2 * f->n_levels) * sizeof(double),
                        cudaMemcpyDeviceToDevice, st);
    return check_cuda("sf_render_frame");
}

extern "C" int sf_render_frame(const SfScene* s, const SfCamera* cam, const SfQuery* q, const SfFrame* f,
                               void* workspace, size_t workspace_bytes, void* stream) {
    return render_frame(s, cam, q, f, workspace, workspace_bytes, (cudaStream_t)stream, (cudaStream_t)stream,
                        nullptr);
}

extern "C" int sf_frame_tile_lists(int64_t G, int32_t W, int32_t H, int32_t n_levels, int32_t L, int32_t K,
                                   int32_t D, int64_t pair_cap, const void* workspace, size_t workspace_bytes,
                                   uint32_t* tile_offsets, uint32_t* tile_rows, int64_t max_pairs, void* stream) {
    if (W < 1 || H < 1 || G < 0) return fail(SF_ERR_VALIDATION, "bad frame shape");
    FrameWs ws;
    size_t need = carve_frame(const_cast<void*>(workspace), workspace_bytes, G, W, H, n_levels, L, K, D, pair_cap, &ws);
    if (need > workspace_bytes) return fail(SF_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, need);
    const int n_tiles = ((W + SF_TILE - 1) / SF_TILE) * ((H + SF_TILE - 1) / SF_TILE);
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t total = 0;
    cudaMemcpyAsync(tile_offsets, ws.tile_offsets, (size_t)(n_tiles + 1) * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                    st);
    cudaMemcpyAsync(&total, ws.tile_offsets + n_tiles, sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if ((int64_t)total > max_pairs || (int64_t)total > pair_cap)
        return fail(SF_ERR_WORKSPACE, "%u pairs exceed the output (%lld)", total, (long long)max_pairs);
    if (total) cudaMemcpyAsync(tile_rows, ws.entries, (size_t)total * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    return check_cuda("sf_frame_tile_lists");
}

extern "C" int sf_query_sweep(const SfScene* s, const SfCamera* cam, const SfFrame* f, const double* prompts,
                              int32_t n_prompts, const double* canon, int32_t n_canon, int32_t window,
                              double threshold, double* filtered, uint8_t* masks, int64_t* stats_i64,
                              double* stats_f64, void* workspace, size_t workspace_bytes, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (!f || !f->coeff_map || f->features || f->grad_coeff_map)
        return fail(SF_ERR_VALIDATION, "a sweep renders a coefficient map (and no features)");
    if (n_prompts < 0 || (n_prompts > 0 && (!prompts || !filtered || !stats_i64 || !stats_f64 || !f->relevancy_raw)))
        return fail(SF_ERR_VALIDATION, "bad prompt buffers");
    if (n_canon < 1 || n_canon > kMaxCanon) return fail(SF_ERR_VALIDATION, "1..%d canonicals required", kMaxCanon);
    if (window < 1 || window % 2 == 0) return fail(SF_ERR_VALIDATION, "filter window must be odd and >= 1");
    int rc = render_frame(s, cam, nullptr, f, workspace, workspace_bytes, st, st, nullptr, window / 2);
    if (rc) return rc;
    const int W = cam->width, H = cam->height, L = s->L, D = s->D, nl = f->n_levels;
    // band mode (tile bands of one view): owned rows [oy0, oy1), rendered rows
    // [ry0, ry1) = the tile rows covering the owned rows +- the filter halo
    const bool band = f->band_y1 > f->band_y0;
    const int oy0 = band ? f->band_y0 : 0, oy1 = band ? f->band_y1 : H, halo = band ? window / 2 : 0;
    const int ry0 = band ? max(0, oy0 - halo) / SF_TILE * SF_TILE : 0;
    const int ry1 = band ? min(H, (min(H, oy1 + halo) + SF_TILE - 1) / SF_TILE * SF_TILE) : H;
    FrameWs ws;
    carve_frame(workspace, workspace_bytes, s->num_gaussians, W, H, nl, L, s->K, D, f->pair_capacity, &ws);
    LevelSelDev lv;
    lv.n = nl;
    for (int b = 0; b < nl; ++b) lv.lv[b] = f->host_levels[b];
    const int64_t hw = (int64_t)W * H, qstride = nl * hw, prow = (int64_t)W * (ry1 - ry0);
    double* raw = f->relevancy_raw;  // (n_prompts, nl, H, W)
    const float* cmap_rows = f->coeff_map + (size_t)ry0 * W * nl * L;
    // every prompt starts from the frame's counters, as a single query would
    for (int i = 0; i < n_prompts; ++i) {
        cudaMemcpyAsync(stats_i64 + (size_t)i * 16, ws.stats, 16 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(stats_f64 + (size_t)i * (8 + 2 * nl), ws.stats_f, (8 + 2 * nl) * sizeof(double),
                        cudaMemcpyDeviceToDevice, st);
    }
    // relevancy of the rendered rows: the map read once per chunk of prompts
    // (projected-codebook columns: chunk prompts + canonicals, within proj_cb's 1 + kMaxCanon)
    const int chunk = kMaxCanon + 1 - n_canon;
    bool batched = filter_select_fusable(window);
    for (int i0 = 0; i0 < n_prompts && batched; i0 += chunk) {
        const int nq = std::min(chunk, n_prompts - i0);
        launch_project_vectors(s->codebooks, lv, L, D, prompts + (size_t)i0 * D, nq, canon, n_canon, ws.proj_cb, st);
        if (launch_relevancy_sweep(prow, nl * L, cmap_rows, ws.proj_cb, nl, L, nq, n_canon,
                                   raw + i0 * qstride + (size_t)ry0 * W, qstride, hw, st)) {
            batched = false;  // shape outside the sweep kernel: per-prompt passes below
        }
    }
    if (batched) {
        // filter + statistics + mask of many prompts per launch over the owned
        // rows; partials in the row-sum buffer (unused by the fused filter)
        const size_t per_q = filter_select_batch_ws_bytes(1, nl, H, W) - 256;
        const size_t cap = sizeof(double) * (size_t)qstride - 256;
        const int qb = (int)std::max<size_t>(1, std::min<size_t>(n_prompts, cap / per_q));
        for (int i0 = 0; i0 < n_prompts; i0 += qb) {
            const int nq = std::min(qb, n_prompts - i0);
            launch_filter_select_batch(nq, nl, H, W, raw + i0 * qstride, window, filtered + i0 * qstride, threshold,
                                       masks ? masks + i0 * hw : nullptr, stats_i64 + (size_t)i0 * 16,
                                       stats_f64 + (size_t)i0 * (8 + 2 * nl), ws.filter_tmp, st, oy0, oy1);
        }
        return check_cuda("sf_query_sweep");
    }
    for (int i = 0; i < n_prompts; ++i) {
        double* ri = raw + i * qstride;
        launch_project_codebook(s->codebooks, lv, L, D, prompts + (size_t)i * D, canon, n_canon, ws.proj_cb, st);
        launch_relevancy_from_cmap(prow, nl * L, cmap_rows, ws.proj_cb, nl, L, n_canon, ri + (size_t)ry0 * W, hw, st);
        double* fi = filtered + i * qstride;
        uint8_t* mi = masks ? masks + i * hw : nullptr;
        int64_t* si = stats_i64 + (size_t)i * 16;
        double* sf = stats_f64 + (size_t)i * (8 + 2 * nl);
        if (filter_select_fusable(window)) {
            launch_filter_select(nl, H, W, ri, window, fi, -1, threshold, mi, si, sf, ws.sel_ws, st, oy0, oy1);
        } else {
            launch_mean_filter(nl, H, W, ri, window, ws.filter_tmp, fi, st, oy0, oy1);
            launch_select_segment(nl, H, W, fi, -1, threshold, mi, si, sf, ws.sel_ws, st, oy0, oy1);
        }
    }
    return check_cuda("sf_query_sweep");
}

extern "C" int sf_render_frame_split(const SfScene* s, const SfCamera* cam, const SfQuery* q, const SfFrame* f,
                                     void* workspace, size_t workspace_bytes, void* stream_prepare,
                                     void* stream_render, void* handoff_event) {
    if (stream_prepare != stream_render && !handoff_event)
        return fail(SF_ERR_VALIDATION, "two streams need a handoff event");
    return render_frame(s, cam, q, f, workspace, workspace_bytes, (cudaStream_t)stream_prepare,
                        (cudaStream_t)stream_render, (cudaEvent_t)handoff_event);
}

// ---------------------------------------------------------------------------
// project_scene

struct ProjWs {
    GeomRec* geom;
    uint64_t* keys;
    uint32_t* vals;
    int64_t* stats;
    int32_t* flags;
    int32_t* scan;
    void* cub_tmp;
    size_t cub_bytes;
};

static size_t carve_project(void* base, size_t cap, int64_t G, ProjWs* w) {
    Carver c(base, cap);
    int64_t Gp = G > 0 ? G : 1;
    w->geom = c.take<GeomRec>(Gp);
    w->keys = c.take<uint64_t>(Gp);
    w->vals = c.take<uint32_t>(Gp);
    w->stats = c.take<int64_t>(16);
    w->flags = c.take<int32_t>(Gp);
    w->scan = c.take<int32_t>(Gp);
    w->cub_bytes = project_compact_cub_bytes(Gp);
    w->cub_tmp = c.take<char>(w->cub_bytes);
    return c.off;
}

extern "C" int sf_project_workspace_bytes(int64_t G, size_t* bytes) {
    ProjWs w;
    *bytes = carve_project(nullptr, 0, G, &w) + 256;
    return SF_OK;
}

extern "C" int sf_project(const SfScene* s, const SfCamera* cam, double* means2d, double* inv_covs,
                          double* depths, double* opacities, int64_t* source_ids, int64_t* rows,
                          int64_t* count_out, void* workspace, size_t workspace_bytes, void* stream_) {
    return sf_project_rows(s, cam, nullptr, means2d, inv_covs, depths, opacities, source_ids, rows,
                           count_out, workspace, workspace_bytes, stream_);
}

extern "C" int sf_project_rows(const SfScene* s, const SfCamera* cam, const int64_t* orig_rows,
                               double* means2d, double* inv_covs, double* depths, double* opacities,
                               int64_t* source_ids, int64_t* rows, int64_t* count_out,
                               void* workspace, size_t workspace_bytes, void* stream_) {
    cudaStream_t st = (cudaStream_t)stream_;
    int rc = validate_scene_cam(s, cam);
    if (rc) return rc;
    ProjWs w;
    size_t need = carve_project(workspace, workspace_bytes, s->num_gaussians, &w);
    if (need > workspace_bytes) return fail(SF_ERR_WORKSPACE, "workspace too small");
    cudaMemsetAsync(w.stats, 0, 16 * sizeof(int64_t), st);
    launch_preprocess(*s, *cam, w.geom, w.keys, w.vals, w.stats, st);
    launch_project_compact(*s, w.geom, w.keys, orig_rows, w.flags, w.scan, means2d, inv_covs, depths,
                           opacities, source_ids, rows, count_out, w.cub_tmp, w.cub_bytes, st);
    return check_cuda("sf_project");
}

// ---------------------------------------------------------------------------
// bin_projected on arbitrary projected arrays

__global__ void k_bin_prepare(int64_t n, const double* means2d, const double* inv_covs,
                              const double* depths, const int64_t* source_ids, Proj64* proj,
                              uint64_t* id_keys, uint32_t* idx) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Proj64 p;
    p.mx = means2d[2 * i];
    p.my = means2d[2 * i + 1];
    p.a = inv_covs[4 * i];
    p.b = inv_covs[4 * i + 1];
    p.c = inv_covs[4 * i + 3];
    proj[i] = p;
    id_keys[i] = (uint64_t)source_ids[i] ^ 0x8000000000000000ull;  // signed -> monotone unsigned
    idx[i] = (uint32_t)i;
}

__device__ __forceinline__ uint64_t depth_key(double d) {
    if (d == 0.0) d = 0.0;  // -0.0 ties with +0.0 like numpy's comparison
    uint64_t b = (uint64_t)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_bin_depth_keys(int64_t n, const double* depths, const uint32_t* idx_by_id,
                                 uint64_t* keys) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = depth_key(depths[idx_by_id[i]]);
}

__global__ void k_bin_finish(int64_t n, const uint32_t* order32, const Proj64* proj, GeomRec* geom,
                             int64_t* order, int64_t* stats) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) stats[SF_STAT_VISIBLE] = n;
    if (i >= n) return;
    uint32_t r = order32[i];
    Proj64 p = proj[r];
    GeomRec g;
    memset(&g, 0, sizeof(g));
    g.mx = p.mx;
    g.my = p.my;
    g.a64 = p.a;
    g.b64 = p.b;
    g.c64 = p.c;
    geom_fill_f32(g);
    geom[i] = g;
    order[i] = r;
}

__global__ void k_offsets_to_i64(int n, const uint32_t* o32, int64_t* o64) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= n) o64[i] = o32[i];
}

struct BinWs {
    Proj64* proj;
    GeomRec* geom;
    uint64_t* k0;
    uint64_t* k1;
    uint32_t* v0;
    uint32_t* v1;
    void* cub_tmp;
    size_t cub_bytes;
    int64_t* stats;
    uint32_t* counts;
    uint32_t* offsets;
    uint32_t* cursor;
    uint32_t* scratch;
    BinAux* aux;
    uint32_t* cta_base;
};

static size_t carve_bin(void* base, size_t cap, int64_t n, int W, int H, int64_t pair_cap, BinWs* w) {
    Carver c(base, cap);
    int64_t np = n > 0 ? n : 1;
    int n_tiles = ((W + SF_TILE - 1) / SF_TILE) * ((H + SF_TILE - 1) / SF_TILE);
    w->proj = c.take<Proj64>(np);
    w->geom = c.take<GeomRec>(np);
    w->k0 = c.take<uint64_t>(np);
    w->k1 = c.take<uint64_t>(np);
    w->v0 = c.take<uint32_t>(np);
    w->v1 = c.take<uint32_t>(np);
    w->cub_bytes = depth_sort_tmp_bytes(np);
    w->cub_tmp = c.take<char>(w->cub_bytes);
    w->stats = c.take<int64_t>(16);
    w->counts = c.take<uint32_t>(2 * n_tiles);
    w->aux = c.take<BinAux>(np);
    w->cta_base = c.take<uint32_t>(bin_cta_base_elems(W, H));
    w->offsets = c.take<uint32_t>(n_tiles + 1);
    w->cursor = c.take<uint32_t>(4 * n_tiles + 3);
    w->scratch = c.take<uint32_t>(pair_cap > 0 ? pair_cap : 1);
    return c.off;
}

extern "C" int sf_bin_workspace_bytes(int64_t n, int32_t W, int32_t H, int64_t pair_cap, size_t* bytes) {
    BinWs w;
    *bytes = carve_bin(nullptr, 0, n, W, H, pair_cap, &w) + 256;
    return SF_OK;
}

extern "C" int sf_bin(int64_t n, const double* means2d, const double* inv_covs, const double* depths,
                      const int64_t* source_ids, int32_t W, int32_t H, int64_t pair_cap, int64_t* order,
                      int64_t* tile_offsets, int32_t* tile_entries, int64_t* stats_i64, void* workspace,
                      size_t workspace_bytes, void* stream_) {
    cudaStream_t st = (cudaStream_t)stream_;
    if (W < 1 || H < 1) return fail(SF_ERR_VALIDATION, "image size must be >= 1 pixel");
    if (n < 0 || n >= (int64_t)1 << 31) return fail(SF_ERR_VALIDATION, "n out of range");
    BinWs w;
    size_t need = carve_bin(workspace, workspace_bytes, n, W, H, pair_cap, &w);
    if (need > workspace_bytes) return fail(SF_ERR_WORKSPACE, "workspace too small");
    int n_tiles = ((W + SF_TILE - 1) / SF_TILE) * ((H + SF_TILE - 1) / SF_TILE);
    cudaMemsetAsync(w.stats, 0, 16 * sizeof(int64_t), st);
    int blocks = n > 0 ? ceil_div(n, 256) : 1;
    if (n > 0) {
        k_bin_prepare<<<blocks, 256, 0, st>>>(n, means2d, inv_covs, depths, source_ids, w.proj, w.k0, w.v0);
        // (depth, id) order = stable depth sort of the id-sorted sequence
        depth_sort(w.k0, w.k1, w.v0, w.v1, n, w.cub_tmp, w.cub_bytes, st);
        k_bin_depth_keys<<<blocks, 256, 0, st>>>(n, depths, w.v1, w.k0);
        depth_sort(w.k0, w.k1, w.v1, w.v0, n, w.cub_tmp, w.cub_bytes, st);
    }
    k_bin_finish<<<blocks, 256, 0, st>>>(n, w.v0, w.proj, w.geom, order, w.stats);
    launch_binning(n, w.stats, w.geom, nullptr, nullptr, W, H, pair_cap, w.counts, w.offsets, w.cursor,
                   (uint32_t*)tile_entries, w.scratch, w.aux, w.cta_base, 0, 0, st);
    k_offsets_to_i64<<<ceil_div(n_tiles + 1, 256), 256, 0, st>>>(n_tiles, w.offsets, tile_offsets);
    if (stats_i64) cudaMemcpyAsync(stats_i64, w.stats, 16 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
    return check_cuda("sf_bin");
}

// ---------------------------------------------------------------------------
// standalone ops

extern "C" size_t sf_decode_workspace_bytes(int32_t L, int32_t D) { return decode_ws_bytes(L, D); }

extern "C" int sf_decode(int64_t P, int32_t L, int32_t D, const float* w, int64_t w_stride,
                         const float* cb, float* out, void* ws, size_t ws_bytes, void* stream) {
    if (ws_bytes < decode_ws_bytes(L, D)) return fail(SF_ERR_WORKSPACE, "decode workspace too small");
    if (launch_decode(P, L, D, w, w_stride, cb, out, ws, (cudaStream_t)stream))
        return fail(SF_ERR_VALIDATION, "decode configuration unsupported (L=%d, D=%d)", L, D);
    return check_cuda("sf_decode");
}

extern "C" size_t sf_channel_plan_bytes(int64_t G, int32_t n_levels, int32_t K) {
    return (size_t)(G > 0 ? G : 1) * chan_rec_bytes(n_levels * K);
}

extern "C" int sf_pack_channels(const SfScene* s, const int32_t* host_levels, int32_t n_levels,
                                void* out, size_t out_bytes, void* stream) {
    if (!s || n_levels < 1 || n_levels > kMaxLevels) return fail(SF_ERR_VALIDATION, "bad level selection");
    if (n_levels * s->K > 16) return fail(SF_ERR_VALIDATION, "levels*K exceeds 16 channels per Gaussian");
    if (out_bytes < sf_channel_plan_bytes(s->num_gaussians, n_levels, s->K))
        return fail(SF_ERR_WORKSPACE, "channel plan buffer too small");
    LevelSelDev lv;
    lv.n = n_levels;
    for (int b = 0; b < n_levels; ++b) {
        if (host_levels[b] < 0 || host_levels[b] >= s->num_levels)
            return fail(SF_ERR_VALIDATION, "level %d out of range", host_levels[b]);
        lv.lv[b] = host_levels[b];
    }
    launch_pack_channels(*s, lv, (unsigned char*)out, (cudaStream_t)stream);
    return check_cuda("sf_pack_channels");
}

extern "C" size_t sf_decode_image_bytes(int32_t n_levels, int32_t L, int32_t K, int32_t D) {
    return blend_dec_supported(n_levels, L, K, D) ? blend_dec_image_bytes(n_levels, D) : 0;
}

extern "C" int sf_pack_decode_image(const SfScene* s, const int32_t* host_levels, int32_t n_levels, void* out,
                                    size_t out_bytes, void* stream) {
    if (!s || n_levels < 1 || n_levels > kMaxLevels) return fail(SF_ERR_VALIDATION, "bad level selection");
    if (!blend_dec_supported(n_levels, s->L, s->K, s->D))
        return fail(SF_ERR_VALIDATION, "the decode is not fused for this shape");
    if (out_bytes < blend_dec_image_bytes(n_levels, s->D)) return fail(SF_ERR_WORKSPACE, "image buffer too small");
    LevelSelDev lv;
    lv.n = n_levels;
    for (int b = 0; b < n_levels; ++b) {
        if (host_levels[b] < 0 || host_levels[b] >= s->num_levels)
            return fail(SF_ERR_VALIDATION, "level %d out of range", host_levels[b]);
        lv.lv[b] = host_levels[b];
    }
    launch_dec_codebook_image(s->codebooks, lv, s->L, s->D, out, (cudaStream_t)stream);
    return check_cuda("sf_pack_decode_image");
}

extern "C" int sf_decode_simt(int64_t P, int32_t L, int32_t D, const float* w, int64_t w_stride,
                              const float* cb, float* out, void* stream) {
    if (launch_decode_simt(P, L, D, w, w_stride, cb, out, (cudaStream_t)stream))
        return fail(SF_ERR_VALIDATION, "decode configuration unsupported (L=%d, D=%d)", L, D);
    return check_cuda("sf_decode_simt");
}

extern "C" int sf_relevancy_f32(int64_t P, int32_t D, const float* f, const double* q, const double* c,
                                int32_t nc, double* out, void* stream) {
    if (nc < 1) return fail(SF_ERR_VALIDATION, "at least one canonical D-vector is required");
    launch_relevancy_f32(P, D, f, q, c, nc, out, (cudaStream_t)stream);
    return check_cuda("sf_relevancy_f32");
}

extern "C" int sf_relevancy_f64(int64_t P, int32_t D, const double* f, const double* q, const double* c,
                                int32_t nc, double* out, void* stream) {
    if (nc < 1) return fail(SF_ERR_VALIDATION, "at least one canonical D-vector is required");
    launch_relevancy_f64(P, D, f, q, c, nc, out, (cudaStream_t)stream);
    return check_cuda("sf_relevancy_f64");
}

extern "C" int sf_mean_filter(int32_t H, int32_t W, const double* in, int32_t window, double* out,
                              void* ws, size_t ws_bytes, void* stream) {
    if (window < 1 || window % 2 == 0)
        return fail(SF_ERR_VALIDATION, "filter window must be odd and >= 1, got %d", window);
    if (ws_bytes < (size_t)H * W * sizeof(double)) return fail(SF_ERR_WORKSPACE, "workspace too small");
    launch_mean_filter(1, H, W, in, window, (double*)ws, out, (cudaStream_t)stream);
    return check_cuda("sf_mean_filter");
}

extern "C" int sf_select_segment(int32_t n_maps, int32_t H, int32_t W, const double* maps,
                                 int32_t fixed_level, double threshold, uint8_t* mask,
                                 int64_t* stats_i64, double* stats_f64, void* ws, size_t ws_bytes,
                                 void* stream) {
    if (n_maps < 1 || n_maps > 32) return fail(SF_ERR_VALIDATION, "1..32 level maps are required, got %d", n_maps);
    if ((int64_t)H * W == 0) return fail(SF_ERR_VALIDATION, "cannot localize an empty map");
    if (ws_bytes < select_segment_ws_bytes(n_maps, H, W)) return fail(SF_ERR_WORKSPACE, "workspace too small");
    launch_select_segment(n_maps, H, W, maps, fixed_level, threshold, mask, stats_i64, stats_f64, ws,
                          (cudaStream_t)stream);
    return check_cuda("sf_select_segment");
}

extern "C" size_t sf_select_segment_workspace_bytes(int32_t n_maps, int32_t H, int32_t W) {
    return select_segment_ws_bytes(n_maps, H, W);
}

extern "C" int sf_mask_rows(const double* maps, int32_t H, int32_t W, int32_t level, double lo, double hi,
                            double threshold, int32_t y0, int32_t y1, uint8_t* mask, void* stream) {
    if (H < 1 || W < 1) return fail(SF_ERR_VALIDATION, "image size must be >= 1 pixel");
    if (level < 0) return fail(SF_ERR_VALIDATION, "level must be >= 0");
    if (y0 < 0 || y1 > H || y1 < y0) return fail(SF_ERR_VALIDATION, "rows [%d, %d) outside [0, %d)", y0, y1, H);
    launch_mask_rows(H, W, maps, level, lo, hi, threshold, y0, y1, mask, (cudaStream_t)stream);
    return check_cuda("sf_mask_rows");
}

// ---------------------------------------------------------------------------
// LSV2 records -> device SoA

extern "C" int sf_lsv2_unpack(const void* records, int64_t G, int32_t num_levels, int32_t K, int32_t L,
                              float* positions, float* rotations, float* scales, float* opacities, float* colors,
                              uint16_t* coeff_indices, float* coeff_values, uint32_t* flags, void* stream) {
    if (G < 0 || num_levels < 0 || K < 1 || L < 1) return fail(SF_ERR_VALIDATION, "bad LSV2 header values");
    if (G > 0 && (!records || !positions || !rotations || !scales || !opacities || !colors || !flags ||
                  (num_levels > 0 && (!coeff_indices || !coeff_values))))
        return fail(SF_ERR_VALIDATION, "null buffer");
    launch_lsv2_unpack((const uint8_t*)records, G, num_levels, K, L, positions, rotations, scales, opacities,
                       colors, coeff_indices, coeff_values, flags, (cudaStream_t)stream);
    return check_cuda("sf_lsv2_unpack");
}
