/*
 * splatfield_b200.h -- C ABI of the B200 (sm_100a) sparse-coefficient
 * splatting + open-vocabulary query path.
 *
 * The reference package (splatfield, /root/reference/pkg/src/splatfield) is
 * pure Python/numpy and has no FFI of its own; its drop-in boundary is the
 * Python module API re-exported in splatfield/__init__.py:10-66.  Each entry
 * point below replaces one of those functions (cited per function).  A
 * maintainer binds them from splatfield with ctypes exactly as
 * paper_2507_07136_b200/_native.py does.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers unless the name says host_.
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*)
 *    and re-entrant: all scratch comes from the caller's workspace, so
 *    concurrent calls on different streams with different workspaces are
 *    safe (the reference server calls the path from many threads,
 *    server.py:11-13).
 *  - Return value: SF_OK or an SF_ERR_* code; sf_last_error() gives text.
 *    Input checks happen before any launch (the reference raises before any
 *    work, sparse_splat.py:114-122).
 */
#ifndef SPLATFIELD_B200_H
#define SPLATFIELD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SF_OK 0
#define SF_ERR_VALIDATION 1   /* -> splatfield.errors.ValidationError */
#define SF_ERR_RESOURCE 2     /* -> splatfield.errors.ResourceLimitError */
#define SF_ERR_CUDA 3         /* -> splatfield.errors.SplatfieldError */
#define SF_ERR_WORKSPACE 4    /* workspace smaller than sf_*_workspace_bytes */

#define SF_TILE 16            /* projection.py:31 DEFAULT_TILE_SIZE; kernels are specialised */

/* Pinhole camera, projection.py:37-65 (Camera).  R row-major world->camera. */
typedef struct SfCamera {
    double R[9];
    double t[3];
    double fx, fy, cx, cy;
    double near_plane;
    int32_t width, height;
} SfCamera;

/* Device-resident scene, core.py:256-279 (Scene, struct of arrays).
 * Rows MUST be ordered by ascending id: the canonical (depth, id) order of
 * projection.py:396 then needs only a stable sort on depth. */
typedef struct SfScene {
    int64_t num_gaussians;
    int32_t num_levels, L, K, D;
    const float* positions;        /* (G,3) */
    const float* rotations;        /* (G,4) w,x,y,z */
    const float* scales;           /* (G,3) */
    const float* opacities;        /* (G,) */
    const uint16_t* coeff_indices; /* (num_levels,G,K) */
    const float* coeff_values;     /* (num_levels,G,K) */
    const int64_t* ids;            /* (G,) ascending */
    const float* codebooks;        /* (num_levels,L,D) row-major */
} SfScene;

/* One text query, query.py:22-37 + the canonical set, query.py:65-84. */
typedef struct SfQuery {
    const double* vector;      /* (D,) */
    const double* canonicals;  /* (n_canonicals,D) */
    int32_t n_canonicals;
    int32_t window;            /* mean_filter window, odd >= 1 (query.py:89-90) */
    int32_t fixed_level;       /* -1 = select_level (query.py:111-118) else block index */
    double threshold;          /* segment threshold (query.py:136) */
} SfQuery;

/* What one frame computes and where it goes.  NULL outputs are skipped. */
typedef struct SfFrame {
    const int32_t* host_levels; /* HOST (n_levels,) semantic levels to splat, sparse_splat.py:103-120 */
    int32_t n_levels;
    int32_t early_exit;         /* rasterizer.py:174-177 */
    int64_t pair_capacity;      /* size of the (tile, rank) pair buffer in the workspace */
    /* outputs */
    float* coeff_map;           /* (H,W,n_levels*L) fp32      CoefficientMap.data (may be NULL;
                                   required with features unless sf_decode_fused) */
    float* final_t;             /* (H,W) fp32                 RenderStats.final_transmittance */
    float* features;            /* (n_levels,H,W,D) fp32      FeatureMapSet.maps */
    double* relevancy_raw;      /* (n_levels,H,W) fp64        relevancy_map() per level */
    double* relevancy_filtered; /* (n_levels,H,W) fp64        mean_filter() per level */
    uint8_t* mask;              /* (H,W) u8                   segment(chosen).mask */
    int64_t* stats_i64;         /* (16,) see SF_STAT_* */
    double* stats_f64;          /* (8 + 2*n_levels,) see SF_STATF_* */
    /* optional cudaEvent_t recorded at: frame start, after blend (render),
     * after decode, after post -- the StageTimings of sparse_splat.py:202-215 --
     * and [4] right before the blend launch (so [4] -> [1] times the blend
     * kernel, which includes the decode when sf_decode_fused) */
    void* events[5];
    /* optional cached per-row scatter plan of host_levels (sf_pack_channels);
     * NULL = built inside the frame */
    const unsigned char* chan_by_row;
    /* Tile-band mode: pixel rows [band_y0, band_y1)
     * are owned by this call; both 0 = the whole image.  The frame renders the
     * tile rows covering the owned rows plus the mean-filter halo (window/2
     * rows each side, clipped to the image) -- every rendered tile is
     * identical to the full-frame one -- decodes and filters only those rows,
     * and reduces select/localize/segment statistics over the owned rows
     * (SF_STAT_LEVEL_ARGMAX / SF_STATF_LEVEL_MIN / LEVEL_MAX per level) for a
     * cross-rank max-all-reduce; sf_mask_rows then applies the global
     * normalisation.  Output buffers stay full-image sized; rows outside the
     * rendered / owned range are not written. */
    int32_t band_y0;
    int32_t band_y1;
    /* optional cached codebook image of host_levels for the fused decode
     * (sf_pack_decode_image); NULL = built inside the frame */
    const void* dec_image;
    /* Training backward (train.py:324-330): when grad_coeff_map (dL/dW,
     * (H,W,n_levels*L) fp32) is set, the frame runs the transpose of the splat
     * instead of the blend -- grad_values (n_levels, G, K) fp32 (zero it first)
     * receives sum_p e(p) dL/dW[p][channel] for every Gaussian's K entries per
     * level -- and nothing after it. */
    const float* grad_coeff_map;
    float* grad_values;
    /* 1: blend with the projection and tile lists the previous frame of this
     * workspace built (same scene, camera, image and shape; no SfQuery; a
     * chan_by_row plan is required) -- render_dense's channel passes and the
     * training backward reuse the forward frame's binning.  0: full frame. */
    int32_t reuse_lists;
} SfFrame;

/* stats_i64 slots */
#define SF_STAT_VISIBLE 0     /* ProjectedScene.count */
#define SF_STAT_PAIRS 1       /* RenderStats.pairs_blended (sum of tile list lengths) */
#define SF_STAT_OVERFLOW 2    /* 1 if pairs > pair_capacity: grow and re-run */
#define SF_STAT_LEVEL 3       /* chosen level block index */
#define SF_STAT_ROW 4         /* localize() row */
#define SF_STAT_COL 5         /* localize() col */
#define SF_STAT_DEGENERATE 6  /* segment().degenerate */
#define SF_STAT_FIXUPS 7      /* pixels replayed exactly in fp64 (ambiguous early exit) */
#define SF_STAT_LEVEL_ARGMAX 8 /* + b: first row-major argmax (flat, whole image) of block b over the owned rows */
/* stats_f64 slots */
#define SF_STATF_MIN 0        /* chosen map min */
#define SF_STATF_MAX 1        /* chosen map max */
#define SF_STATF_LEVEL_MAX 8  /* + b: max of filtered map of block b (owned rows) */
/* stats_f64[8 + n_levels + b]: min of filtered map of block b (owned rows) */

/* Per-row scatter plan (channel ids level*L+idx and values of the selected
 * levels, sparse_splat.py:126-132) -- a scene constant worth caching. */
size_t sf_channel_plan_bytes(int64_t num_gaussians, int32_t n_levels, int32_t K);
int sf_pack_channels(const SfScene* scene, const int32_t* host_levels, int32_t n_levels, void* out,
                     size_t out_bytes, void* stream);

/* The fused decode's codebook image of host_levels (pre-swizzled fp16 hi/lo
 * tiles + per-level scales) -- a scene constant worth caching; 0 bytes when
 * sf_decode_fused is false for the shape. */
size_t sf_decode_image_bytes(int32_t n_levels, int32_t L, int32_t K, int32_t D);
int sf_pack_decode_image(const SfScene* scene, const int32_t* host_levels, int32_t n_levels, void* out,
                         size_t out_bytes, void* stream);

/* Capacity of the exact fp64 replay list (k_blend_fixup_cta) of a W x H
 * frame: every pixel at most once, so W * H unless lowered for tests by
 * SF_FIXUP_CAPACITY.  A frame whose stats_i64[SF_STAT_FIXUPS] exceeds it left
 * pixels uncertified; the host shim raises (it never happens at W * H). */
int64_t sf_fixup_capacity(int32_t width, int32_t height);

/* Scratch needed by sf_render_frame for this scene/frame shape. */
int sf_frame_workspace_bytes(int64_t num_gaussians, int32_t width, int32_t height,
                             int32_t n_levels, int32_t L, int32_t K, int32_t D,
                             int64_t pair_capacity, size_t* bytes);

/*
 * One full frame: preprocess -> depth-rank sort -> tile binning -> blend
 * (+ fused projected-codebook relevancy) -> codebook GEMM -> mean filter ->
 * select_level / localize / segment.
 * Replaces, end to end, splat_multilevel (sparse_splat.py:178-180) +
 * decode (:183-199) + query_pipeline (:243-297) + segment (query.py:136-145).
 * query may be NULL (pure feature splatting).
 */
int sf_render_frame(const SfScene* scene, const SfCamera* cam, const SfQuery* query,
                    const SfFrame* frame, void* workspace, size_t workspace_bytes, void* stream);

/*
 * sf_render_frame with its first half -- projection, depth sort, tile
 * binning and the per-frame codebook products -- on stream_prepare, and the
 * rest -- blend (+ fused decode), filter, selection -- on stream_render,
 * ordered by handoff_event (a cudaEvent_t from sf_event_create).  With two
 * workspaces and output sets a caller can prepare frame i+1 (e.g. on a
 * higher-priority stream) while frame i blends; it must not reuse a
 * workspace before the frame that used it has finished on stream_render.
 */
int sf_render_frame_split(const SfScene* scene, const SfCamera* cam, const SfQuery* query,
                          const SfFrame* frame, void* workspace, size_t workspace_bytes,
                          void* stream_prepare, void* stream_render, void* handoff_event);

/*
 * The per-tile lists of the last frame rendered with `workspace` (same shape
 * arguments as sf_frame_workspace_bytes): tile_offsets (n_tiles+1) u32 and
 * tile_rows (pairs) u32 scene rows in canonical (depth, id) order per tile --
 * TileBinning.tile_lists (projection.py:342-376) of the frame itself, for
 * parity checks of the frame path's binning.  Synchronises `stream`.
 */
int sf_frame_tile_lists(int64_t num_gaussians, int32_t width, int32_t height, int32_t n_levels, int32_t L,
                        int32_t K, int32_t D, int64_t pair_capacity, const void* workspace,
                        size_t workspace_bytes, uint32_t* tile_offsets, uint32_t* tile_rows, int64_t max_pairs,
                        void* stream);

/*
 * A sweep of text prompts over one frame (BASELINE config E): the
 * coefficient map is rendered once (frame->coeff_map required; frame must
 * carry no features), then every prompt gets the query_pipeline post --
 * relevancy from the map through the projected codebook (fp64), mean filter,
 * select_level / localize / segment with an automatic level.  The map is
 * read once per 65 - n_canonicals prompts; frame->relevancy_raw is the
 * (n_prompts, n_levels, H, W) fp64 raw-relevancy buffer.
 *   prompts (n_prompts, D) fp64; relevancy_filtered (n_prompts, n_levels, H, W)
 *   fp64; masks (n_prompts, H, W) u8; stats_i64 (n_prompts, 16) and stats_f64
 *   (n_prompts, 8 + 2 n_levels) laid out like SfFrame's.
 */
int sf_query_sweep(const SfScene* scene, const SfCamera* cam, const SfFrame* frame, const double* prompts,
                   int32_t n_prompts, const double* canonicals, int32_t n_canonicals, int32_t window,
                   double threshold, double* relevancy_filtered, uint8_t* masks, int64_t* stats_i64,
                   double* stats_f64, void* workspace, size_t workspace_bytes, void* stream);

/*
 * project_scene, projection.py:240-315: the same surviving set, in scene-row
 * order, with bitwise-identical fp64 values.  Outputs sized for G rows;
 * *count_out (device int64) receives N.  inv_covs is (N,2,2).
 */
int sf_project_workspace_bytes(int64_t num_gaussians, size_t* bytes);
int sf_project(const SfScene* scene, const SfCamera* cam, double* means2d, double* inv_covs,
               double* depths, double* opacities, int64_t* source_ids, int64_t* rows,
               int64_t* count_out, void* workspace, size_t workspace_bytes, void* stream);
/* Same, for a device scene whose rows were permuted into id order at upload:
 * orig_rows[g] is the caller's row of device row g (output keeps caller order). */
int sf_project_rows(const SfScene* scene, const SfCamera* cam, const int64_t* orig_rows,
                    double* means2d, double* inv_covs, double* depths, double* opacities,
                    int64_t* source_ids, int64_t* rows, int64_t* count_out, void* workspace,
                    size_t workspace_bytes, void* stream);

/*
 * bin_projected, projection.py:379-450, on arbitrary projected arrays
 * (N rows; inv_covs (N,2,2)).  Produces the canonical (depth, id) order
 * (order[k] = input row of canonical rank k) and CSR per-tile lists of
 * canonical ranks, byte-identical to the reference's tile_lists.
 * tile_offsets has n_tiles+1 entries; *stats_i64 gets SF_STAT_PAIRS/OVERFLOW.
 */
int sf_bin_workspace_bytes(int64_t n, int32_t width, int32_t height, int64_t pair_capacity,
                           size_t* bytes);
int sf_bin(int64_t n, const double* means2d, const double* inv_covs, const double* depths,
           const int64_t* source_ids, int32_t width, int32_t height, int64_t pair_capacity,
           int64_t* order, int64_t* tile_offsets, int32_t* tile_entries, int64_t* stats_i64,
           void* workspace, size_t workspace_bytes, void* stream);

/* decode, sparse_splat.py:183-199: one level block, (P,L) @ (L,D) -> (P,D) fp32,
 * 3xTF32 on tcgen05 tensor cores (L in {32,64}, D % 256 == 0; other shapes
 * use the SIMT kernel).  w has row stride w_stride floats. */
size_t sf_decode_workspace_bytes(int32_t L, int32_t D);
int sf_decode(int64_t n_pixels, int32_t L, int32_t D, const float* w, int64_t w_stride,
              const float* codebook, float* out, void* workspace, size_t workspace_bytes,
              void* stream);
/* Plain fp32 FMA-chain decode on CUDA cores: the independent cross-check the
 * parity tests hold the tensor-core kernel against (not used by any frame). */
int sf_decode_simt(int64_t n_pixels, int32_t L, int32_t D, const float* w, int64_t w_stride,
                   const float* codebook, float* out, void* stream);

/* relevancy_map, query.py:65-84, on an (P,D) feature map (fp32 or fp64). */
int sf_relevancy_f32(int64_t n_pixels, int32_t D, const float* feats, const double* q,
                     const double* canonicals, int32_t n_canonicals, double* out, void* stream);
int sf_relevancy_f64(int64_t n_pixels, int32_t D, const double* feats, const double* q,
                     const double* canonicals, int32_t n_canonicals, double* out, void* stream);

/* mean_filter, query.py:87-108 (edge-clamped box filter), fp64 (H,W). */
int sf_mean_filter(int32_t height, int32_t width, const double* in, int32_t window, double* out,
                   void* workspace, size_t workspace_bytes, void* stream);

/* select_level / localize / segment, query.py:111-145 over n (1..32) maps (H,W) fp64:
 * stats_i64[SF_STAT_LEVEL/ROW/COL/DEGENERATE], stats_f64[MIN/MAX/LEVEL_MAX+b];
 * stats_i64 needs max(16, 8 + n) entries and stats_f64 8 + 2 n (per-map argmax / max / min);
 * mask may be NULL.  fixed_level >= 0 skips selection. */
size_t sf_select_segment_workspace_bytes(int32_t n_maps, int32_t height, int32_t width);
int sf_select_segment(int32_t n_maps, int32_t height, int32_t width, const double* maps,
                      int32_t fixed_level, double threshold, uint8_t* mask, int64_t* stats_i64,
                      double* stats_f64, void* workspace, size_t workspace_bytes, void* stream);
/* segment().mask rows [y0, y1) of map `level` of (n_maps,H,W) fp64 maps with
 * the given (global) min/max: mask = (m - lo)/(hi - lo) > threshold, all zero
 * when hi <= lo (query.py:136-145).  The band-mode step after the cross-rank
 * reduction of the per-band statistics. */
int sf_mask_rows(const double* maps, int32_t height, int32_t width, int32_t level, double lo, double hi,
                 double threshold, int32_t y0, int32_t y1, uint8_t* mask, void* stream);

/* Timing-event helpers for SfFrame.events (cudaEventCreate / elapsed ms). */
void* sf_event_create(void);
void sf_event_destroy(void* ev);
float sf_event_elapsed_ms(void* start, void* end);

/* Human-readable text of the last error on this thread. */
const char* sf_last_error(void);
/* ABI version (bumped on any signature change). */
/*
 * LSV2 scene records (io.py:7-11, 42-124) -> SoA on the device, with the
 * checks of Scene.validate (core.py:285-331) OR-ed into *flags (device u32,
 * zero it first): the file is read once into pinned host memory and copied
 * raw to the device; one thread per record de-interleaves it.  coeff_indices /
 * coeff_values are [levels][G][K].  The codebook tail is already SoA (copy it).
 */
#define SF_LSV2_NONFINITE 1u
#define SF_LSV2_QUATERNION 2u
#define SF_LSV2_SCALE 4u
#define SF_LSV2_OPACITY 8u
#define SF_LSV2_INDEX_RANGE 16u
#define SF_LSV2_INDEX_ORDER 32u
#define SF_LSV2_VALUE_SIGN 64u
#define SF_LSV2_VALUE_SUM 128u
int sf_lsv2_unpack(const void* records, int64_t num_gaussians, int32_t num_levels, int32_t K, int32_t L,
                   float* positions, float* rotations, float* scales, float* opacities, float* colors,
                   uint16_t* coeff_indices, float* coeff_values, uint32_t* flags, void* stream);

int sf_abi_version(void); /* 2: SfFrame band fields; 3: fused decode (coeff_map optional with features); 4: SfFrame.reuse_lists, training entry points */

/* 1 if sf_render_frame decodes features inside the blend kernel for this
 * shape (then SfFrame.coeff_map may be NULL when features are requested);
 * 0 if the decode runs as a separate tcgen05 GEMM over the coefficient map. */
int sf_decode_fused(int32_t n_levels, int32_t L, int32_t K, int32_t D);

/* 1 if a query frame of this shape computes the relevancy inside the blend
 * kernel; 0 if from the coefficient map in HBM (then SfFrame.coeff_map is
 * required with an SfQuery).  Replaces the relevancy_map call of
 * query_pipeline (splatfield/sparse_splat.py:281-283, query.py:65-84). */
int sf_relevancy_fused(int32_t n_levels, int32_t L, int32_t K, int32_t n_canon);

/* ---- training step (splatfield/train.py; kernels in csrc/sf_train.cu) ----
 * Parameters live in HBM in device row order: logits (levels, G, L) fp64,
 * codebooks (levels, L, D) fp64.  All sums run in a fixed order. */

/* softmax -> top-K -> renormalise per (row, level) into the scatter plan
 * (sf_channel_plan_bytes bytes); replaces normalize_batch (train.py:131-139). */
int sf_train_plan(int64_t G, int32_t levels, int32_t L, int32_t K, const double* logits, void* plan, void* stream);
/* loss partial blocks per level of a frame of HW pixels; codebook-gradient splits */
int64_t sf_train_loss_blocks(int64_t HW);
int32_t sf_train_cb_splits(void);
/* F = W atoms, r = (F - T) mask, loss partials (levels * blocks, 2) = (sum r^2,
 * sum (1 - cos) mask), dF = 2 scale r + cos_w scale dcos, dW = dF atoms^T
 * (forward_loss train.py:201-279, backward train.py:303-329).  wmap / dW:
 * (HW, levels L) fp32; targets / dF: (levels, HW, D) fp64; mask (HW) fp64 or
 * NULL; pix_stats (levels, HW, 3) fp64, required when cos_w != 0. */
int sf_train_residual(int64_t HW, int32_t levels, int32_t L, int32_t D, const float* wmap, const double* atoms,
                      const double* targets, const double* mask, double scale, double cos_w, double* pix_stats,
                      double* dF, float* dW, double* loss_part, void* stream);
/* dL/datoms = W^T dF (train.py:321); part: sf_train_cb_splits x levels x L x D */
int sf_train_cbgrad(int64_t HW, int32_t levels, int32_t L, int32_t D, const float* wmap, const double* dF,
                    double* part, double* grad_cb, void* stream);
int64_t sf_train_logit_blocks(int64_t G, int32_t levels);
int64_t sf_train_adam_blocks(int64_t n);
/* top-K softmax backward from ghat (levels, G, K) fp32 (the transpose splat's
 * output, SfFrame.grad_values); grad_out (levels, G, L) or NULL; with t > 0
 * and m, v: Adam step t on the logits in place (train.py:79-107, 331-340).
 * norm_part: sf_train_logit_blocks squared-gradient partials. */
int sf_train_logits(int64_t G, int32_t levels, int32_t L, int32_t K, double* logits, const float* ghat,
                    double* grad_out, double* m, double* v, double lr, double beta1, double beta2, double eps,
                    int64_t t, double* norm_part, void* stream);
/* Adam step t on n parameters (t = 0: only the squared-gradient partials) */
int sf_train_adam(int64_t n, double* param, const double* grad, double* m, double* v, double lr, double beta1,
                  double beta2, double eps, int64_t t, double* norm_part, void* stream);
/* out[j] = sum_i part[i * stride + j] in order, j < width */
int sf_train_reduce(int64_t n, int32_t stride, int32_t width, const double* part, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPLATFIELD_B200_H */
