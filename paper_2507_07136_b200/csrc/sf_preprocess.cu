// sf_preprocess.cu -- K1: per-Gaussian EWA projection, culling and depth keys.
//
// Restates project_arrays (projection.py:240-308) and batch_covariances
// (core.py:193-209) in fp64 with the reference's exact operation order: the
// numpy matmul sites (pos @ R.T, m @ m.T, jw @ cov @ jw.T) are evaluated by
// OpenBLAS as the FMA chain fma(a2,b2, fma(a1,b1, a0*b0)), reproduced with
// explicit fma(); everything else is an IEEE op in source order.  This file
// is compiled with -fmad=false so nvcc cannot contract anything else, which
// makes means2d / inv_covs / depths bitwise equal to the reference.
//
// HBM layout: one thread per scene row (rows ordered by id).  Reads 44 B of
// geometry per Gaussian (pos 12 + quat 16 + scale 12 + opacity 4), writes the
// row's 80 B blend record (GeomRec: fp32 rejection inputs + the fp64
// projected values), an 8 B depth key and a 4 B row index.
#include <cub/cub.cuh>

#include "sf_common.cuh"

namespace sf {

#ifndef SF_PRE_MINB
#define SF_PRE_MINB 5
#endif
__global__ void __launch_bounds__(256, SF_PRE_MINB) k_preprocess(SfScene s, SfCamera cam, GeomRec* __restrict__ geom,
                                                    uint64_t* __restrict__ keys,
                                                    uint32_t* __restrict__ vals,
                                                    unsigned long long* __restrict__ n_visible) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool vis = false;
    if (g < s.num_gaussians) {
        const double* R = cam.R;
        double p0 = s.positions[3 * g], p1 = s.positions[3 * g + 1], p2 = s.positions[3 * g + 2];
        double cp[3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
            cp[r] = fma(p2, R[3 * r + 2], fma(p1, R[3 * r + 1], p0 * R[3 * r])) + cam.t[r];
        double x = cp[0], y = cp[1], z = cp[2];
        if (z > cam.near_plane) {
            double m0 = (cam.fx * x) / z + cam.cx;
            double m1 = (cam.fy * y) / z + cam.cy;
            const float4 q4 = reinterpret_cast<const float4*>(s.rotations)[g];
            double w = q4.x, qx = q4.y, qy = q4.z, qz = q4.w;
            double rot[9];
            rot[0] = 1 - 2 * (qy * qy + qz * qz);
            rot[1] = 2 * (qx * qy - w * qz);
            rot[2] = 2 * (qx * qz + w * qy);
            rot[3] = 2 * (qx * qy + w * qz);
            rot[4] = 1 - 2 * (qx * qx + qz * qz);
            rot[5] = 2 * (qy * qz - w * qx);
            rot[6] = 2 * (qx * qz - w * qy);
            rot[7] = 2 * (qy * qz + w * qx);
            rot[8] = 1 - 2 * (qx * qx + qy * qy);
            double sc[3] = {s.scales[3 * g], s.scales[3 * g + 1], s.scales[3 * g + 2]};
            double m[9];
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) m[3 * r + c] = rot[3 * r + c] * sc[c];
            double cov[9];
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    cov[3 * r + c] = fma(m[3 * r + 2], m[3 * c + 2],
                                         fma(m[3 * r + 1], m[3 * c + 1], m[3 * r] * m[3 * c]));
            double cs[9];
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) cs[3 * r + c] = (cov[3 * r + c] + cov[3 * c + r]) * 0.5;
            double fxz = cam.fx / z, fyz = cam.fy / z;
            double gx = (cam.fx * x) / (z * z), gy = (cam.fy * y) / (z * z);
            double jw[6];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                jw[k] = fxz * R[k] - gx * R[6 + k];
                jw[3 + k] = fyz * R[3 + k] - gy * R[6 + k];
            }
            double tmp[6];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    tmp[3 * r + c] = fma(jw[3 * r + 2], cs[6 + c],
                                         fma(jw[3 * r + 1], cs[3 + c], jw[3 * r] * cs[c]));
            double c2[4];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    c2[2 * r + c] = fma(tmp[3 * r + 2], jw[3 * c + 2],
                                        fma(tmp[3 * r + 1], jw[3 * c + 1], tmp[3 * r] * jw[3 * c]));
            c2[0] += SF_LOWPASS;
            c2[3] += SF_LOWPASS;
            double det = c2[0] * c2[3] - c2[1] * c2[2];
            bool ok = isfinite(det) && (det > 0) && isfinite(m0) && isfinite(m1);
            if (ok) {
                double i00 = c2[3] / det, i11 = c2[0] / det, off = -c2[1] / det;
                double qmin = min_mahal_sq_to_rect(m0, m1, i00, off, i11, 0.0, 0.0,
                                                   (double)(cam.width - 1), (double)(cam.height - 1));
                if (qmin <= SF_CUTOFF) {
                    vis = true;
                    // blend record of this row: fp32 rejection inputs + the fp64 values
                    GeomRec q;
                    q.mx = m0;
                    q.my = m1;
                    q.a64 = i00;
                    q.b64 = off;
                    q.c64 = i11;
                    geom_fill_f32(q);
                    q.opacity = s.opacities[g];
                    q.row = (uint32_t)g;
                    q.pad = 0;
                    geom[g] = q;
                    keys[g] = (uint64_t)__double_as_longlong(z);  // z > near > 0: bits are monotone
                }
            }
        }
        if (!vis) keys[g] = ~0ull;  // culled rows sort after every visible one
        vals[g] = (uint32_t)g;
    }
    unsigned ballot = __ballot_sync(0xffffffffu, vis);
    if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(n_visible, (unsigned long long)__popc(ballot));
}

void launch_preprocess(const SfScene& s, const SfCamera& cam, GeomRec* geom, uint64_t* keys,
                       uint32_t* vals, int64_t* stats, cudaStream_t st) {
    if (s.num_gaussians == 0) return;
    int blocks = ceil_div(s.num_gaussians, 256);
    k_preprocess<<<blocks, 256, 0, st>>>(s, cam, geom, keys, vals,
                                         (unsigned long long*)(stats + SF_STAT_VISIBLE));
}

// ---- project_scene API path: compaction in original scene-row order ----

__global__ void k_flags(int64_t G, const uint64_t* keys, const int64_t* orig_rows, int32_t* flags) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    int64_t r = orig_rows ? orig_rows[g] : g;
    flags[r] = keys[g] != ~0ull;
}

__global__ void k_compact(SfScene s, const GeomRec* geom, const uint64_t* keys,
                          const int64_t* orig_rows, const int32_t* flags, const int32_t* scan,
                          double* means2d, double* inv_covs, double* depths, double* opac,
                          int64_t* source_ids, int64_t* rows, int64_t* count) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t G = s.num_gaussians;
    if (g >= G) return;
    int64_t r = orig_rows ? orig_rows[g] : g;
    if (r == G - 1) *count = (int64_t)scan[r] + flags[r];
    if (keys[g] == ~0ull) return;
    int64_t o = scan[r];
    Proj64 p = geom_proj(geom[g]);
    means2d[2 * o] = p.mx;
    means2d[2 * o + 1] = p.my;
    inv_covs[4 * o] = p.a;
    inv_covs[4 * o + 1] = p.b;
    inv_covs[4 * o + 2] = p.b;
    inv_covs[4 * o + 3] = p.c;
    depths[o] = __longlong_as_double((long long)keys[g]);
    opac[o] = (double)s.opacities[g];
    source_ids[o] = s.ids[g];
    rows[o] = r;
}

size_t project_compact_cub_bytes(int64_t G) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int32_t*)nullptr, (int32_t*)nullptr, (int)G);
    return bytes;
}

void launch_project_compact(const SfScene& s, const GeomRec* geom, const uint64_t* keys,
                            const int64_t* orig_rows, int32_t* flags, int32_t* scan,
                            double* means2d, double* inv_covs, double* depths, double* opac,
                            int64_t* source_ids, int64_t* rows, int64_t* count, void* cub_tmp,
                            size_t cub_bytes, cudaStream_t st) {
    int64_t G = s.num_gaussians;
    if (G == 0) {
        cudaMemsetAsync(count, 0, sizeof(int64_t), st);
        return;
    }
    int blocks = ceil_div(G, 256);
    k_flags<<<blocks, 256, 0, st>>>(G, keys, orig_rows, flags);
    cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, flags, scan, (int)G, st);
    k_compact<<<blocks, 256, 0, st>>>(s, geom, keys, orig_rows, flags, scan, means2d, inv_covs,
                                      depths, opac, source_ids, rows, count);
}

}  // namespace sf
