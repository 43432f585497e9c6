// sf_decode.cu -- K7: codebook decode, (P, L) @ (L, D) per level.
//
// Reference: decode, sparse_splat.py:183-199 (fp64 BLAS dgemm per level).
// This file holds the SIMT fp32 kernel (exact fp32 FMA chain, used as the
// cross-check for the tensor-core kernel in sf_decode_tc.cu).
#include "sf_common.cuh"

namespace sf {

// One warp per pixel row chunk: lane owns 4 consecutive output columns.
// The coefficient row is broadcast through shared memory; the codebook is
// read as float4 (L2 resident: 128 KB per level).
__global__ void __launch_bounds__(256) k_decode_simt(int64_t P, int L, int D, const float* __restrict__ w,
                                                     int64_t w_stride, const float* __restrict__ cb,
                                                     float* __restrict__ out) {
    extern __shared__ float sw[];  // [8 rows][L]
    const int rows_per_block = 8;
    int64_t row0 = (int64_t)blockIdx.x * rows_per_block;
    for (int i = threadIdx.x; i < rows_per_block * L; i += blockDim.x) {
        int r = i / L, l = i % L;
        int64_t p = row0 + r;
        sw[i] = (p < P) ? w[p * w_stride + l] : 0.f;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t p = row0 + warp;
    if (p >= P) return;
    const float* wr = sw + warp * L;
    if (D % 4) {  // any D: one column per lane
        for (int d = lane; d < D; d += 32) {
            float acc = 0.f;
            for (int l = 0; l < L; ++l) acc = fmaf(wr[l], __ldg(cb + (size_t)l * D + d), acc);
            out[p * D + d] = acc;
        }
        return;
    }
    for (int d0 = lane * 4; d0 < D; d0 += 128) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int l = 0; l < L; ++l) {
            float wl = wr[l];
            float4 c = *reinterpret_cast<const float4*>(cb + (size_t)l * D + d0);
            acc.x = fmaf(wl, c.x, acc.x);
            acc.y = fmaf(wl, c.y, acc.y);
            acc.z = fmaf(wl, c.z, acc.z);
            acc.w = fmaf(wl, c.w, acc.w);
        }
        *reinterpret_cast<float4*>(out + p * D + d0) = acc;
    }
}

int launch_decode_simt(int64_t P, int L, int D, const float* w, int64_t w_stride, const float* cb,
                       float* out, cudaStream_t st) {
    if (P == 0) return 0;
    size_t smem = sizeof(float) * 8 * L;
    k_decode_simt<<<ceil_div(P, 8), 256, smem, st>>>(P, L, D, w, w_stride, cb, out);
    return 0;
}

}  // namespace sf
