// sf_io.cu -- LSV2 scene records -> device SoA, with the scene validation.
//
// Reference: io.py:7-11 (record layout), io.py:42-124 (save / load_scene) and
// Scene.validate (core.py:285-331).  The file's packed little-endian records
//     position f32x3 | quaternion f32x4 | scale f32x3 | opacity f32 |
//     color f32x3 | per level: K u16 indices, K f32 values
// arrive in HBM as raw bytes (one pinned-host read, one H2D copy); one thread
// per record de-interleaves them into the SoA arrays the frame kernels read
// and raises validation flags (atomicOr) instead of raising per record.
// Records are byte-packed (56 + 6 K per level bytes), so fields are
// assembled from 16-bit loads.
#include "sf_common.cuh"

namespace sf {

__device__ __forceinline__ uint32_t ld_u32(const uint8_t* p) {
    // 2-byte aligned (records are 56 + 6K per level bytes, 56 and 6K are even)
    const uint16_t* q = reinterpret_cast<const uint16_t*>(p);
    return (uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 16);
}
__device__ __forceinline__ float ld_f32(const uint8_t* p) { return __uint_as_float(ld_u32(p)); }

__global__ void __launch_bounds__(256) k_lsv2_unpack(const uint8_t* __restrict__ rec, int64_t G, int levels, int K,
                                                     int L, float* __restrict__ pos, float* __restrict__ rot,
                                                     float* __restrict__ scl, float* __restrict__ opa,
                                                     float* __restrict__ col, uint16_t* __restrict__ cidx,
                                                     float* __restrict__ cval, uint32_t* __restrict__ flags) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    const int64_t rs = 56 + (int64_t)levels * 6 * K;
    const uint8_t* r = rec + g * rs;
    uint32_t bad = 0;
    float v[14];
#pragma unroll
    for (int i = 0; i < 14; ++i) {
        v[i] = ld_f32(r + 4 * i);
        if (!isfinite(v[i])) bad |= SF_LSV2_NONFINITE;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) pos[g * 3 + i] = v[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) rot[g * 4 + i] = v[3 + i];
#pragma unroll
    for (int i = 0; i < 3; ++i) scl[g * 3 + i] = v[7 + i];
    opa[g] = v[10];
#pragma unroll
    for (int i = 0; i < 3; ++i) col[g * 3 + i] = v[11 + i];
    // core.py:317-323: |norm(q) - 1| <= 1e-6 (fp64 norm), scales > 0, opacity in [0, 1]
    double n2 = 0.0;  // numpy: sum of rounded squares, then sqrt
#pragma unroll
    for (int i = 3; i < 7; ++i) n2 = __dadd_rn(n2, __dmul_rn((double)v[i], (double)v[i]));
    if (fabs(sqrt(n2) - 1.0) > 1e-6) bad |= SF_LSV2_QUATERNION;
    if (!(v[7] > 0.f && v[8] > 0.f && v[9] > 0.f)) bad |= SF_LSV2_SCALE;
    if (v[10] < 0.f || v[10] > 1.f) bad |= SF_LSV2_OPACITY;
    const uint8_t* lp = r + 56;
    for (int b = 0; b < levels; ++b, lp += 6 * K) {
        double sum = 0.0;
        int prev = -1;
        for (int k = 0; k < K; ++k) {
            const int idx = __ldg(reinterpret_cast<const uint16_t*>(lp) + k);
            const float val = ld_f32(lp + 2 * K + 4 * k);
            cidx[((int64_t)b * G + g) * K + k] = (uint16_t)idx;
            cval[((int64_t)b * G + g) * K + k] = val;
            if (idx >= L) bad |= SF_LSV2_INDEX_RANGE;
            if (idx <= prev) bad |= SF_LSV2_INDEX_ORDER;
            prev = idx;
            if (!isfinite(val)) bad |= SF_LSV2_NONFINITE;
            if (val < 0.f) bad |= SF_LSV2_VALUE_SIGN;
            sum += (double)val;
        }
        if (fabs(sum - 1.0) > 1e-6) bad |= SF_LSV2_VALUE_SUM;
    }
    if (bad) atomicOr(flags, bad);
}

void launch_lsv2_unpack(const uint8_t* rec, int64_t G, int levels, int K, int L, float* pos, float* rot,
                        float* scl, float* opa, float* col, uint16_t* cidx, float* cval, uint32_t* flags,
                        cudaStream_t st) {
    if (G > 0)
        k_lsv2_unpack<<<ceil_div(G, 256), 256, 0, st>>>(rec, G, levels, K, L, pos, rot, scl, opa, col, cidx, cval,
                                                        flags);
}

}  // namespace sf
