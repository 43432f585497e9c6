// Microbenchmark (development aid): the blend's per-member scatter RMW of 4
// channels (the same channel column for all 32 pixels of a warp, random per
// member) into an fp32 accumulator held in shared memory (acc[ch][px], pitch
// 129, as k_blend) vs in TMEM (lane = pixel, column = channel; tcgen05.ld /
// add / tcgen05.st per member).  4 warps (128 pixels) per CTA, 1-4 CTAs per
// SM; prints cycles per member per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scatter_bench scatter_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kMembers = 2048, kCh = 64, kPitch = 129;

__global__ void __launch_bounds__(128) k(int mode, const uint32_t* __restrict__ chans, unsigned long long* out,
                                         float* sink) {
    extern __shared__ __align__(16) float acc[];  // [kCh][kPitch] (mode 0)
    __shared__ uint32_t tbase;
    __shared__ __align__(16) uint32_t ch[kMembers * 4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, slot = threadIdx.x;
    for (int i = threadIdx.x; i < kMembers * 4; i += blockDim.x) ch[i] = chans[i];
    for (int i = threadIdx.x; i < kCh * kPitch; i += blockDim.x) acc[i] = 0.f;
    if (mode == 1 && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase + ((uint32_t)(warp * 32) << 16);
    const float e = 0.001f * (lane + 1);
    long long t0 = clock64();
    if (mode == 0) {
        for (int m = 0; m < kMembers; ++m) {
            const uint4 c = *reinterpret_cast<const uint4*>(&ch[4 * m]);
            const uint32_t cc[4] = {c.x, c.y, c.z, c.w};
            float v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = acc[cc[k] * kPitch + slot];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = fmaf(e, 0.5f + k, v[k]);
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[cc[k] * kPitch + slot] = v[k];
        }
    } else {
        if (warp == 0) {
        }
        for (int m = 0; m < kMembers; ++m) {
            const uint4 c = *reinterpret_cast<const uint4*>(&ch[4 * m]);
            const uint32_t cc[4] = {c.x, c.y, c.z, c.w};
            uint32_t v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v[k]) : "r"(tm + cc[k]));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = __float_as_uint(fmaf(e, 0.5f + k, __uint_as_float(v[k])));
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tm + cc[k]), "r"(v[k]) : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    long long t1 = clock64();
    float s = 0.f;
    if (mode == 0) {
        for (int c = 0; c < kCh; ++c) s += acc[c * kPitch + slot];
    } else {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + 5));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        s = __uint_as_float(v);
    }
    sink[blockIdx.x * 128 + threadIdx.x] = s;
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (mode == 1 && warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
    }
}

int main() {
    uint32_t h[kMembers * 4];
    uint32_t s = 12345;
    for (int m = 0; m < kMembers; ++m)
        for (int k = 0; k < 4; ++k) {
            s = s * 1664525u + 1013904223u;
            h[4 * m + k] = (uint32_t)(16 * k + (s >> 28));  // 4 distinct channels per member (one per 16-block)
        }
    uint32_t* d;
    unsigned long long* o;
    float* sink;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&o, 148 * 4 * sizeof(unsigned long long));
    cudaMalloc(&sink, 148 * 4 * 128 * sizeof(float));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    const int smem = kCh * kPitch * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 2; ++mode)
        for (int per_sm = 1; per_sm <= 4; per_sm *= 2) {
            const int grid = 148 * per_sm;
            k<<<grid, 128, smem>>>(mode, d, o, sink);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long r[148 * 4];
            cudaMemcpy(r, o, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < grid; ++i) avg += (double)r[i];
            avg /= grid;
            printf("%s  CTAs/SM %d: %.1f cycles per member per warp (%s)\n", mode ? "TMEM" : "SMEM", per_sm,
                   avg / kMembers, cudaGetErrorString(e));
        }
    return 0;
}
