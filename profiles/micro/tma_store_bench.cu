// TMA store-pattern microbenchmark (profiling aid for k_decode_tc's epilogue).
// 148 CTAs x 8 warps; each warp streams 4 KB SMEM boxes to a [P, 512] fp32
// buffer (3.36 GB) with one of several patterns; prints GB/s per pattern.
//   0: box {32 cols, 32 rows}, decode order (CTA = column quarter x tile group)
//   1: box {32 cols, 32 rows}, each warp walks the 4 column boxes of its rows back to back
//   2: 1-D bulk copies of 4 KB contiguous chunks (fill-like)
//   3: box {32 cols, 32 rows}, 2 KB-wide rows fully written by one warp (16 boxes) before moving on
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_store_bench.cu -o tma_store_bench
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NBUF>
__global__ void __launch_bounds__(256, 1) k_store(const __grid_constant__ CUtensorMap map, float* out, int64_t P,
                                                  int pattern) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float* buf = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* mine = buf + warp * NBUF * 1024;
    for (int i = lane; i < NBUF * 1024; i += 32) mine[i] = 1.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const int64_t n_rowblk = P / 32;  // 32-row blocks
    int n = 0;
    if (pattern == 0 || pattern == 1 || pattern == 3) {
        // work item = (row block, column box); 16 column boxes per row (512 cols)
        const int64_t items = n_rowblk * 16;
        const int64_t nw = (int64_t)gridDim.x * 8;
        const int64_t w = (int64_t)blockIdx.x * 8 + warp;
        for (int64_t it = w; it < items; it += nw) {
            int64_t rb, cb;
            if (pattern == 0) {  // decode-like: CTA c -> column quarter c % 4, warps split rows/boxes
                const int64_t per = items / nw;
                (void)per;
                const int q = blockIdx.x % 4;
                const int64_t g = blockIdx.x / 4, ng = gridDim.x / 4;
                const int64_t k = (it - w) / nw;  // iteration index
                const int64_t tile = g + (k / 2) * ng;  // 128-row tile
                rb = tile * 4 + (warp & 3);
                cb = q * 4 + (warp >> 2) + 2 * (k & 1);
                if (rb >= n_rowblk) break;
            } else if (pattern == 1) {
                rb = it / 4 % n_rowblk;
                cb = (it % 4) + 4 * ((it / 4) / n_rowblk);
            } else {
                rb = it / 16;
                cb = it % 16;
            }
            if (lane == 0) {
                if (n >= NBUF) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                        (uint64_t)&map),
                    "r"(su32(mine + (n % NBUF) * 1024)), "r"((int)(cb * 32)), "r"((int)(rb * 32))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++n;
        }
    } else {
        const int64_t chunks = P * 512 / 1024;  // 4 KB chunks
        const int64_t nw = (int64_t)gridDim.x * 8;
        for (int64_t c = (int64_t)blockIdx.x * 8 + warp; c < chunks; c += nw) {
            if (lane == 0) {
                if (n >= NBUF) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(out + c * 1024),
                             "r"(su32(mine + (n % NBUF) * 1024))
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++n;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const int64_t P = 1440 * 1080;
    float* out;
    cudaMalloc(&out, P * 512 * 4);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[2] = {512, (cuuint64_t)P};
    cuuint64_t strides[1] = {512 * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[4] = {"decode-like boxes", "4 boxes/row back to back", "1-D 4KB contiguous", "16 boxes/row (full rows)"};
    for (int nbuf : {2, 4}) {
        size_t smem = (size_t)8 * nbuf * 4096 + 1024;
        auto kern = nbuf == 2 ? k_store<2> : k_store<4>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int pat = 0; pat < 4; ++pat) {
            for (int w = 0; w < 2; ++w) kern<<<148, 256, smem>>>(map, out, P, pat);
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                cudaEventRecord(e0);
                kern<<<148, 256, smem>>>(map, out, P, pat);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("nbuf %d  %-28s %7.0f GB/s (%.3f ms)  %s\n", nbuf, names[pat], P * 512 * 4 / best / 1e6, best,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
