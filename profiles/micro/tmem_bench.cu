// Microbenchmark (development aid): TMEM read throughput (tcgen05.ld) and
// A-from-TMEM vs A-from-SMEM tcgen05.mma (kind::f16) issue rates on one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
#define X32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
#define O32(v) "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])

__global__ void k(int mode, int iters, int N, unsigned long long* out) {
    __shared__ __align__(1024) unsigned char sm[40 * 1024];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    long long t0 = clock64();
    if (mode == 0) {  // tcgen05.ld 32x32b.x32, every warp its lane quarter
        uint32_t v[32], acc = 0;
        for (int i = 0; i < iters; ++i) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " X32 ", [%32];" : O32(v) : "r"(tm + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((i * 32) & 511)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc += v[i & 31];
        }
        if (acc == 12345) out[1] = acc;
    } else if (warp == 0) {  // MMAs, N cols, A from TMEM (mode 1) or SMEM (mode 2), into D at col 256
        const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t bd = desc(sa(sm));
        const uint64_t ad = desc(sa(sm + 24576));
        for (int i = 0; i < iters; ++i) {
            if (lane == 0) {
                if ((mode & 3) == 1)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm + 256 + (uint32_t)((mode & 4) ? (i & 3) * 64 : 0)), "r"(tm + (uint32_t)(8 * (i & 3))), "l"(bd + 2 * (i & 3)), "r"(idesc), "r"(1) : "memory");
                else
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + 256 + (uint32_t)((mode & 4) ? (i & 3) * 64 : 0)), "l"(ad + 2 * (i & 3)), "l"(bd + 2 * (i & 3)), "r"(idesc), "r"(1) : "memory");
            }
            __syncwarp();
        }
        if (lane == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sa(&bar)) : "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    unsigned long long h[2];
    const int iters = 4096;
    for (int warps : {1, 4}) {
        k<<<1, 32 * warps>>>(0, iters, 64, d);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("tcgen05.ld 32x32b.x32 (4 KB/warp), %d warps: %.1f cyc/ld/warp -> %.1f B/clk per SM\n", warps,
               (double)h[0] / iters, 4096.0 * warps * iters / h[0]);
    }
    for (int mode : {1, 2, 5, 6})
        for (int N : {32, 64, 128, 256}) {
            if ((mode & 4) && N > 64) continue;
            k<<<1, 128>>>(mode, iters, N, d);
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            printf("mma kind::f16 M=128 N=%3d K=16, A from %s%s: %.1f cyc/mma (math floor %d)\n", N, (mode & 3) == 1 ? "TMEM" : "SMEM", (mode & 4) ? ", 4 rotating accumulators" : ", one accumulator",
                   (double)h[0] / iters, 128 * N / 256);
        }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
