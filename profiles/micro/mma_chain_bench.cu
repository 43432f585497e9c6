// Microbenchmark (development aid): tcgen05.mma kind::f16 M=128, K=16 throughput
// on one SM as a function of N, the A source (TMEM / SMEM) and the number of
// independent accumulators the issue order rotates through (1 = every MMA
// depends on the previous one).  Issue is one thread, fully unrolled (no
// per-MMA warp sync).  Optional background load: 4 warps streaming
// tcgen05.ld (like the fused decode's drains).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_chain_bench mma_chain_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
#define X32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"
#define O32(v) "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),"=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])

template <bool ATMEM, int NACC>
__device__ __forceinline__ void issue(uint32_t tm, uint64_t ad, uint64_t bd, uint32_t idesc, int n, int i) {
    const uint32_t d = tm + 256 + (uint32_t)((i % NACC) * (256 / NACC));
    if (ATMEM)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                     "r"(tm + (uint32_t)(8 * (i & 3))), "l"(bd + 2 * (i & 3)), "r"(idesc), "r"(1)
                     : "memory");
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                     "l"(ad + 2 * (i & 3)), "l"(bd + 2 * (i & 3)), "r"(idesc), "r"(1)
                     : "memory");
}

template <bool ATMEM, int NACC>
__global__ void k(int iters, int N, int bg, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];  // B: [0, 32 KB), A: [32 KB, 48 KB)
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        stop = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (warp == 0) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t bd = desc(sa(sm));
        const uint64_t ad = desc(sa(sm + 32768));
        long long t0 = clock64();
        if (lane == 0) {
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) issue<ATMEM, NACC>(tm, ad, bd, idesc, N, i + u);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
        }
        __syncwarp();
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sa(&bar)) : "memory");
        long long t1 = clock64();
        if (lane == 0) {
            out[0] = (unsigned long long)(t1 - t0);
            stop = 1;
        }
    } else if (bg == 2 && warp >= 1) {
        // background: shared-memory load/store traffic (like the blend warps'), on [48 KB, 64 KB)
        uint32_t a = sa(sm + 48 * 1024) + (uint32_t)((threadIdx.x * 16) & 16383);
        uint32_t x = threadIdx.x, acc = 0;
        for (int i = 0; !stop; ++i) {
            uint32_t v0, v1, v2, v3;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(a));
            acc += v0 ^ v3;
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a ^ 512u), "r"(x), "r"(acc), "r"(v1), "r"(v2));
            a = sa(sm + 48 * 1024) + (uint32_t)(((threadIdx.x + i * 37) * 16) & 16383);
        }
        if (acc == 12345) out[1] = acc;
    } else if (bg == 1 && warp >= 1 && warp <= 4) {
        // background: TMEM reads of the accumulator area's lane quarter (like the drains)
        uint32_t v[32], acc = 0;
        const int q = warp - 1;
        for (int i = 0; !stop; ++i) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " X32 ", [%32];" : O32(v) : "r"(tm + ((uint32_t)(q * 32) << 16) + (uint32_t)(256 + ((i * 32) & 255))));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc += v[i & 31];
        }
        if (acc == 12345) out[1] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

template <bool ATMEM, int NACC>
void run(int N, int bg, unsigned long long* d) {
    const int iters = 2048;
    unsigned long long h[2];
    cudaFuncSetAttribute(k<ATMEM, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<ATMEM, NACC><<<1, bg == 2 ? 512 : 160, 64 * 1024>>>(iters, N, bg, d);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("N=%3d A=%s acc=%d bg=%d: %6.1f cyc/mma (floor %d)\n", N, ATMEM ? "TMEM" : "SMEM", NACC, bg,
           (double)h[0] / iters, 128 * N / 256);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    for (int bg : {0, 1, 2})
        for (int N : {64, 128, 256}) {
            run<true, 1>(N, bg, d);
            if (N <= 128) run<true, 2>(N, bg, d);
            if (N <= 64) run<true, 4>(N, bg, d);
            run<false, 1>(N, bg, d);
            if (N <= 128) run<false, 2>(N, bg, d);
        }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
