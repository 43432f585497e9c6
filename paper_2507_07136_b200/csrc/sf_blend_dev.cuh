// sf_blend_dev.cuh -- device helpers shared by the blend kernels (k_blend,
// k_splat_tc): mbarrier / bulk-copy / tcgen05 / TMA wrappers and the fp32
// alpha evaluation with its fp64 guard band (rasterizer.py:161-168).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include "sf_common.cuh"

namespace sf {

// fp32 part of a GeomRec (its first 32 bytes): all the blend needs outside
// the guard band, where the fp64 fields are read from global memory
struct __align__(16) GeomF32 {
    float mx_hi, mx_lo, my_hi, my_lo;
    float a, k, d, opacity;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(b)),
        "r"(parity), "r"(0x989680)  // suspend-time hint: the thread sleeps in hardware until the phase flips
        : "memory");
}

__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
                 : "memory");
}
// 1-D bulk copy global -> shared, completion on an mbarrier (tx bytes)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(b))
        : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// K-major, 128B-swizzled operand: rows of 128 B, 8-row atoms 1024 B apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
// D (TMEM) [+]= A (TMEM, tf32, row = lane, K = column) x B (SMEM descriptor)
__device__ __forceinline__ void mma_tf32_tmem_a(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(b))
                 : "memory");
}
#define SF_X32_REGS(v)                                                                                     \
    "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),     \
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),    \
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),   \
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
#define SF_X32_OUTS(v)                                                                                     \
    "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),        \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),           \
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),         \
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),         \
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
#define SF_X32_LIST                                                                                        \
    "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27," \
    "%28,%29,%30,%31}"
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%32], " SF_X32_LIST ";" ::SF_X32_REGS(v), "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " SF_X32_LIST ", [%32];" : SF_X32_OUTS(v) : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%16], "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15};" ::"r"(v[0]),
        "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(taddr)
        : "memory");
}
// D (TMEM, f32) [+]= A (TMEM, f16 pairs per column, row = lane) x B (SMEM descriptor, f16)
__device__ __forceinline__ void mma_f16_tmem_a(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"((uint64_t)map),
        "r"(smem_addr(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// two-branch logistic (query.py:65-84), evaluated branch-free: both branches
// take exp(-|x|), so a warp with mixed signs runs one exp instead of two
__device__ __forceinline__ double sigmoid2(double x) {
    const double e = exp(-fabs(x));
    return (x >= 0 ? 1.0 : e) / (1.0 + e);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// alpha = min(o exp(-q/2), 0.99) with q <= 9 membership (0 if outside).
// q is evaluated in fp32 as a (dx + k dy)^2 + d dy^2 (no cancellation),
// branch-free; inside the guard band around 9 (`amb`) the reference's fp64 q
// decides instead (blend_alpha_exact, rasterizer.py:161-168).
__device__ __forceinline__ float blend_alpha_fast(const GeomF32& g, float pxf, float pyf, bool& amb) {
    constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // -0.5 / ln 2
    const float dx = (pxf - g.mx_hi) - g.mx_lo;
    const float dy = (pyf - g.my_hi) - g.my_lo;
    const float u = fmaf(g.k, dy, dx);
    const float ddy = g.d * dy * dy;
    const float q32 = fmaf(g.a * u, u, ddy);
    const float su = fabsf(dx) + fabsf(g.k * dy);
    const float guard = fmaf(1e-5f, fmaf(g.a * su, su, ddy), 1e-5f);
    amb = fabsf(q32 - 9.f) <= guard;
    const float al = fminf(g.opacity * exp2f(kNegHalfLog2e * fminf(q32, 9.5f)), 0.99f);
    return q32 > 9.f ? 0.f : al;
}
static __device__ __noinline__ float blend_alpha_exact(const GeomF32& g, const GeomRec* __restrict__ g64, double pxd,
                                                double pyd) {
    constexpr float kNegHalfLog2e = -0.72134752044448170368f;
    const GeomRec& G = *g64;  // rare: the reference's fp64 values from global memory
    double ddx = __dadd_rn(pxd, -G.mx), ddyd = __dadd_rn(pyd, -G.my);
    double t1 = __dmul_rn(__dmul_rn(G.a64, ddx), ddx);
    double t2 = __dmul_rn(__dmul_rn(__dmul_rn(2.0, G.b64), ddx), ddyd);
    double t3 = __dmul_rn(__dmul_rn(G.c64, ddyd), ddyd);
    double q = __dadd_rn(__dadd_rn(t1, t2), t3);
    if (!(q <= SF_CUTOFF)) return 0.f;
    return fminf(g.opacity * exp2f(kNegHalfLog2e * (float)q), 0.99f);
}

// Conservative patch culling: may any pixel of the 8x4 patch with corner
// (x0, y0) have q <= 9?  q = a (dx + k dy)^2 + d dy^2 is convex, so its
// minimum over the pixel-centre rectangle is 0 when the mean lies inside,
// else on one of the four edges (1-D minimisation with clamping).  fp32 with
// the same relative guard as blend_alpha; false positives only cost work,
// blend_alpha still decides every pixel (exactly, inside the guard band).
__device__ __forceinline__ bool patch_may_hit(const GeomF32& g, float x0, float y0) {
    const float dx0 = (x0 - g.mx_hi) - g.mx_lo, dx1 = dx0 + 7.f;
    const float dy0 = (y0 - g.my_hi) - g.my_lo, dy1 = dy0 + 3.f;
    if (dx0 <= 0.f && dx1 >= 0.f && dy0 <= 0.f && dy1 >= 0.f) return true;
    const float a = g.a, k = g.k, d = g.d;
    const float c = fmaf(a * k, k, d);
    const float s = -(a * k) / c;  // dy* = s * dx on an x edge
    float best = INFINITY, bs = 0.f;
    auto eval = [&](float dx, float dy) {
        const float u = fmaf(k, dy, dx);
        const float q = fmaf(a * u, u, d * dy * dy);
        if (q < best) {
            best = q;
            const float su = fabsf(dx) + fabsf(k * dy);
            bs = fmaf(a * su, su, d * dy * dy);
        }
    };
    eval(dx0, fminf(fmaxf(s * dx0, dy0), dy1));
    eval(dx1, fminf(fmaxf(s * dx1, dy0), dy1));
    eval(fminf(fmaxf(-k * dy0, dx0), dx1), dy0);
    eval(fminf(fmaxf(-k * dy1, dx0), dx1), dy1);
    return best <= 9.f + fmaf(1e-4f, bs, 1e-4f);
}

// Guard band of blend_alpha_fast bounded over the whole 8x4 patch: the
// per-pixel guard 1e-5 (a su^2 + d dy^2) + 1e-5 (su = |dx| + |k dy|) is
// maximal at the patch's largest |dx| and |dy|, so one value per (entry,
// patch) is conservative for every pixel (it can only add exact evaluations).
__device__ __forceinline__ float patch_guard(const GeomF32& g, float x0, float y0) {
    const float dx0 = (x0 - g.mx_hi) - g.mx_lo, dy0 = (y0 - g.my_hi) - g.my_lo;
    const float mdx = fmaxf(fabsf(dx0), fabsf(dx0 + 7.f)), mdy = fmaxf(fabsf(dy0), fabsf(dy0 + 3.f));
    const float su = fmaf(fabsf(g.k), mdy, mdx);
    return fmaf(1e-5f, fmaf(g.a * su, su, g.d * mdy * mdy), 1e-5f);
}
// blend_alpha_fast with a given guard (patch_guard): the same alpha and
// decision, a (possibly) wider ambiguity band
__device__ __forceinline__ float blend_alpha_guarded(const GeomF32& g, float pxf, float pyf, float guard, bool& amb) {
    constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // -0.5 / ln 2
    const float dx = (pxf - g.mx_hi) - g.mx_lo;
    const float dy = (pyf - g.my_hi) - g.my_lo;
    const float u = fmaf(g.k, dy, dx);
    const float q32 = fmaf(g.a * u, u, g.d * dy * dy);
    amb = fabsf(q32 - 9.f) <= guard;
    const float al = fminf(g.opacity * exp2f(kNegHalfLog2e * fminf(q32, 9.5f)), 0.99f);
    return q32 > 9.f ? 0.f : al;
}

// Warm L2 with the records of a later batch (lane j: record j)
__device__ __forceinline__ void prefetch_records(const BlendArgs& A, uint32_t r, int cs) {
    const char* g = reinterpret_cast<const char*>(A.geom + r);
    const char* c = reinterpret_cast<const char*>(A.chan) + (size_t)r * cs;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(g));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(c));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(c + cs - 1));
}

}  // namespace sf
