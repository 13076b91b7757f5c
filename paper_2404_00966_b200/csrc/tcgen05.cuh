// tcgen05.cuh -- minimal sm_100a tensor-core plumbing (inline PTX): TMEM
// allocation, shared-memory matrix descriptors (K-major, 128-byte swizzle),
// the tf32 MMA, its mbarrier commit, and TMEM -> register loads.
// Bit layouts follow the PTX ISA tcgen05 descriptors (cross-checked against
// CUTLASS cute/arch/mma_sm100_desc.hpp, vendored read-only in flashinfer).
#pragma once
#include <cstdint>

namespace gts {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Shared-memory matrix descriptor: K-major operand, SWIZZLE_128B atoms of
// 8 rows x 128 bytes, 8-row groups packed (SBO = 1024 B), version 1 (sm100).
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);       // [0,14)  start address >> 4
    d |= (uint64_t)1u << 16;                        // [16,30) LBO (ignored for swizzled K-major)
    d |= (uint64_t)(1024u >> 4) << 32;              // [32,46) SBO: stride between 8-row groups
    d |= (uint64_t)1u << 46;                        // [46,48) descriptor version 1
    d |= (uint64_t)2u << 61;                        // [61,64) SWIZZLE_128B
    return d;
}

// Instruction descriptor, kind::tf32: D f32, A/B tf32, both K-major.
__device__ __forceinline__ uint32_t idesc_tf32(int M, int N)
{
    return (1u << 4)                          // c_format = F32
         | (2u << 7)                          // a_format = TF32
         | (2u << 10)                         // b_format = TF32
         | ((uint32_t)(N >> 3) << 17)         // n_dim
         | ((uint32_t)(M >> 4) << 24);        // m_dim
}

// Byte offset of element (row, k) in a K-major SW128 tile whose rows are 128 B
// (32 fp32): 16-byte chunk index XOR-ed with (row mod 8).
__device__ __forceinline__ uint32_t sw128_offset(int row, int chunk16)
{
    return (uint32_t)row * 128u + (uint32_t)((chunk16 ^ (row & 7)) << 4);
}

__device__ __forceinline__ void tmem_alloc(uint32_t *slot_smem, uint32_t ncols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *mbar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(mbar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count));
}

// try_wait's suspend-time hint: a waiting thread may sleep until the phase
// completes (or the hint expires) instead of re-issuing the probe, leaving
// the issue slots to the warps that have work
constexpr uint32_t kMbarSuspendHint = 0x989680u;

__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t phase)
{
    uint32_t done = 0;
    const uint32_t a = smem_u32(mbar);
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(phase), "r"(kMbarSuspendHint)
            : "memory");
    }
}

__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Instruction descriptor, kind::f16 with BF16 A/B, F32 accumulate, K-major.
__device__ __forceinline__ uint32_t idesc_bf16(int M, int N)
{
    return (1u << 4)                          // c_format = F32
         | (1u << 7)                          // a_format = BF16
         | (1u << 10)                         // b_format = BF16
         | ((uint32_t)(N >> 3) << 17)         // n_dim
         | ((uint32_t)(M >> 4) << 24);        // m_dim
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// 16 consecutive fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16])
{
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

// the same load without the wait (pair it with tmem_wait_ld before use)
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// after tmem_wait_ld: make every later use of r depend on the wait (the
// registers of an issued tcgen05.ld are undefined until it)
__device__ __forceinline__ void tmem_tie(uint32_t (&r)[16])
{
#pragma unroll
    for (int i = 0; i < 16; i++) asm volatile("" : "+r"(r[i]));
}

// 16-byte global -> shared async copy; src_size 0 zero-fills the chunk
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *g, uint32_t src_size)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// arrive on `mbar` once every cp.async this thread issued so far has landed
// (noinc: the barrier's expected count already includes this arrival)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *mbar)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *mbar)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(mbar))
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Bulk (TMA-engine) copies: one thread posts the stage's byte count on the
// mbarrier (an arrival) and issues cp.async.bulk copies that complete it.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *mbar, uint32_t bytes)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(mbar)),
                 "r"(bytes)
                 : "memory");
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(uint32_t saddr, const void *g, uint32_t bytes, uint64_t *mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(saddr),
                 "l"(g), "r"(bytes), "r"(smem_u32(mbar))
                 : "memory");
}

}  // namespace tc
}  // namespace gts
