// ptx.cuh — thin inline-PTX wrappers for the sm_100a features the kernels use:
// mbarriers, TMA (cp.async.bulk.tensor), cp.async, tcgen05 (alloc / mma.sp / commit / ld / st / fences)
// and the UMMA shared-memory / instruction descriptors.  Bit layouts follow the sm_100 hardware
// interface (verified on B200 by csrc/probes.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vnm {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---------------------------------------------------------------- programmatic dependent launch
// Wait until the grids this one depends on (launched before it on the stream with programmatic serialization)
// have completed and their memory is visible; no-op without such a grid.  Called after the prologue
// (barriers, TMEM, descriptor prefetch: no global memory) so that part overlaps the previous kernel's tail.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Let the next grid on the stream be scheduled (its CTAs take SMs as this grid's CTAs exit).
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- proxies / fences
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
// 1-D bulk copy global -> shared (size and both addresses multiples of 16 B), completes on `bar` (tx bytes)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// TMA tensor store shared -> global (bulk-group completion), and the bulk-group waits
__device__ __forceinline__ void tma_store_2d(const void* tmap, int32_t x, int32_t y, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(x), "r"(y), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// TMA prefetch of a 2D box into L2 (no shared memory, no completion): warms the lines a later
// tma_load_2d of the same box will read, so that load sees L2 rather than HBM latency
__device__ __forceinline__ void tma_prefetch_l2(const void* tmap, int32_t x, int32_t y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(tmap)),
                 "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// ---------------------------------------------------------------- cp.async (16 B, zero-fill past src_bytes)
__device__ __forceinline__ void cp_async_16(void* dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_4(void* dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- tcgen05: TMEM
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// 32 lanes x 32 bit, 4 consecutive columns (warp w may only touch lanes 32*(w%4) .. +31)
__device__ __forceinline__ void tmem_st_32x32b_x4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a), "r"(b),
                 "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x1(uint32_t taddr, uint32_t a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(a) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers per thread (thread t = lane base + t)
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}

// ---------------------------------------------------------------- tcgen05: MMA
// D[tmem] (+)= A[smem, 2:4-compressed] * B[smem], metadata E in TMEM.  kind::f16 (bf16 in, fp32 acc).
__device__ __forceinline__ void mma_sp_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t e_tmem,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(e_tmem), "r"(idesc), "r"(accumulate)
        : "memory");
}
// dense variant (used by the probes / microbenchmarks only)
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// shared [128 rows][16 B] (descriptor: no swizzle, SBO 128 B) -> TMEM lanes 0..127, 4 consecutive columns
// (measured identity placement, csrc/probes2.cu); ordered with later tcgen05.mma of the same thread
__device__ __forceinline__ void tmem_cp_128x128b(uint32_t taddr, uint64_t d) {
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(d) : "memory");
}
// arrive on an mbarrier when all previously issued tcgen05 ops of this thread have completed
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// the 4 sparse MMAs of one stage (K-groups of 8 blocks: A +32 B, B +4096 B, metadata column pair
// e, e+2 with id2 = k & 1), issued by one elected lane of a converged warp
__device__ __forceinline__ void mma_sp_x4(uint32_t d, uint64_t ad, uint64_t bd, uint32_t e, uint32_t idesc0,
                                              uint32_t idesc1, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, acc, one;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t.reg .b32 e2;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "setp.ne.b32 acc, %6, 0;\n\t"
        "setp.eq.b32 one, 0, 0;\n\t"
        "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
        "add.s64 b1, %2, 256;\n\tadd.s64 b2, %2, 512;\n\tadd.s64 b3, %2, 768;\n\t"
        "add.u32 e2, %3, 2;\n\t"
        "@p tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, acc;\n\t"
        "@p tcgen05.mma.sp.cta_group::1.kind::f16 [%0], a1, b1, [%3], %5, one;\n\t"
        "@p tcgen05.mma.sp.cta_group::1.kind::f16 [%0], a2, b2, [e2], %4, one;\n\t"
        "@p tcgen05.mma.sp.cta_group::1.kind::f16 [%0], a3, b3, [e2], %5, one;\n\t"
        "}" ::"r"(d),
        "l"(ad), "l"(bd), "r"(e), "r"(idesc0), "r"(idesc1), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(p));
    return p != 0;
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
        "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

// ---------------------------------------------------------------- descriptors
// UMMA shared-memory matrix descriptor (sm_100): start addr>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version 1 at [46,48), base offset [49,52) = 0, LBO mode [52] = 0, layout type [61,64)
// (0 none, 1 128B_base32B, 2 128B, 4 64B, 6 32B).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(layout & 7u) << 61;
    return d;
}
constexpr uint32_t kLayoutSW128 = 2;

// Instruction descriptor, kind::f16: sparse id2 [0,2), sparse flag [2], c fmt [4,6) (F32 = 1),
// a fmt [7,10) / b fmt [10,13) (BF16 = 1), a major [15] (K = 0), b major [16] (MN = 1),
// N>>3 [17,23), M>>4 [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N, bool sparse, uint32_t id2, bool b_mn_major) {
    return (id2 & 3u) | ((sparse ? 1u : 0u) << 2) | (1u << 4) | (1u << 7) | (1u << 10) |
           ((b_mn_major ? 1u : 0u) << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// 128-byte swizzle (Swizzle<3,4,3>): 16-byte chunk index c (0..7) of row r (0..7) of an 8 x 128 B atom
__device__ __forceinline__ uint32_t sw128_offset(uint32_t row_in_atom, uint32_t byte_in_row) {
    return row_in_atom * 128u + ((((byte_in_row >> 4) ^ row_in_atom) & 7u) << 4) + (byte_in_row & 15u);
}

}  // namespace vnm

// ---------------------------------------------------------------- CTA pairs (cta_group::2)
namespace vnm {
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
// all threads of every CTA of the cluster
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address of this CTA's object -> the same object in the pair's rank-0 (leader) CTA
__device__ __forceinline__ uint32_t leader_addr(const void* p) { return smem_u32(p) & 0xFEFFFFFFu; }
// arrive on an mbarrier of another CTA of the cluster (cluster-scope release)
__device__ __forceinline__ void mbar_arrive_cluster(const void* own_bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(own_bar)),
        "r"(cta)
        : "memory");
}
// the same arrive with the default (CTA-scope) release: for signals that publish no memory writes to the peer,
// e.g. "my tcgen05.ld reads of the accumulator are complete" (tcgen05.wait::ld + fence::before_thread_sync
// order those); the cluster-scope release costs a MEMBAR.ALL.GPU per arrival (profiles/r01c_*)
__device__ __forceinline__ void mbar_arrive_remote(const void* own_bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(own_bar)),
        "r"(cta)
        : "memory");
}
// 2D TMA load into this CTA's shared memory whose completion is counted on the LEADER CTA's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(leader_addr(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// M = 256 sparse MMA over the CTA pair: A rows 0-127 / 128-255 and B columns 0..N/2-1 / N/2..N-1 from the
// shared memory of rank 0 / rank 1 (same offsets), D and metadata in each CTA's own TMEM
__device__ __forceinline__ void mma_sp_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t e_tmem,
                                                 uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(e_tmem), "r"(idesc), "r"(accumulate)
        : "memory");
}
// [128 rows][16 B] of each CTA's shared memory -> its own TMEM (issued by the leader for both)
__device__ __forceinline__ void tmem_cp_128x128b_pair(uint32_t taddr, uint64_t d) {
    asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(taddr), "l"(d) : "memory");
}
// arrive on the mbarrier at this offset in every CTA of `mask` when the pair's tcgen05 ops complete
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// 32 lanes x 32 bit, 32 consecutive columns
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
}  // namespace vnm

namespace vnm {
// ---------------------------------------------------------------- warp-converged stage issue (window form)
// One stage of the window-form main loop, issued by ONE elected lane of a CONVERGED warp (all 32 lanes call
// it with the same arguments): keeping the issuing warp converged lets ptxas hold the descriptors in uniform
// registers, so the MMAs leave back to back (a lane-0 branch cost ~30 dependent instructions per MMA and
// capped the tensor pipe at ~210 cycles per MMA, profiles/r01c_*).
// n (2 or 4) sparse MMAs k = 0..n-1: A descriptor + 2 (32 B) per k, B descriptor + b_step per k, metadata
// column e for k < 2 and e + 2 for k >= 2, id2 = k & 1 (idesc0 / idesc1); `accumulate` applies to k = 0.
template <int CG>
__device__ __forceinline__ void mma_sp_stage(uint32_t d, uint64_t ad, uint64_t bd, uint64_t b_step, uint64_t b_step2, uint32_t e,
                                             uint32_t idesc0, uint32_t idesc1, uint32_t accumulate, uint32_t n) {
    static_assert(CG == 1 || CG == 2, "cta_group");
    if constexpr (CG == 1) {
        asm volatile(
            "{\n\t.reg .pred p, p3, acc, one;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t.reg .b32 e2;\n\t"
            "elect.sync _|p, 0xffffffff;\n\t"
            "setp.ne.b32 acc, %6, 0;\n\t"
            "setp.eq.b32 one, 0, 0;\n\t"
            "setp.gt.and.u32 p3, %8, 2, p;\n\t"
            "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
            "add.s64 b1, %2, %7;\n\tadd.s64 b2, %2, %9;\n\tadd.s64 b3, b2, %7;\n\t"
            "add.u32 e2, %3, 2;\n\t"
            "@p tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, acc;\n\t"
            "@p tcgen05.mma.sp.cta_group::1.kind::f16 [%0], a1, b1, [%3], %5, one;\n\t"
            "@p3 tcgen05.mma.sp.cta_group::1.kind::f16 [%0], a2, b2, [e2], %4, one;\n\t"
            "@p3 tcgen05.mma.sp.cta_group::1.kind::f16 [%0], a3, b3, [e2], %5, one;\n\t"
            "}" ::"r"(d),
            "l"(ad), "l"(bd), "r"(e), "r"(idesc0), "r"(idesc1), "r"(accumulate), "l"(b_step), "r"(n), "l"(b_step2)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p, p3, acc, one;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t.reg .b32 e2;\n\t"
            "elect.sync _|p, 0xffffffff;\n\t"
            "setp.ne.b32 acc, %6, 0;\n\t"
            "setp.eq.b32 one, 0, 0;\n\t"
            "setp.gt.and.u32 p3, %8, 2, p;\n\t"
            "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
            "add.s64 b1, %2, %7;\n\tadd.s64 b2, %2, %9;\n\tadd.s64 b3, b2, %7;\n\t"
            "add.u32 e2, %3, 2;\n\t"
            "@p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%3], %4, acc;\n\t"
            "@p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], a1, b1, [%3], %5, one;\n\t"
            "@p3 tcgen05.mma.sp.cta_group::2.kind::f16 [%0], a2, b2, [e2], %4, one;\n\t"
            "@p3 tcgen05.mma.sp.cta_group::2.kind::f16 [%0], a3, b3, [e2], %5, one;\n\t"
            "}" ::"r"(d),
            "l"(ad), "l"(bd), "r"(e), "r"(idesc0), "r"(idesc1), "r"(accumulate), "l"(b_step), "r"(n), "l"(b_step2)
            : "memory");
    }
}
#ifdef VNM_ABLATIONS
// timing ablation only (results invalid): mma_sp_stage<2> with every MMA of the stage reading A at ad + a_step * k
__device__ __forceinline__ void mma_sp_stage_astep_pair(uint32_t d, uint64_t ad, uint64_t a_step, uint64_t bd,
                                                        uint64_t b_step, uint32_t e, uint32_t idesc0, uint32_t idesc1,
                                                        uint32_t accumulate, uint32_t n) {
    asm volatile(
        "{\n\t.reg .pred p, p3, acc, one;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t.reg .b32 e2;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "setp.ne.b32 acc, %6, 0;\n\t"
        "setp.eq.b32 one, 0, 0;\n\t"
        "setp.gt.and.u32 p3, %8, 2, p;\n\t"
        "add.s64 a1, %1, %9;\n\tadd.s64 a2, a1, %9;\n\tadd.s64 a3, a2, %9;\n\t"
        "add.s64 b1, %2, %7;\n\tadd.s64 b2, b1, %7;\n\tadd.s64 b3, b2, %7;\n\t"
        "add.u32 e2, %3, 2;\n\t"
        "@p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%3], %4, acc;\n\t"
        "@p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], a1, b1, [%3], %5, one;\n\t"
        "@p3 tcgen05.mma.sp.cta_group::2.kind::f16 [%0], a2, b2, [e2], %4, one;\n\t"
        "@p3 tcgen05.mma.sp.cta_group::2.kind::f16 [%0], a3, b3, [e2], %5, one;\n\t"
        "}" ::"r"(d),
        "l"(ad), "l"(bd), "r"(e), "r"(idesc0), "r"(idesc1), "r"(accumulate), "l"(b_step), "r"(n), "l"(a_step)
        : "memory");
}
#endif
// the window form: MMA i of the stage reads B at bd + i * b_step.  The window-16 form (8 < M < 16) interleaves two
// steps: MMAs 0 / 1 read the two half-windows of one block group (bd, bd + b_step = +8 rows), MMAs 2 / 3 those of
// the next (bd + b_step2, + b_step)
template <int CG>
__device__ __forceinline__ void mma_sp_stage(uint32_t d, uint64_t ad, uint64_t bd, uint64_t b_step, uint32_t e,
                                             uint32_t idesc0, uint32_t idesc1, uint32_t accumulate, uint32_t n) {
    mma_sp_stage<CG>(d, ad, bd, b_step, 2 * b_step, e, idesc0, idesc1, accumulate, n);
}
// tcgen05.cp 128x128b (smem [128 rows][16 B] -> TMEM), elected lane of a converged warp
template <int CG>
__device__ __forceinline__ void tmem_cp_elect(uint32_t taddr, uint64_t d) {
    if constexpr (CG == 1)
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t@p tcgen05.cp.cta_group::1.128x128b [%0], %1;\n\t}" ::"r"(taddr), "l"(d)
                     : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t@p tcgen05.cp.cta_group::2.128x128b [%0], %1;\n\t}" ::"r"(taddr), "l"(d)
                     : "memory");
}
// tcgen05.cp 128x256b (128 rows x 32 B of a shared-memory operand described by d -> 8 TMEM columns), elected lane
template <int CG>
__device__ __forceinline__ void tmem_cp256_elect(uint32_t taddr, uint64_t d) {
    if constexpr (CG == 1)
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t@p tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(taddr), "l"(d)
                     : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t@p tcgen05.cp.cta_group::2.128x256b [%0], %1;\n\t}" ::"r"(taddr), "l"(d)
                     : "memory");
}
// mma_sp_stage with A in TMEM (TS form): MMA i of the stage reads A at TMEM column a + 8 i (16 compressed bf16 per row)
__device__ __forceinline__ void mma_sp_stage_ts_pair(uint32_t d, uint32_t a, uint64_t bd, uint64_t b_step, uint32_t e,
                                                     uint32_t idesc0, uint32_t idesc1, uint32_t accumulate, uint32_t n) {
    asm volatile(
        "{\n\t.reg .pred p, p3, acc, one;\n\t.reg .b64 b1, b2, b3;\n\t.reg .b32 a1, a2, a3, e2;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "setp.ne.b32 acc, %6, 0;\n\t"
        "setp.eq.b32 one, 0, 0;\n\t"
        "setp.gt.and.u32 p3, %8, 2, p;\n\t"
        "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
        "add.s64 b1, %2, %7;\n\tadd.s64 b2, b1, %7;\n\tadd.s64 b3, b2, %7;\n\t"
        "add.u32 e2, %3, 2;\n\t"
        "@p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], [%1], %2, [%3], %4, acc;\n\t"
        "@p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], [a1], b1, [%3], %5, one;\n\t"
        "@p3 tcgen05.mma.sp.cta_group::2.kind::f16 [%0], [a2], b2, [e2], %4, one;\n\t"
        "@p3 tcgen05.mma.sp.cta_group::2.kind::f16 [%0], [a3], b3, [e2], %5, one;\n\t"
        "}" ::"r"(d),
        "r"(a), "l"(bd), "r"(e), "r"(idesc0), "r"(idesc1), "r"(accumulate), "l"(b_step), "r"(n)
        : "memory");
}
// commit of the pair's tcgen05 ops, multicast to the CTAs of `mask`, elected lane of a converged warp
__device__ __forceinline__ void mma_commit_pair_elect(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
        "@p tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
}  // namespace vnm
