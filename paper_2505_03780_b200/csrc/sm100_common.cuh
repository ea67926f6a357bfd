// sm100_common.cuh — thin inline-PTX layer for the sm_100a attention kernels.
//
// Everything the kernels need from Blackwell lives here: mbarriers, TMA
// tensor loads, tcgen05 (TMEM alloc / MMA / commit / ld / st) and the UMMA
// shared-memory + instruction descriptors.  No CUTLASS/CuTe: the bit layouts
// follow the PTX ISA's tcgen05 "matrix descriptor" and "instruction
// descriptor" tables (cross-checked against the vendored CuTe headers'
// SmemDescriptor / InstrDescriptor unions, cute/arch/mma_sm100_desc.hpp).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#ifndef B200_WAIT_TRAP_SPINS
// A wedged pipeline traps (sticky launch error, process exits) instead of
// hanging the GPU: ~2^28 failed try_wait probes is several seconds.
#define B200_WAIT_TRAP_SPINS (1u << 28)
#endif

namespace b200 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- programmatic dependent launch
// A kernel launched with the programmatic-serialization attribute may start while its predecessor
// in the stream drains: everything before griddep_wait() (barrier init, TMEM alloc, descriptor
// prefetch) overlaps the predecessor's tail; griddep_wait() returns once the predecessor grid has
// completed and its memory is visible, so no global memory is touched before it.  Without the
// attribute both are no-ops.  griddep_launch() lets the NEXT kernel in the stream start its own
// prologue as soon as SMs free up (it still waits for this grid to finish before any data access).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
#ifndef B200_WAIT_HINT_NS
#define B200_WAIT_HINT_NS 0  // > 0: try_wait suspend-time hint (fewer spin iterations / issue slots)
#endif
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar_addr, uint32_t parity) {
  uint32_t ok;
#if B200_WAIT_HINT_NS > 0
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar_addr), "r"(parity), "n"(B200_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar_addr), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}
// non-blocking probe of a phase (mbarrier.test_wait): true iff the phase with this parity completed
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t spins = 0;
  while (!mbar_try_wait(a, parity)) {
    if (++spins == B200_WAIT_TRAP_SPINS) __trap();
  }
}
#ifndef B200_PRODUCER_SLEEP_NS
#define B200_PRODUCER_SLEEP_NS 0  // > 0: producer-side (TMA / MMA warp) waits back off with nanosleep
#endif
// Wait used by warps that share an SMSP with softmax warps but have no arithmetic of their own:
// optionally yields the issue slot between polls.
__device__ __forceinline__ void mbar_wait_producer(uint64_t* bar, uint32_t parity) {
#if B200_PRODUCER_SLEEP_NS > 0
  const uint32_t a = smem_u32(bar);
  uint32_t spins = 0;
  while (!mbar_try_wait(a, parity)) {
    if (++spins == B200_WAIT_TRAP_SPINS) __trap();
    __nanosleep(B200_PRODUCER_SLEEP_NS);
  }
#else
  mbar_wait(bar, parity);
#endif
}

// Named barrier among a subset of warps (ids 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// Named barrier that also ANDs a predicate over the participating threads.
__device__ __forceinline__ bool named_bar_and(uint32_t id, uint32_t nthreads, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "bar.red.and.pred q, %2, %3, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(id), "r"(nthreads)
      : "memory");
  return r != 0;
}

// Generic-proxy smem writes -> visible to the async proxy (tensor core / TMA).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// --------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// Same, with an L2 eviction-priority policy (createpolicy result).
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                                 int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
// TMA store of a shared-memory box to global (bulk-group completion), and its group waits
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the sources of every committed group have been read (the smem may be rewritten)
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed group has completed (its global writes are performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------------------ tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T   (kind::f16, bf16 in, fp32 accumulate)
__device__ __forceinline__ void umma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// kind::f8f6f4 (e4m3 x e4m3 -> f32): D[tmem] (+)= A[smem] * B[smem]^T, K = 32 bytes per instruction.
// Warp-convergent, K = 128 as 4 x K32 steps; A advances AS and B advances BS 16-byte units per step.
template <int AS, int BS>
__device__ __forceinline__ void umma_f8_ss_k128(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred e, p;\n\t.reg .b64 ta, tb;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t"
      "setp.eq.u32 p, 0, 0;\n\t"
      "add.s64 ta, %1, %5;\n\tadd.s64 tb, %2, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %7;\n\tadd.s64 tb, %2, %8;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %9;\n\tadd.s64 tb, %2, %10;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], ta, tb, %3, p;\n\t"
      "}"
      :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "n"(AS), "n"(BS), "n"(2 * AS), "n"(2 * BS),
         "n"(3 * AS), "n"(3 * BS)
      : "memory");
}

// Warp-convergent variants: the whole warp executes them (operands warp-uniform, so they stay
// in uniform registers) and one elected lane issues — no divergent wrapper per MMA.
__device__ __forceinline__ void umma_ss_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// Eight K=16 steps of one MMA (K = 128) in one asm block: operand k of step kk is
// base + (kk & 3) * S + (kk >> 2) * H (16-byte descriptor units). Issued by one elected lane of a
// convergent warp; keeps the issuing warp's instruction count (and SMSP pressure) minimal.
template <int AS, int AH, int BS, int BH>
__device__ __forceinline__ void umma_ss_k128(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred e, p;\n\t.reg .b64 ta, tb;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "setp.eq.u32 p, 0, 0;\n\t"
      "add.s64 ta, %1, %5;\n\tadd.s64 tb, %2, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %7;\n\tadd.s64 tb, %2, %8;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %9;\n\tadd.s64 tb, %2, %10;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %11;\n\tadd.s64 tb, %2, %12;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %13;\n\tadd.s64 tb, %2, %14;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %15;\n\tadd.s64 tb, %2, %16;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %17;\n\tadd.s64 tb, %2, %18;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "}"
      :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "n"(((1 & 3) * AS + (1 >> 2) * AH)), "n"(((1 & 3) * BS + (1 >> 2) * BH)),
         "n"(((2 & 3) * AS + (2 >> 2) * AH)), "n"(((2 & 3) * BS + (2 >> 2) * BH)),
         "n"(((3 & 3) * AS + (3 >> 2) * AH)), "n"(((3 & 3) * BS + (3 >> 2) * BH)),
         "n"(((4 & 3) * AS + (4 >> 2) * AH)), "n"(((4 & 3) * BS + (4 >> 2) * BH)),
         "n"(((5 & 3) * AS + (5 >> 2) * AH)), "n"(((5 & 3) * BS + (5 >> 2) * BH)),
         "n"(((6 & 3) * AS + (6 >> 2) * AH)), "n"(((6 & 3) * BS + (6 >> 2) * BH)),
         "n"(((7 & 3) * AS + (7 >> 2) * AH)), "n"(((7 & 3) * BS + (7 >> 2) * BH))
      : "memory");
}

// TS variant: A from TMEM, step kk at a_tmem + 8 kk + (kk >= 4 ? AGAP : 0) (16 bf16 = 8 columns;
// AGAP > 0 when the two 64-row K halves of P were written by different warps into their own S
// column ranges); B as above.
template <int BS, int BH, int AGAP = 0>
__device__ __forceinline__ void umma_ts_k128(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred e, p;\n\t.reg .b32 ta;\n\t.reg .b64 tb;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "setp.eq.u32 p, 0, 0;\n\t"
      "add.s32 ta, %1, 8;\n\tadd.s64 tb, %2, %5;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, 16;\n\tadd.s64 tb, %2, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, 24;\n\tadd.s64 tb, %2, %7;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, %12;\n\tadd.s64 tb, %2, %8;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, %13;\n\tadd.s64 tb, %2, %9;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, %14;\n\tadd.s64 tb, %2, %10;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, %15;\n\tadd.s64 tb, %2, %11;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "}"
      :: "r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc), "n"(((1 & 3) * BS + (1 >> 2) * BH)), "n"(((2 & 3) * BS + (2 >> 2) * BH)), "n"(((3 & 3) * BS + (3 >> 2) * BH)), "n"(((4 & 3) * BS + (4 >> 2) * BH)), "n"(((5 & 3) * BS + (5 >> 2) * BH)), "n"(((6 & 3) * BS + (6 >> 2) * BH)), "n"(((7 & 3) * BS + (7 >> 2) * BH)),
         "n"(32 + AGAP), "n"(40 + AGAP), "n"(48 + AGAP), "n"(56 + AGAP)
      : "memory");
}

// ------------------------------------------------ CTA pair (cta_group::2, a 2-CTA cluster on one TPC)
// One elected thread of the leader CTA (cluster rank 0) issues an M = 256 MMA: rows 0..127 of A
// come from the leader's shared memory (or TMEM), rows 128..255 from the peer's at the same
// offset; B is split along N across the pair (each CTA holds N/2 rows of it at the same offset);
// each CTA's TMEM receives its own 128 rows of D at the same TMEM address.
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cta address of this CTA -> shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
// wait with cluster-scope acquire: arrivals came from the peer CTA (release.cluster) or its TMA
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t spins = 0;
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (++spins == B200_WAIT_TRAP_SPINS) __trap();
  }
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load into this CTA's shared memory whose completion is counted on an mbarrier of either CTA
// of the pair (`bar_cluster` from mapa_shared): both CTAs' halves land on the leader's barrier.
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
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
// commit of the pair's MMAs, arriving on the barrier at this offset in both CTAs
__device__ __forceinline__ void umma_commit_pair_w(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::
          "r"(smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
// cta_group::2 versions (issued by the leader CTA of a pair; same operand stepping)
template <int AS, int AH, int BS, int BH>
__device__ __forceinline__ void umma_ss_k128_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred e, p;\n\t.reg .b64 ta, tb;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "setp.eq.u32 p, 0, 0;\n\t"
      "add.s64 ta, %1, %5;\n\tadd.s64 tb, %2, %6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %7;\n\tadd.s64 tb, %2, %8;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %9;\n\tadd.s64 tb, %2, %10;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %11;\n\tadd.s64 tb, %2, %12;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %13;\n\tadd.s64 tb, %2, %14;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %15;\n\tadd.s64 tb, %2, %16;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "add.s64 ta, %1, %17;\n\tadd.s64 tb, %2, %18;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ta, tb, %3, p;\n\t"
      "}"
      :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "n"(((1 & 3) * AS + (1 >> 2) * AH)), "n"(((1 & 3) * BS + (1 >> 2) * BH)),
         "n"(((2 & 3) * AS + (2 >> 2) * AH)), "n"(((2 & 3) * BS + (2 >> 2) * BH)),
         "n"(((3 & 3) * AS + (3 >> 2) * AH)), "n"(((3 & 3) * BS + (3 >> 2) * BH)),
         "n"(((4 & 3) * AS + (4 >> 2) * AH)), "n"(((4 & 3) * BS + (4 >> 2) * BH)),
         "n"(((5 & 3) * AS + (5 >> 2) * AH)), "n"(((5 & 3) * BS + (5 >> 2) * BH)),
         "n"(((6 & 3) * AS + (6 >> 2) * AH)), "n"(((6 & 3) * BS + (6 >> 2) * BH)),
         "n"(((7 & 3) * AS + (7 >> 2) * AH)), "n"(((7 & 3) * BS + (7 >> 2) * BH))
      : "memory");
}

template <int BS, int BH, int AGAP = 0>
__device__ __forceinline__ void umma_ts_k128_pair(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred e, p;\n\t.reg .b32 ta;\n\t.reg .b64 tb;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "setp.eq.u32 p, 0, 0;\n\t"
      "add.s32 ta, %1, 8;\n\tadd.s64 tb, %2, %5;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, 16;\n\tadd.s64 tb, %2, %6;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, 24;\n\tadd.s64 tb, %2, %7;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, %12;\n\tadd.s64 tb, %2, %8;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, %13;\n\tadd.s64 tb, %2, %9;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, %14;\n\tadd.s64 tb, %2, %10;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "add.s32 ta, %1, %15;\n\tadd.s64 tb, %2, %11;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [ta], tb, %3, p;\n\t"
      "}"
      :: "r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc), "n"(((1 & 3) * BS + (1 >> 2) * BH)), "n"(((2 & 3) * BS + (2 >> 2) * BH)), "n"(((3 & 3) * BS + (3 >> 2) * BH)), "n"(((4 & 3) * BS + (4 >> 2) * BH)), "n"(((5 & 3) * BS + (5 >> 2) * BH)), "n"(((6 & 3) * BS + (6 >> 2) * BH)), "n"(((7 & 3) * BS + (7 >> 2) * BH)),
         "n"(32 + AGAP), "n"(40 + AGAP), "n"(48 + AGAP), "n"(56 + AGAP)
      : "memory");
}

// Arrive on an mbarrier once every previously issued tcgen05 op of this thread completes.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// TMEM -> registers, 32 lanes x 32b, 16 / 32 consecutive columns per thread.
// The wait::ld is fused into the same asm so no consumer can be hoisted above it.
__device__ __forceinline__ void tmem_ld1(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
// N consecutive fp32 columns (N in {1,2,4,8,16,32,64,...}) into r[0..N)
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t* r) {
  if constexpr (N == 1) {
    tmem_ld1(taddr, r);
  } else if constexpr (N == 2) {
    tmem_ld2(taddr, r);
  } else if constexpr (N == 4) {
    tmem_ld4(taddr, r);
  } else if constexpr (N == 8) {
    tmem_ld8(taddr, r);
  } else if constexpr (N == 16) {
    tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(r));
  } else {
    static_assert(N % 32 == 0, "column count");
#pragma unroll
    for (int c = 0; c < N / 32; ++c) tmem_ld32(taddr + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r + c * 32));
  }
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(r[32])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st1(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(r[0]) : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(r[0]), "r"(r[1]) : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3])
               : "memory");
}
// N consecutive fp32 columns (N in {1, 2, 4, 8, 16, 32, 64, ...}) from r[0..N)
template <int N>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t* r) {
  if constexpr (N == 1) {
    tmem_st1(taddr, r);
  } else if constexpr (N == 2) {
    tmem_st2(taddr, r);
  } else if constexpr (N == 4) {
    tmem_st4(taddr, r);
  } else if constexpr (N == 8) {
    tmem_st8(taddr, r);
  } else if constexpr (N == 16) {
    tmem_st16(taddr, *reinterpret_cast<const uint32_t(*)[16]>(r));
  } else {
    static_assert(N % 32 == 0, "column count");
#pragma unroll
    for (int c = 0; c < N / 32; ++c) tmem_st32(taddr + c * 32, *reinterpret_cast<const uint32_t(*)[32]>(r + c * 32));
  }
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------ descriptors
// UMMA shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bits.
//   [0,14) start>>4  [16,30) LBO>>4  [32,46) SBO>>4  [46,48) version=1
//   [49,52) base offset (0: tiles are 1024-B aligned)  [61,64) layout (2 = SW128)
// K-major SW128  : rows of 128 B, 8-row atoms 1024 B apart -> SBO = 1024, LBO unused (16).
// MN-major SW128 : 128-B rows run along M/N (64 bf16), K rows 128 B apart;
//                  LBO = byte stride between 64-wide M/N blocks, SBO = stride between 8-row K groups.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// Instruction descriptor, kind::f16: bf16 x bf16 -> f32.
//   [4,6) c_format=1 (F32)  [7,10) a_format=1 (BF16)  [10,13) b_format=1 (BF16)
//   [15] a_major (1 = MN)  [16] b_major (1 = MN)  [17,23) N>>3  [24,29) M>>4
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}

// ------------------------------------------------------------- numerics
// Blackwell packed fp32 pairs (FFMA2 / FADD2): two elements per issue slot.
// Instruction descriptor, kind::f8f6f4: e4m3 x e4m3 -> f32 (a_format = b_format = 0 = E4M3).
__host__ __device__ constexpr uint32_t idesc_e4m3_f32(uint32_t M, uint32_t N, bool a_mn, bool b_mn) {
  return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void ffma2(float& y0, float& y1, float x0, float x1, float a, float b) {
  // (y0, y1) = (x0, x1) * a + b
  asm("{\n\t.reg .b64 x, s, c;\n\t"
      "mov.b64 x, {%2, %3};\n\t"
      "mov.b64 s, {%4, %4};\n\t"
      "mov.b64 c, {%5, %5};\n\t"
      "fma.rn.ftz.f32x2 x, x, s, c;\n\t"
      "mov.b64 {%0, %1}, x;\n\t}"
      : "=f"(y0), "=f"(y1)
      : "f"(x0), "f"(x1), "f"(a), "f"(b));
}
// (y0, y1) = (a0, a1) * (b0, b1) + c
__device__ __forceinline__ void ffma2_v(float& y0, float& y1, float a0, float a1, float b0, float b1, float c) {
  asm("{\n\t.reg .b64 a, b, c;\n\t"
      "mov.b64 a, {%2, %3};\n\t"
      "mov.b64 b, {%4, %5};\n\t"
      "mov.b64 c, {%6, %6};\n\t"
      "fma.rn.ftz.f32x2 a, a, b, c;\n\t"
      "mov.b64 {%0, %1}, a;\n\t}"
      : "=f"(y0), "=f"(y1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c));
}
__device__ __forceinline__ void fadd2(float& a0, float& a1, float b0, float b1) {
  asm("{\n\t.reg .b64 a, b;\n\t"
      "mov.b64 a, {%0, %1};\n\t"
      "mov.b64 b, {%2, %3};\n\t"
      "add.rn.ftz.f32x2 a, a, b;\n\t"
      "mov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(b0), "f"(b1));
}
// TMEM -> registers, two 32-column chunks behind one wait::ld (halves the exposed latency)
__device__ __forceinline__ void tmem_ld32x2(uint32_t taddr0, uint32_t taddr1, uint32_t (&a)[32], uint32_t (&b)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%64];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%65];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]),
        "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15]),
        "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]), "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]),
        "=r"(a[24]), "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31]),
        "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]),
        "=r"(b[8]), "=r"(b[9]), "=r"(b[10]), "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15]),
        "=r"(b[16]), "=r"(b[17]), "=r"(b[18]), "=r"(b[19]), "=r"(b[20]), "=r"(b[21]), "=r"(b[22]), "=r"(b[23]),
        "=r"(b[24]), "=r"(b[25]), "=r"(b[26]), "=r"(b[27]), "=r"(b[28]), "=r"(b[29]), "=r"(b[30]), "=r"(b[31])
      : "r"(taddr0), "r"(taddr1)
      : "memory");
}

// Split load / wait for software pipelining: the wait names the loaded registers as in/out
// operands, so no consumer of them can be scheduled above it.
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld_regs(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31]) : : "memory");
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
// 256-bit store (STG.E.256 on sm_100): one full 32-byte sector per thread
__device__ __forceinline__ void st_global_v8(void* ptr, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(ptr), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void st_global_v4(void* ptr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

}  // namespace b200
