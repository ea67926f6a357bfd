// selftest_sm100.cuh — one-CTA tcgen05 GEMM that exercises exactly the descriptor / swizzle
// encodings the attention kernels use (K-major and MN-major SWIZZLE_128B operands, M=128 with
// N=128 and N=16), with operands staged by plain threads so TMA is not involved.
#pragma once
#include "sm100_common.cuh"

namespace b200 {

constexpr int kSelftestSmem = 2 * 128 * 128 * 2 + 16 + 1024;

// byte offset of element (row, col) in a K-major SW128 tile with `rows` rows (col = K index)
__device__ __forceinline__ uint32_t sw128_kmajor(int row, int col, int rows) {
  return (col >> 6) * rows * 128 + row * 128 + ((((col & 63) >> 3) ^ (row & 7)) << 4) + (col & 7) * 2;
}

__global__ void __launch_bounds__(128) umma_selftest_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B,
                                                            float* D, int mode) {
  extern __shared__ uint8_t st_raw[];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(st_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sA + 128 * 128 * 2;
  uint64_t& bar = *reinterpret_cast<uint64_t*>(sB + 128 * 128 * 2);
  uint32_t& tslot = *reinterpret_cast<uint32_t*>(sB + 128 * 128 * 2 + 8);
  const int tid = threadIdx.x;
  // A: modes 0/1 K-major [M=128][K=128]; mode 2 MN-major given as [K][M] (same swizzle formula
  // with the 128-B rows running along M).
  for (int i = tid; i < 128 * 128; i += 128) {
    const int r = i / 128, c = i % 128;
    *reinterpret_cast<__nv_bfloat16*>(sA + sw128_kmajor(r, c, 128)) = A[i];
  }
  const int brows = (mode == 2) ? 16 : 128;
  for (int i = tid; i < brows * 128; i += 128) {
    const int r = i / 128, c = i % 128;
    *reinterpret_cast<__nv_bfloat16*>(sB + sw128_kmajor(r, c, brows)) = B[i];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc(&tslot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int N = (mode == 2) ? 16 : 128;
  if (mode == 3) {
    // A -> TMEM columns [128, 192): lane r = row r, column c holds (A[r][2c] lo, A[r][2c+1] hi)
    const uint32_t arow = tmem + 128 + (static_cast<uint32_t>((tid >> 5) << 5) << 16);
    for (int c = 0; c < 4; ++c) {
      uint32_t r[16];
      for (int j = 0; j < 16; ++j) {
        const __nv_bfloat16 lo = A[tid * 128 + c * 32 + 2 * j], hi = A[tid * 128 + c * 32 + 2 * j + 1];
        r[j] = static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(&lo)) |
               (static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(&hi)) << 16);
      }
      tmem_st16(arow + c * 16, r);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (tid == 0 && mode == 3) {
    const uint32_t b0 = smem_u32(sB);
    const uint32_t idesc = idesc_bf16_f32(128, 128, false, false);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t db = sdesc_sw128(b0 + (kk >> 2) * 128 * 128 + (kk & 3) * 32, 16, 1024);
      umma_ts(tmem, tmem + 128 + kk * 8, db, idesc, kk > 0);
    }
    umma_commit(&bar);
  } else if (tid == 0) {
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    const uint32_t idesc = idesc_bf16_f32(128, N, mode == 2, mode == 1);
    for (int kk = 0; kk < 8; ++kk) {
      uint64_t da, db;
      if (mode == 2) da = sdesc_sw128(a0 + kk * 2048, 16384, 1024);
      else da = sdesc_sw128(a0 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
      if (mode == 1) db = sdesc_sw128(b0 + kk * 2048, 16384, 1024);
      else db = sdesc_sw128(b0 + (kk >> 2) * brows * 128 + (kk & 3) * 32, 16, 1024);
      umma_ss(tmem, da, db, idesc, kk > 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t taddr = tmem + (static_cast<uint32_t>((tid >> 5) << 5) << 16);
  if (N == 16) {
    uint32_t r[16];
    tmem_ld16(taddr, r);
    for (int j = 0; j < 16; ++j) D[tid * 16 + j] = __uint_as_float(r[j]);
  } else {
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      tmem_ld32(taddr + c * 32, r);
      for (int j = 0; j < 32; ++j) D[tid * 128 + c * 32 + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// Paged KV-cache append: one warp per (token, kv head), 16-B vectors (128 x bf16 = 256 B row).
__device__ __forceinline__ void append_row_bf16(long long w, int lane, const uint4* __restrict__ nk,
                                                const uint4* __restrict__ nv, uint4* __restrict__ kc,
                                                uint4* __restrict__ vc, const int64_t* __restrict__ slots,
                                                int num_tokens, int kv_heads, int64_t num_slots) {
  if (w >= static_cast<long long>(num_tokens) * kv_heads) return;
  const int tok = static_cast<int>(w / kv_heads), h = static_cast<int>(w % kv_heads);
  const int64_t slot = slots[tok];
  if (slot < 0 || slot >= num_slots) return;
  const int64_t src = (static_cast<int64_t>(tok) * kv_heads + h) * 16;  // 16 uint4 per 128-wide row
  const int64_t dst = (slot * kv_heads + h) * 16;
  if (lane < 16) kc[dst + lane] = nk[src + lane];
  else vc[dst + lane - 16] = nv[src + lane - 16];
}

__global__ void cache_append_kernel(const uint4* __restrict__ nk, const uint4* __restrict__ nv,
                                    uint4* __restrict__ kc, uint4* __restrict__ vc,
                                    const int64_t* __restrict__ slots, int num_tokens, int kv_heads,
                                    int64_t num_slots) {
  append_row_bf16((static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5, threadIdx.x & 31, nk, nv,
                  kc, vc, slots, num_tokens, kv_heads, num_slots);
}

// fp8 variant: 16 lanes per (token, kv head) row, 8 bf16 -> 8 e4m3 each (satfinite, RN), K and V.
__device__ __forceinline__ uint32_t f32x4_to_e4m3x4(float a, float b, float c, float d) {
  uint16_t lo, hi;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"(b), "f"(a));
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(d), "f"(c));
  return static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
}

__device__ __forceinline__ uint2 bf16x8_to_e4m3x8(uint4 x, float inv) {
  auto f = [&](uint32_t w, int hi) { return __uint_as_float(hi ? (w & 0xFFFF0000u) : (w << 16)) * inv; };
  return make_uint2(f32x4_to_e4m3x4(f(x.x, 0), f(x.x, 1), f(x.y, 0), f(x.y, 1)),
                    f32x4_to_e4m3x4(f(x.z, 0), f(x.z, 1), f(x.w, 0), f(x.w, 1)));
}

__device__ __forceinline__ void append_row_fp8(long long g, int l, const uint4* __restrict__ nk,
                                               const uint4* __restrict__ nv, uint2* __restrict__ kc,
                                               uint2* __restrict__ vc, const int64_t* __restrict__ slots,
                                               int num_tokens, int kv_heads, int64_t num_slots, float inv_k,
                                               float inv_v) {
  if (g >= static_cast<long long>(num_tokens) * kv_heads) return;
  const int tok = static_cast<int>(g / kv_heads), h = static_cast<int>(g % kv_heads);
  const int64_t slot = slots[tok];
  if (slot < 0 || slot >= num_slots) return;
  const int64_t src = (static_cast<int64_t>(tok) * kv_heads + h) * 16 + l;  // 8 bf16 per lane
  const int64_t dst = (slot * kv_heads + h) * 16 + l;                       // 8 fp8 per lane
  kc[dst] = bf16x8_to_e4m3x8(nk[src], inv_k);
  vc[dst] = bf16x8_to_e4m3x8(nv[src], inv_v);
}

__global__ void cache_append_fp8_kernel(const uint4* __restrict__ nk, const uint4* __restrict__ nv,
                                        uint2* __restrict__ kc, uint2* __restrict__ vc,
                                        const int64_t* __restrict__ slots, int num_tokens, int kv_heads,
                                        int64_t num_slots, float inv_k, float inv_v) {
  append_row_fp8((static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 4, threadIdx.x & 15, nk, nv, kc,
                 vc, slots, num_tokens, kv_heads, num_slots, inv_k, inv_v);
}

// One serving decode step's host inputs in ONE kernel (attention.DecodeStep), read by the SMs
// straight from pinned, device-mapped host memory over PCIe: blocks [0, copy_blocks) copy the
// step's q and seq_lens (one contiguous staging range, 16-B vectors, 4 loads in flight per thread)
// into device memory; the remaining blocks append the new token's K/V into its page slot (the
// cache_append rows above, reading new_k / new_v / slot_mapping from the host).  Replaces an H2D
// copy node + the append kernel: both are PCIe-latency-bound and now overlap each other.
__global__ void __launch_bounds__(256) decode_ingest_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                            long long n16, int copy_blocks,
                                                            const uint4* __restrict__ nk,
                                                            const uint4* __restrict__ nv, void* kc, void* vc,
                                                            const int64_t* __restrict__ slots, int num_tokens,
                                                            int kv_heads, int64_t num_slots, int fp8, float inv_k,
                                                            float inv_v) {
  // PDL: K2' (launched programmatically behind this kernel) may start its prologue — barrier
  // init, TMEM alloc, descriptor prefetch — while the PCIe reads are in flight; its
  // griddepcontrol.wait still orders every data access after this grid's completion
  griddep_launch();
  if (static_cast<int>(blockIdx.x) < copy_blocks) {
    const long long stride = static_cast<long long>(copy_blocks) * blockDim.x;
    long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
      const uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
      dst[i] = a;
      dst[i + stride] = b;
      dst[i + 2 * stride] = c;
      dst[i + 3 * stride] = d;
    }
    for (; i < n16; i += stride) dst[i] = src[i];
    return;
  }
  const long long t = static_cast<long long>(blockIdx.x - copy_blocks) * blockDim.x + threadIdx.x;
  if (fp8)
    append_row_fp8(t >> 4, threadIdx.x & 15, nk, nv, reinterpret_cast<uint2*>(kc), reinterpret_cast<uint2*>(vc),
                   slots, num_tokens, kv_heads, num_slots, inv_k, inv_v);
  else
    append_row_bf16(t >> 5, threadIdx.x & 31, nk, nv, reinterpret_cast<uint4*>(kc), reinterpret_cast<uint4*>(vc),
                    slots, num_tokens, kv_heads, num_slots);
}

// fp8 (e4m3) descriptor self-test: D[128x128] = A . B^T with 128-byte rows.
//   mode 4: A [M=128][K=128] K-major, B [N=128][K=128] K-major
//   mode 5: A given as [K=128][M=128] (MN-major), B K-major
// Operands are byte tiles in the SW128 layout (16-byte chunk index ^ row % 8).
__global__ void __launch_bounds__(128) umma_selftest_fp8_kernel(const uint8_t* A, const uint8_t* B, float* D,
                                                                int mode) {
  extern __shared__ uint8_t st_raw[];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(st_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sA + 128 * 128;
  uint64_t& bar = *reinterpret_cast<uint64_t*>(sB + 128 * 128);
  uint32_t& tslot = *reinterpret_cast<uint32_t*>(sB + 128 * 128 + 8);
  const int tid = threadIdx.x;
  auto sw = [](int r, int c) { return r * 128 + ((((c >> 4) ^ (r & 7)) << 4) | (c & 15)); };
  for (int i = tid; i < 128 * 128; i += 128) {
    const int r = i / 128, c = i % 128;
    sA[sw(r, c)] = A[i];
    sB[sw(r, c)] = B[i];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc(&tslot, 128);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (tid < 32) {
    const uint32_t idesc = idesc_e4m3_f32(128, 128, mode == 5, false);
    const uint64_t da = sdesc_sw128(smem_u32(sA), 16, 1024), db = sdesc_sw128(smem_u32(sB), 16, 1024);
    // K step of 32: K-major operands advance 32 B within the row; MN-major A advances 32 rows
    if (mode == 5) umma_f8_ss_k128<((32 * 128) >> 4), 2>(tmem, da, db, idesc, 0u);
    else umma_f8_ss_k128<2, 2>(tmem, da, db, idesc, 0u);
    umma_commit_w(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t taddr = tmem + (static_cast<uint32_t>((tid >> 5) << 5) << 16);
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    for (int j = 0; j < 32; ++j) D[tid * 128 + c * 32 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

}  // namespace b200

namespace b200 {
// MMA throughput probe (timing only; operands are whatever is in smem/TMEM).
// A_TMEM: A operand from TMEM (TS) else smem K-major; B_MN: B operand MN-major else K-major.
// Descriptors are precomputed so the single issuing thread only issues tcgen05.mma.
template <int N, bool A_TMEM, bool B_MN, int LOAD_WARPS = 0>
__global__ void __launch_bounds__(128 + 32 * LOAD_WARPS) umma_rate_kernel(int iters, long long* out) {
  extern __shared__ uint8_t st_raw[];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(st_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sA + 32768;
  uint64_t& bar = *reinterpret_cast<uint64_t*>(sB + 65536);
  uint32_t& tslot = *reinterpret_cast<uint32_t*>(sB + 65536 + 8);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) *(&tslot + 1) = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, false, B_MN);
    uint64_t da[8], db[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      da[kk] = sdesc_sw128(a0 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
      db[kk] = B_MN ? sdesc_sw128(b0 + kk * 2048, N == 256 ? 16384 : 16384, 1024)
                    : sdesc_sw128(b0 + (kk >> 2) * N * 128 + (kk & 3) * 32, 16, 1024);
    }
    constexpr uint32_t DSTRIDE = N <= 128 ? 256 : 256;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + (it & 1) * (N <= 128 ? 128 : 256);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if constexpr (A_TMEM) umma_ts(d, tmem + 384 + kk * 8, db[kk], idesc, kk > 0);
        else umma_ss(d, da[kk], db[kk], idesc, kk > 0);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = (clock64() - t0) / iters;
    (void)DSTRIDE;
    *reinterpret_cast<volatile int*>(&tslot + 1) = 1;  // stop flag for the load warps
  }
  if constexpr (LOAD_WARPS > 0) {
    // contention: warps 4.. stream tcgen05.ld + tcgen05.st over TMEM columns [256+..) like a
    // softmax pass (read 64 cols, write 16 packed cols back)
    if (threadIdx.x >= 128) {
      const int w = (threadIdx.x >> 5) & 3;
      const uint32_t base = tmem + (static_cast<uint32_t>(w << 5) << 16) + 448;
      float acc = 0.f;
      while (*reinterpret_cast<volatile int*>(&tslot + 1) == 0) {
        uint32_t ra[32], rb[32];
        tmem_ld32x2(base, base + 32, ra, rb);
        uint32_t pk[16];
        for (int i = 0; i < 16; ++i) pk[i] = ra[2 * i] ^ rb[2 * i + 1];
        tmem_st16(base, pk);
        acc += __uint_as_float(ra[0]);
      }
      if (acc == 12345.f) out[0] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}
}  // namespace b200
