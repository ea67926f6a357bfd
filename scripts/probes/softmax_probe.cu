// Per-SMSP cost of the prefill softmax on one 128-column S row slice (sm_100a).  One CTA per SM,
// NW warps; warp w works on TMEM lanes 32*(w%4), columns 128*(w/4).  Modes:
//   0 full speculative pass (tcgen05.ld, exp2, sum, pack, tcgen05.st)   [prefill_sm100.cuh]
//   1 loads only (4 x tcgen05.ld.32x32b.x32 + wait, then a trivial use)
//   2 full pass with every exponential on MUFU (EMU 0)
//   3 full pass with every other pair on the FMA pipe (EMU 2)
//   4 loads + exp2 + sum, no P pack/store
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --use_fast_math -I../../include \
//      -I../../paper_2505_03780_b200/csrc -o softmax_probe softmax_probe.cu
#include <cstdio>
#include "prefill_sm100.cuh"

using namespace b200;

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(long long* out, float* sink, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t addr = tmem + (static_cast<uint32_t>((warp & 3) << 5) << 16) + (warp >> 2) * 128;
  {
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(0.01f * ((threadIdx.x * 7 + i) % 97) - 0.3f);
    for (int c = 0; c < 4; ++c) tmem_st32(addr + c * 32, r);
    tmem_wait_st();
  }
  __syncthreads();
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float l = 0.f;
    if constexpr (MODE == 0) {
      softmax_speculative<128, 3, 1>(addr, 1.4427f, 2.0f + it * 1e-9f, l, 0);
      tmem_wait_st();
      // restore S (P overwrote the first 64 columns) so the next iteration reads scores, off the clock
    } else if constexpr (MODE == 2) {
      softmax_speculative<128, 0, 1>(addr, 1.4427f, 2.0f + it * 1e-9f, l, 0);
      tmem_wait_st();
    } else if constexpr (MODE == 3) {
      softmax_speculative<128, 2, 1>(addr, 1.4427f, 2.0f + it * 1e-9f, l, 0);
      tmem_wait_st();
    } else if constexpr (MODE == 1) {
      uint32_t r[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32_nowait(addr + c * 32, r[c]);
      tmem_wait_ld_regs(r[0]);
      tmem_wait_ld_regs(r[1]);
      tmem_wait_ld_regs(r[2]);
      tmem_wait_ld_regs(r[3]);
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) l += __uint_as_float(r[c][i]);
    } else if constexpr (MODE == 4) {
      uint32_t r[2][32];
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      tmem_ld32_nowait(addr, r[0]);
      tmem_wait_ld_regs(r[0]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c + 1 < 4) tmem_ld32_nowait(addr + (c + 1) * 32, r[(c + 1) & 1]);
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float x0, x1;
          ffma2(x0, x1, __uint_as_float(r[c & 1][i]), __uint_as_float(r[c & 1][i + 1]), 1.4427f, -2.0f);
          const float e0 = fast_exp2(x0), e1 = fast_exp2(x1);
          if (i & 2) fadd2(s0, s1, e0, e1); else fadd2(s2, s3, e0, e1);
        }
        if (c + 1 < 4) tmem_wait_ld_regs(r[(c + 1) & 1]);
      }
      l = s0 + s1 + s2 + s3;
    }
    acc += l;
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// the nw8 kernel's work split: each warp owns NCOL columns, registers capped by a LB-thread bound
template <int NCOL, int LB>
__global__ void __launch_bounds__(LB, 1) probe_split(long long* out, float* sink, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t addr = tmem + (static_cast<uint32_t>((warp & 3) << 5) << 16) + (warp >> 2) * NCOL;
  {
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(0.01f * ((threadIdx.x * 7 + i) % 97) - 0.3f);
    for (int c = 0; c < NCOL / 32; ++c) tmem_st32(addr + c * 32, r);
    tmem_wait_st();
  }
  __syncthreads();
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float l = 0.f;
    softmax_speculative<NCOL, 3, 1>(addr, 1.4427f, 2.0f + it * 1e-9f, l, 0);
    tmem_wait_st();
    acc += l;
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int NCOL, int LB>
void run_split(const char* name, int nw, long long* d_out, float* sink) {
  const int iters = 2000;
  probe_split<NCOL, LB><<<148, nw * 32>>>(d_out, sink, iters);
  probe_split<NCOL, LB><<<148, nw * 32>>>(d_out, sink, iters);
  long long h[16];
  cudaMemcpy(h, d_out, sizeof(long long) * nw, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < nw; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-28s warps/SMSP=%d: %7.1f cycles per %d-column slice per warp\n", name, nw / 4, (double)mx / iters, NCOL);
}

// softmax warps (NW, NCOL columns each, TMEM columns [0, 256)) while one MMA warp keeps the tensor
// core busy with 128x128x128 SS MMAs into TMEM columns [256, 512) (MMA = false: the warp idles)
template <int NCOL, int NW, bool MMA>
__global__ void __launch_bounds__(NW * 32 + 32, 1) probe_mma(long long* out, float* sink, int iters) {
  extern __shared__ uint8_t raw[];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sA + 32768;
  __shared__ uint32_t slot;
  __shared__ int done;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    done = 0;
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == NW) {
    long long n = 0;
    if (MMA) {
      const uint64_t da = sdesc_sw128(smem_u32(sA), 16, 1024), db = sdesc_sw128(smem_u32(sB), 16, 1024);
      constexpr uint32_t idesc = idesc_bf16_f32(128, 128, false, false);
      while (*reinterpret_cast<volatile int*>(&done) < NW * 32) {
        umma_ss_k128<2, 1024, 2, 1024>(tmem + 256 + (n & 1) * 128, da, db, idesc, 0u);
        ++n;
        if ((n & 3) == 0) {  // keep the queue bounded: wait for the MMAs issued so far
          umma_commit_w(&bar);
          mbar_wait(&bar, ((n >> 2) - 1) & 1);
        }
      }
    }
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[15] = n;
  } else {
    const uint32_t addr = tmem + (static_cast<uint32_t>((warp & 3) << 5) << 16) + (warp >> 2) * NCOL;
    {
      uint32_t r[32];
      for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(0.01f * ((threadIdx.x * 7 + i) % 97) - 0.3f);
      for (int c = 0; c < NCOL / 32; ++c) tmem_st32(addr + c * 32, r);
      tmem_wait_st();
    }
    named_bar_sync(1, NW * 32);
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      float l = 0.f;
      softmax_speculative<NCOL, 3, 1>(addr, 1.4427f, 2.0f + it * 1e-9f, l, 0);
      tmem_wait_st();
      acc += l;
    }
    long long t1 = clock64();
    atomicAdd(&done, 1);
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[warp] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int NCOL, int NW, bool MMA>
void run_mma(const char* name, long long* d_out, float* sink) {
  const int iters = 2000, smem = 65536 + 1024;
  auto k = probe_mma<NCOL, NW, MMA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaMemset(d_out, 0, 16 * sizeof(long long));
  k<<<148, NW * 32 + 32, smem>>>(d_out, sink, iters);
  k<<<148, NW * 32 + 32, smem>>>(d_out, sink, iters);
  long long h[16];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < NW; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-34s: %7.1f cycles per %d-column slice per warp; %lld MMA(K=128) issued in CTA 0 (%.0f cycles each)\n",
         name, (double)mx / iters, NCOL, h[15], h[15] ? (double)mx / h[15] : 0.0);
}

template <int MODE>
void run(const char* name, int nw, long long* d_out, float* sink) {
  const int iters = 2000;
  probe<MODE><<<148, nw * 32>>>(d_out, sink, iters);
  probe<MODE><<<148, nw * 32>>>(d_out, sink, iters);
  long long h[16];
  cudaMemcpy(h, d_out, sizeof(long long) * nw, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < nw; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-28s warps/SMSP=%d: %7.1f cycles per 128-column row slice per warp (%.1f per SMSP)\n", name, nw / 4,
         (double)mx / iters, (double)mx / iters / (nw / 4));
}

int main() {
  long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 16 * sizeof(long long));
  cudaMalloc(&sink, 148 * 512 * sizeof(float));
  for (int nw : {4, 8}) {
    run<0>("speculative EMU3", nw, d_out, sink);
    run<2>("speculative EMU0 (all MUFU)", nw, d_out, sink);
    run<3>("speculative EMU2", nw, d_out, sink);
    run<1>("tcgen05.ld only", nw, d_out, sink);
    run<4>("ld+exp2+sum (no P)", nw, d_out, sink);
  }
  run_split<64, 576>("split 64 cols, 96-reg cap", 8, d_out, sink);
  run_split<64, 256>("split 64 cols, no cap", 8, d_out, sink);
  run_split<128, 576>("128 cols, 96-reg cap", 4, d_out, sink);
  run_split<64, 256>("64 cols, 1 warp/SMSP", 4, d_out, sink);
  run_mma<128, 4, false>("128 cols x 4 warps, MMA idle", d_out, sink);
  run_mma<128, 4, true>("128 cols x 4 warps, MMA busy", d_out, sink);
  run_mma<64, 8, false>("64 cols x 8 warps, MMA idle", d_out, sink);
  run_mma<64, 8, true>("64 cols x 8 warps, MMA busy", d_out, sink);
  run_mma<128, 8, true>("128 cols x 8 warps (2 tiles), MMA busy", d_out, sink);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
