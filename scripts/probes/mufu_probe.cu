// MUFU.EX2 / softmax-mix throughput probe (sm_100a).  Prints cycles per warp-instruction per SMSP
// for: ex2 with W warps per SMSP, and a softmax-like element mix with 1 and 2 warps per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_probe mufu_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int CH>
__global__ void ex2_kernel(float* out, long long* cyc, int iters) {
  float v[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) v[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) v[i] = ex2(v[i]) - 1.0f;
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

// softmax-like: per pair of elements: FFMA2 (x*s - m), 2x MUFU, FADD2 (sum), F2FP (pack)
__global__ void mix_kernel(float* out, long long* cyc, int iters, float sl2, float nm) {
  float a[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) a[i] = 0.01f * (threadIdx.x ^ i);
  float l0 = 0, l1 = 0, l2 = 0, l3 = 0;
  unsigned pk = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 64; i += 2) {
      float x0 = fmaf(a[i], sl2, nm), x1 = fmaf(a[i + 1], sl2, nm);
      float e0 = ex2(x0), e1 = ex2(x1);
      if (i & 2) { l0 += e0; l1 += e1; } else { l2 += e0; l3 += e1; }
      unsigned r;
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(e1), "f"(e0));
      pk ^= r;
    }
    nm += 1e-7f;
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l0 + l1 + l2 + l3 + (float)pk;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  long long h;
  const int iters = 4096;
  for (int wps : {1, 2, 4, 8}) {
    int thr = 128 * wps;
    ex2_kernel<16><<<148, thr>>>(out, cyc, iters);
    ex2_kernel<16><<<148, thr>>>(out, cyc, iters);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double instr_per_smsp = (double)iters * 16 * wps;  // warp-instructions of ex2 per SMSP
    printf("ex2: %d warps/SMSP: %.2f cycles per warp-ex2 per SMSP (%.1f lanes/clk/SM)\n", wps, h / instr_per_smsp,
           4 * 32 / (h / instr_per_smsp));
  }
  for (int wps : {1, 2, 4}) {
    int thr = 128 * wps;
    mix_kernel<<<148, thr>>>(out, cyc, iters, 1.44f, -3.0f);
    mix_kernel<<<148, thr>>>(out, cyc, iters, 1.44f, -3.0f);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double elems_per_thread = (double)iters * 64;
    printf("mix: %d warps/SMSP: %.2f cycles per 32 elements per SMSP (per warp: %.2f)\n", wps,
           h / (elems_per_thread * wps / 32), h / (elems_per_thread / 32));
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
