// Issue/pipe throughput of the softmax's instruction types on sm_100a: cycles per warp-instruction
// per SMSP with W warps per SMSP, 8 independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__device__ __forceinline__ void op(uint32_t& a, uint32_t& b, uint32_t c) {
  if constexpr (OP == 0) {  // FFMA2
    asm volatile("{.reg .b64 x, y, z;\n\tmov.b64 x, {%0, %1};\n\tmov.b64 z, {%2, %2};\n\t"
                 "fma.rn.ftz.f32x2 x, x, z, z;\n\tmov.b64 {%0, %1}, x;}"
                 : "+r"(a), "+r"(b) : "r"(c));
  } else if constexpr (OP == 1) {  // FADD2
    asm volatile("{.reg .b64 x, z;\n\tmov.b64 x, {%0, %1};\n\tmov.b64 z, {%2, %2};\n\t"
                 "add.rn.ftz.f32x2 x, x, z;\n\tmov.b64 {%0, %1}, x;}"
                 : "+r"(a), "+r"(b) : "r"(c));
  } else if constexpr (OP == 2) {  // F2FP bf16x2 pack
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(a) : "f"(__uint_as_float(b)), "f"(__uint_as_float(a)));
    b ^= c;
  } else if constexpr (OP == 3) {  // MUFU.EX2
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(a));
    b += c;
  } else if constexpr (OP == 4) {  // FFMA (scalar)
    asm volatile("fma.rn.ftz.f32 %0, %0, %2, %2;\n\tfma.rn.ftz.f32 %1, %1, %2, %2;" : "+r"(a), "+r"(b) : "r"(c));
  } else if constexpr (OP == 5) {  // FMNMX
    asm volatile("max.ftz.f32 %0, %0, %2;\n\tmax.ftz.f32 %1, %1, %2;" : "+r"(a), "+r"(b) : "r"(c));
  } else if constexpr (OP == 6) {  // SHL + IADD (exponent insert)
    asm volatile("{.reg .b32 t;\n\tshl.b32 t, %1, 23;\n\tadd.s32 %0, %0, t;}" : "+r"(a) : "r"(b));
    b += c;
  }
}

template <int OP>
__global__ void k(uint32_t* out, long long* cyc, int iters) {
  uint32_t a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x + i; b[i] = threadIdx.x * 3 + i; }
  const uint32_t c = 0x3f000001u + (blockIdx.x & 1);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) op<OP>(a[i], b[i], c);
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] ^ b[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
void run(const char* name, int instr_per_op) {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  for (int w : {1, 4}) {
    k<OP><<<148, 128 * w>>>(out, cyc, iters);
    k<OP><<<148, 128 * w>>>(out, cyc, iters);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double n = (double)iters * 8 * instr_per_op * w;  // warp-instructions of this type per SMSP
    printf("%-10s %d warps/SMSP: %.2f cycles per warp-instruction per SMSP\n", name, w, h / n);
  }
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("FFMA2", 1);
  run<1>("FADD2", 1);
  run<2>("F2FP", 1);
  run<3>("MUFU.EX2", 1);
  run<4>("FFMA", 2);
  run<5>("FMNMX", 2);
  run<6>("SHL+IADD", 2);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
