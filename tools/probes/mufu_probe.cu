// MUFU exp2 throughput probe (sm_100a): f32 ex2.approx vs packed f16x2 / bf16x2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_probe mufu_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

constexpr int ITERS = 4096, CH = 8;

__global__ void k_f32(float* out, float seed) {
  float x[CH];
  for (int c = 0; c < CH; ++c) x[c] = seed * (threadIdx.x + c) * 1e-6f - 1.f;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
  float s = 0;
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_f16x2(float* out, float seed) {
  uint32_t x[CH];
  for (int c = 0; c < CH; ++c) {
    __half2 h = __floats2half2_rn(seed * (threadIdx.x + c) * 1e-6f - 1.f, -0.5f);
    x[c] = *reinterpret_cast<uint32_t*>(&h);
  }
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[c]));
  float s = 0;
  for (int c = 0; c < CH; ++c) s += __half2float(reinterpret_cast<__half2*>(&x[c])->x);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_bf16x2(float* out, float seed) {
  uint32_t x[CH];
  for (int c = 0; c < CH; ++c) {
    __nv_bfloat162 h = __floats2bfloat162_rn(seed * (threadIdx.x + c) * 1e-6f - 1.f, -0.5f);
    x[c] = *reinterpret_cast<uint32_t*>(&h);
  }
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x[c]));
  float s = 0;
  for (int c = 0; c < CH; ++c) s += __bfloat162float(reinterpret_cast<__nv_bfloat162*>(&x[c])->x);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(float* out, float seed) {
  float x[CH];
  for (int c = 0; c < CH; ++c) x[c] = seed * (threadIdx.x + c) * 1e-6f;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A800000;" : "+f"(x[c]));
  float s = 0;
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float seed) {
  unsigned long long x[CH];
  for (int c = 0; c < CH; ++c) {
    float a = seed * (threadIdx.x + c) * 1e-6f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[c]) : "f"(a), "f"(a));
  }
  unsigned long long m, k;
  asm("mov.b64 %0, {%1, %2};" : "=l"(m) : "f"(0.99999994f), "f"(0.99999994f));
  asm("mov.b64 %0, {%1, %2};" : "=l"(k) : "f"(0.0009765625f), "f"(0.0009765625f));
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(m), "l"(k));
  float s = 0;
  for (int c = 0; c < CH; ++c) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x[c]));
    s += a + b;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K k, int elems_per_op, float* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 4, threads = 256;
  k<<<blocks, threads>>>(out, 1.f);
  cudaEventRecord(a);
  k<<<blocks, threads>>>(out, 1.f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ops = (double)blocks * threads * ITERS * CH;
  printf("%-8s %.3f ms  %.1f Gop/s  %.1f G elem/s\n", name, ms, ops / ms / 1e6,
         ops * elems_per_op / ms / 1e6);
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 4 * 256 * 4);
  for (int r = 0; r < 2; ++r) {
    run("f32", k_f32, 1, out);
    run("f16x2", k_f16x2, 2, out);
    run("bf16x2", k_bf16x2, 2, out);
    run("ffma", k_ffma, 1, out);
    run("ffma2", k_ffma2, 2, out);
  }
  printf("(MUFU ex2 at 16 lanes/clk/SM x 148 SMs x 1.9 GHz = %.0f G op/s; FFMA at 128 = %.0f)\n",
         16 * 148 * 1.9, 128 * 148 * 1.9);
  return 0;
}
