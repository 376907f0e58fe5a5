// Pipe-throughput probe for the scorer redesign: FP32 scalar vs packed
// (f32x2) adds/FMAs, FP64, and 8-byte shared-memory exchange bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_probe fp_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

__global__ void k_ffma(float* out, float a, float b) {
  float x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], a, x[(i + 1) % CH]);
  float s = 0;
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_fadd(float* out, float a) {
  float x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = x[i] + x[(i + 3) % CH];
  float s = 0;
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *(unsigned long long*)&a, rb = *(unsigned long long*)&b,
                     rc = *(unsigned long long*)&c, rd;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *(float2*)&rd;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long ra = *(unsigned long long*)&a, rb = *(unsigned long long*)&b, rd;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
  return *(float2*)&rd;
}

__global__ void k_ffma2(float* out, float a, float b) {
  float2 x[CH];
  float2 m = make_float2(a, b);
  for (int i = 0; i < CH; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = ffma2(x[i], m, x[(i + 1) % CH]);
  float s = 0;
  for (int i = 0; i < CH; ++i) s += x[i].x + x[i].y;
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_fadd2(float* out, float a) {
  float2 x[CH];
  for (int i = 0; i < CH; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fadd2(x[i], x[(i + 3) % CH]);
  float s = 0;
  for (int i = 0; i < CH; ++i) s += x[i].x + x[i].y;
  if (s == 1.2345f) out[0] = s;
}

__global__ void k_dfma(float* out, double a) {
  double x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, x[(i + 1) % CH]);
  double s = 0;
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1.2345) out[0] = (float)s;
}

__global__ void k_dadd(float* out) {
  double x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = x[i] + x[(i + 3) % CH];
  double s = 0;
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1.2345) out[0] = (float)s;
}

// 8-byte exchange: every thread stores 16 float2 at a conflict-free pattern
// and reads back a transposed (stride) pattern.
__global__ void k_smem(float* out, int rounds) {
  extern __shared__ float2 buf[];
  const int t = threadIdx.x, nt = blockDim.x;
  float2 v[16];
  for (int i = 0; i < 16; ++i) v[i] = make_float2(t + i, i);
  for (int r = 0; r < rounds; ++r) {
#pragma unroll
    for (int i = 0; i < 16; ++i) buf[i * nt + t] = v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int idx = ((t * 16 + i) ^ (t >> 1)) % (16 * nt);
      float2 w = buf[idx];
      v[i].x += w.y;
      v[i].y += w.x;
    }
    __syncthreads();
  }
  float s = 0;
  for (int i = 0; i < 16; ++i) s += v[i].x + v[i].y;
  if (s == 1.2345f) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256;
  const double thr = (double)blocks * threads;
  auto timeit = [&](const char* name, auto launch, double ops_per_thread) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double gops = thr * ops_per_thread / (ms * 1e6);
    printf("%-10s %8.3f ms  %9.1f G lane-ops/s  = %6.1f lane-ops/clk/SM @1.965GHz\n", name,
           ms, gops, gops / (sms * 1.965));
  };
  double ops = (double)ITERS * CH;
  timeit("ffma", [&] { k_ffma<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, ops);
  timeit("fadd", [&] { k_fadd<<<blocks, threads>>>(out, 1.0f); }, ops);
  timeit("ffma2(x2)", [&] { k_ffma2<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, 2 * ops);
  timeit("fadd2(x2)", [&] { k_fadd2<<<blocks, threads>>>(out, 1.0f); }, 2 * ops);
  timeit("dfma", [&] { k_dfma<<<blocks, threads>>>(out, 1.0001); }, ops);
  timeit("dadd", [&] { k_dadd<<<blocks, threads>>>(out); }, ops);
  const int rounds = 512;
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 256 * 8);
  timeit("smem8B", [&] { k_smem<<<blocks, threads, 16 * 256 * 8>>>(out, rounds); },
         (double)rounds * 16 * 2 * 8 /*bytes*/);
  printf("(smem8B line: 'lane-ops' = bytes moved st+ld)\n");
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
