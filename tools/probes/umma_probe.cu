// tcgen05.mma throughput probe (sm_100a): one CTA per SM, one thread issues
// back-to-back kind::f16 MMAs (bf16 in, f32 accumulate in TMEM), operands
// in SWIZZLE_128B K-major shared memory (values irrelevant for timing).
//   mode 0: SS  M128 N128 K16 (the attention's S = Q K^T shape)
//   mode 1: SS  M128 N256 K16
//   mode 2: TS  M128 N128 K16 (A from TMEM, the attention's O += P V shape)
//   mode 3: blocks of 8 SS N128 then 8 TS N128 (the attention's MMA mix)
//   mode 4: mode 3 while warps 1-3 stream 16-byte st.shared (TMA-like
//           shared-memory write traffic, ~32 B/clk/SM)
//   mode 5: the attention's sequence PV0(j) S0(j+1) PV1(j) S1(j+1): S_x SS
//           N128 into TMEM [128x, +128), PV_x TS with A = P_x aliasing S_x,
//           D = O_x [256 + 128x, +128), B = V MN-major; a commit per group
//   mode 6: mode 5 with a K-major B for PV
//   mode 7: mode 5 with PV_x reading the other tile's S columns (the
//           write-after-read of S_x(j+1) over P_x(j) is 3 MMA groups away)
//   mode 8: mode 5 without the per-group commits
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int BLOCKS = 2048;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

__global__ void __launch_bounds__(128, 1) probe(int mode, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (su32(sm) + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 32768;         // A 128x128, B 256x128 (bf16)
  const uint32_t bar = base + 32768 + 65536;
  __shared__ uint32_t tptr;
  const int warp = threadIdx.x / 32;
  uint4* fill = reinterpret_cast<uint4*>(sm + (base - su32(sm)));
  for (int i = threadIdx.x; i < (32768 + 65536) / 16; i += blockDim.x) fill[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar + 8) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar + 16) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tptr)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tptr;
  volatile int* stop = reinterpret_cast<volatile int*>(sm + (base - su32(sm)) + 32768 + 65536 + 64);
  if (threadIdx.x == 0) *stop = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long c0 = clock64();
    if (mode >= 5) {
      const uint64_t qd = sdesc(sA, 16, 1024), kd = sdesc(sB, 16, 1024);
      const uint64_t vd = mode == 6 ? sdesc(sB + 32768, 16, 1024) : sdesc(sB + 32768, 16384, 1024);
      const uint32_t id_o = mode == 6 ? idesc(128) : (idesc(128) | (1u << 16));
      auto S = [&](int x) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          mma_ss(t + 128 * x, qd + off, kd + off, idesc(128), kk > 0);
        }
        if (mode != 8)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar + 8) : "memory");
      };
      auto PV = [&](int x) {
        const uint32_t a = t + 128 * (mode == 7 ? 1 - x : x);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = mode == 6 ? (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4) : (kk * 2048) >> 4;
          mma_ts(t + 256 + 128 * x, a + kk * 8, vd + off, id_o, kk > 0);
        }
        if (mode != 8)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar + 16) : "memory");
      };
      S(0);
      S(1);
      for (int blk = 0; blk < BLOCKS / 2; ++blk) {
        PV(0);
        S(0);
        PV(1);
        S(1);
      }
    }
    for (int blk = 0; blk < (mode >= 5 ? 0 : BLOCKS); ++blk) {
      if (mode == 0 || mode == 3 || mode == 4) {
        const uint64_t ad = sdesc(sA, 16, 1024), bd = sdesc(sB, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          mma_ss(t, ad + off, bd + off, idesc(128), kk > 0);
        }
      }
      if (mode == 1) {
        const uint64_t ad = sdesc(sA, 16, 1024), bd = sdesc(sB, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offa = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          const uint32_t offb = ((kk >> 2) * 32768 + (kk & 3) * 32) >> 4;
          mma_ss(t, ad + offa, bd + offb, idesc(256), kk > 0);
        }
      }
      if (mode == 2 || mode == 3 || mode == 4) {
        const uint64_t bd = sdesc(sB, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
          mma_ts(t + 256, t + 384 + kk * 8, bd + off, idesc(128), kk > 0);
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
                 "@!P1 bra W;\n\t}" ::"r"(bar) : "memory");
    const unsigned long long c1 = clock64();
    if (blockIdx.x == 0) *cyc = c1 - c0;
    *stop = 1;
  } else if (mode == 4 && warp > 0) {
    // ~32 B/clk/SM of 16-byte shared stores into B's upper half (not read by N128)
    uint4* dst = reinterpret_cast<uint4*>(sm + (base - su32(sm)) + 32768 + 32768);
    int i = threadIdx.x - 32;
    while (!*stop) {
#pragma unroll 1
      for (int r = 0; r < 64; ++r) {
        dst[(i + 96 * r) & 2047] = make_uint4(r, r, r, r);
        __nanosleep(0);
      }
      for (int w = 0; w < 20; ++w) asm volatile("nanosleep.u32 32;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t) : "memory");
  }
}

int main() {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  const int smem = 1024 + 32768 + 65536 + 128;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"SS N128", "SS N256", "TS N128", "SS128+TS128", "mix + st.shared",
                         "attn seq", "attn seq Kmaj V", "attn seq no WAR", "attn no commit"};
  const double fl[] = {2.0 * 128 * 128 * 128, 2.0 * 128 * 256 * 128, 2.0 * 128 * 128 * 128,
                       4.0 * 128 * 128 * 128, 4.0 * 128 * 128 * 128, 4.0 * 128 * 128 * 128,
                       4.0 * 128 * 128 * 128, 4.0 * 128 * 128 * 128, 4.0 * 128 * 128 * 128};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 9; ++mode) {
      probe<<<148, 128, smem>>>(mode, cyc);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      probe<<<148, 128, smem>>>(mode, cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      unsigned long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double flops = fl[mode] * BLOCKS * 148;
      printf("%-16s %.3f ms  %.0f TFLOP/s  %.0f flop/clk/SM (CTA 0: %llu clk)  err=%s\n", names[mode], ms,
             flops / ms / 1e9, fl[mode] * BLOCKS / (double)c, c, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
