// Throughput of legacy integer MMA (mma.sync m16n8k32 u8 x u8 -> s32) on sm_100a,
// alone and interleaved with IMAD.WIDE, to size a tensor-core trailing update.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o imma imma.cu && ./imma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8;       // independent accumulator chains per warp
constexpr int ITERS = 1024;

__device__ __forceinline__ void mma_u8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void k_imma(int* out, uint32_t s) {
  int acc[CH][4] = {};
  uint32_t a = s ^ threadIdx.x, b = s * 3 + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) mma_u8(acc[c], a + c, a ^ c, a - c, a * 3, b + c, b ^ c);
  }
  int t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) t += acc[c][0] ^ acc[c][1] ^ acc[c][2] ^ acc[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

// one MMA + 16 IMAD.WIDE per chain step
__global__ void k_mix(int* out, uint32_t s) {
  int acc[CH][4] = {};
  uint32_t lo[8], hi[8];
  uint32_t a = s ^ threadIdx.x, b = s * 3 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) { lo[i] = i; hi[i] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      mma_u8(acc[c], a + c, a ^ c, a - c, a * 3, b + c, b ^ c);
#pragma unroll
      for (int i = 0; i < 2; ++i)
        asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo[(c * 2 + i) & 7]), "+r"(hi[(c * 2 + i) & 7]) : "r"(a + i), "r"(b));
    }
  }
  int t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) t += acc[c][0] ^ acc[c][1] ^ acc[c][2] ^ acc[c][3];
#pragma unroll
  for (int i = 0; i < 8; ++i) t ^= lo[i] ^ hi[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  int* d;
  const int blocks = sms * 4, threads = 256;
  cudaMalloc(&d, sizeof(int) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, double per_warp_iter) {
    kern<<<blocks, threads>>>(d, 7u);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(d, 7u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double warps = (double)blocks * threads / 32;
    const double mmas = warps * ITERS * CH;
    printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"mma_per_clk_sm\": %.3f, \"int8_macs_per_clk_sm\": %.1f, \"err\": \"%s\"}\n",
           name, best, mmas / (best * 1e-3) / (sms * (double)khz * 1e3),
           mmas * 16 * 8 * 32 / (best * 1e-3) / (sms * (double)khz * 1e3), cudaGetErrorString(cudaGetLastError()));
    (void)per_warp_iter;
  };
  run("imma m16n8k32 u8", k_imma, 0);
  run("imma + 2 imad.wide per mma", k_mix, 0);
  cudaFree(d);
  return 0;
}
