// Issue cost of the 64-bit multiply-accumulate forms on sm_100a.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mac mac.cu && ./mac
// Each kernel runs ILP independent accumulator chains per thread; the reported
// figure is MACs per clock per SM at the measured SM clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ILP = 8;
constexpr int ITERS = 4096;

// (a) mad.wide.u32 (ptxas may split it into IMAD.WIDE + IADD3/IADD3.X)
__global__ void k_madwide(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint64_t acc[ILP];
  uint32_t x[ILP], b[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { acc[i] = a0 + i; x[i] = a0 ^ (threadIdx.x * 3 + i); b[i] = b0 + i * 7; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(x[i]), "r"(b[i]));
    }
#pragma unroll
    for (int i = 0; i < ILP; ++i) b[i] ^= (uint32_t)acc[(i + 1) % ILP];
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= (uint32_t)acc[i] ^ (uint32_t)(acc[i] >> 32);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// (b) carry-chained 32-bit halves: mad.lo.cc + madc.hi
__global__ void k_madcc(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t lo[ILP], hi[ILP], x[ILP], b[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { lo[i] = a0 + i; hi[i] = 0; x[i] = a0 ^ (threadIdx.x * 3 + i); b[i] = b0 + i * 7; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;"
                   : "+r"(lo[i]), "+r"(hi[i]) : "r"(x[i]), "r"(b[i]));
    }
#pragma unroll
    for (int i = 0; i < ILP; ++i) b[i] ^= lo[(i + 1) % ILP];
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= lo[i] ^ hi[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// (c) the T-pass shape: 8 products into one accumulator, then REDC + 2 csubs
__global__ void k_tpass(uint32_t* out, uint32_t a0, uint32_t p, uint32_t qinv) {
  uint32_t a[4], t[8], n[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = (a0 + threadIdx.x * 4 + i) % p;
#pragma unroll
  for (int q = 0; q < 8; ++q) { t[q] = (a0 * (q + 3)) % p; n[q] = (a0 * (q + 7) + threadIdx.x) % p; }
  for (int it = 0; it < ITERS / 8; ++it) {
    uint64_t acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = (uint64_t)a[i] * n[i];
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] += (uint64_t)t[q] * (n[q] ^ i);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t mq = (uint32_t)acc[i] * qinv;
      uint32_t v = (uint32_t)(acc[i] >> 32) + p - __umulhi(mq, p);
      v = min(v, v - 2 * p);
      a[i] = min(v, v - p);
    }
    // loop-carried multipliers: otherwise the compiler hoists the 32 products
    // t[q] * (n[q] ^ i) out of the loop and the figure is meaningless
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = a[q & 3] ^ q;
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  uint32_t* d;
  const int blocks = sms * 8, threads = 256;
  cudaMalloc(&d, sizeof(uint32_t) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, double macs_per_thread, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double ops = macs_per_thread * blocks * threads;
    printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"mac_per_clk_sm\": %.2f}\n", name, best,
           ops / (best * 1e-3) / (sms * (double)khz * 1e3));
  };
  run("mad.wide.u32", (double)ITERS * ILP, [&] { k_madwide<<<blocks, threads>>>(d, 3u, 0x9e3779b9u); });
  run("mad.lo.cc+madc.hi", (double)ITERS * ILP, [&] { k_madcc<<<blocks, threads>>>(d, 3u, 0x9e3779b9u); });
  const uint32_t p = 1000000513u;
  uint32_t inv = 1;
  for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
  run("tpass 9 MAC + REDC (per MAC)", (double)(ITERS / 8) * 4 * 9, [&] { k_tpass<<<blocks, threads>>>(d, 3u, p, inv); });
  cudaFree(d);
  return 0;
}
