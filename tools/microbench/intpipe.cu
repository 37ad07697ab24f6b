// Integer-pipe microbenchmarks for the mod-p update primitives on sm_100a.
//
// Establishes the measured P_upd denominator used by bench.py's roofline
// (SURVEY.md §8(d) "measured: a mulmod_peak microbenchmark of the identical
// update primitive with full ILP and no memory traffic").
//
// Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o intpipe intpipe.cu
// Run:    ./intpipe   (prints one JSON object)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
#define ITERS 2048

__global__ void k_imad(uint32_t* out, uint32_t a0, uint32_t b) {
  uint32_t a[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = a0 + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = a[i] * b + 0x9e3779b9u;
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imadhi(uint32_t* out, uint32_t a0, uint32_t b) {
  uint32_t a[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = a0 + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = __umulhi(a[i], b) ^ a[i];
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imadwide(uint32_t* out, uint32_t a0, uint32_t b) {
  uint64_t acc[ILP];
  uint32_t x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { acc[i] = a0 + i; x[i] = a0 ^ (threadIdx.x + i); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] += (uint64_t)x[i] * b;
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] += 1;  // keeps products distinct
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= (uint32_t)acc[i] ^ (uint32_t)(acc[i] >> 32);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Shoup update: a <- a - x*w mod p, lazily kept in [0, 2p) (p < 2^30).
__global__ void k_shoup(uint32_t* out, uint32_t a0, uint32_t w, uint32_t wp, uint32_t p) {
  uint32_t a[ILP], x[ILP];
  const uint32_t p2 = 2 * p;
#pragma unroll
  for (int i = 0; i < ILP; ++i) { a[i] = (a0 + threadIdx.x + i) % p; x[i] = (a0 * 7 + i) % p; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      uint32_t q = __umulhi(x[i], wp);
      uint32_t r = x[i] * w - q * p;           // [0, 2p)
      uint32_t t = a[i] + p2 - r;              // (0, 4p)
      uint32_t t2 = t - p2;
      a[i] = min(t, t2);                       // [0, 2p)
      x[i] = a[i];
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Delayed reduction: 8 u32*u32 MACs into u64, then one reduction mod p.
__global__ void k_delayed(uint32_t* out, uint32_t a0, uint32_t p, uint32_t c32, uint32_t c32p) {
  uint32_t a[ILP], l[8], u[8];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = (a0 + threadIdx.x + i) % p;
#pragma unroll
  for (int t = 0; t < 8; ++t) { l[t] = (a0 * (t + 3)) % p; u[t] = (a0 * (t + 11) + threadIdx.x) % p; }
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      uint64_t acc = a[i];
#pragma unroll
      for (int t = 0; t < 8; ++t) acc += (uint64_t)l[t] * (u[t] ^ i);
      uint32_t hi = (uint32_t)(acc >> 32), lo = (uint32_t)acc;
      uint32_t q = __umulhi(hi, c32p);
      uint32_t r = hi * c32 - q * p;           // hi*2^32 mod p in [0, 2p)
      uint32_t s1 = lo % 1u;                   // placeholder (no-op)
      uint32_t v = r + (lo - (lo >= 2 * p ? 2 * p : 0)) + s1;
      v = min(v, v - 2 * p);
      a[i] = min(v, v - p);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, double a0, double b) {
  double a[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = a0 + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, 0.5);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  int sms = prop.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int threads = 256, per_sm = 8;
  const int blocks = sms * per_sm;
  const long long nthreads = (long long)threads * blocks;
  uint32_t* d_out; double* d_dout;
  cudaMalloc(&d_out, nthreads * 4);
  cudaMalloc(&d_dout, nthreads * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const uint32_t p = 1000000513u;
  const uint32_t w = 123456789u;
  const uint32_t wp = (uint32_t)(((uint64_t)w << 32) / p);
  const uint32_t c32 = (uint32_t)((1ull << 32) % p);
  const uint32_t c32p = (uint32_t)(((uint64_t)c32 << 32) / p);
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk_khz);
  auto run = [&](const char* name, double ops_per_thread, auto launch) {
    launch();  // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    double ops = ops_per_thread * nthreads;
    double per_s = ops / (best * 1e-3);
    printf(", \"%s\": {\"ms\": %.4f, \"ops_per_s\": %.4e, \"ops_per_clk_sm_at_1965\": %.2f}", name, best,
           per_s, per_s / (sms * 1.965e9));
  };
  run("imad", (double)ITERS * ILP, [&] { k_imad<<<blocks, threads>>>(d_out, 3u, 0x01000193u); });
  run("imad_hi", (double)ITERS * ILP, [&] { k_imadhi<<<blocks, threads>>>(d_out, 3u, 0x9e3779b9u); });
  run("imad_wide_mac", (double)ITERS * ILP, [&] { k_imadwide<<<blocks, threads>>>(d_out, 3u, 0x9e3779b9u); });
  run("shoup_update", (double)ITERS * ILP, [&] { k_shoup<<<blocks, threads>>>(d_out, 12345u, w, wp, p); });
  run("delayed8_mac", (double)(ITERS / 8) * ILP * 8, [&] { k_delayed<<<blocks, threads>>>(d_out, 12345u, p, c32, c32p); });
  run("dfma", (double)ITERS * ILP, [&] { k_dfma<<<blocks, threads>>>(d_dout, 1.0, 0.999); });
  printf("}\n");
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
