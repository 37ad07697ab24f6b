// Issue rates of the multiply forms the det kernel can use, alone and mixed
// (is the FP64 pipe a second multiplier next to the IMAD.WIDE one?).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pipes pipes.cu && ./pipes
// Reported: thread-operations per clock per SM (at the attribute clock).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ILP = 8;
constexpr int ITERS = 2048;

#define LOOP(body)                                   \
  for (int it = 0; it < ITERS; ++it) {               \
    _Pragma("unroll") for (int i = 0; i < ILP; ++i) { body; } \
  }

__global__ void k_imadwide(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t lo[ILP], hi[ILP];
  const uint32_t x = a0 ^ threadIdx.x, y = b0 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) { lo[i] = i; hi[i] = 0; }
  LOOP(asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo[i]), "+r"(hi[i]) : "r"(x + i), "r"(y)));
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= lo[i] ^ hi[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// loop-invariant operands: nothing but the accumulating IMAD.WIDE in the loop
__global__ void k_imadwide_pure(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t lo[ILP], hi[ILP], x[ILP];
  const uint32_t y = b0 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) { lo[i] = i; hi[i] = 0; x[i] = (a0 ^ threadIdx.x) + i; }
  LOOP(asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo[i]), "+r"(hi[i]) : "r"(x[i]), "r"(y)));
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= lo[i] ^ hi[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// IMAD.WIDE interleaved 1:1 with IMAD.HI / with IMAD (loop-invariant operands)
template <int KIND>
__global__ void k_wide_plus(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t lo[ILP], hi[ILP], x[ILP], z[ILP];
  const uint32_t y = b0 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) { lo[i] = i; hi[i] = 0; x[i] = (a0 ^ threadIdx.x) + i; z[i] = i * 7; }
  LOOP(asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo[i]), "+r"(hi[i]) : "r"(x[i]), "r"(y));
       if (KIND == 0) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(z[i]) : "r"(y));
       else if (KIND == 1) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(z[i]) : "r"(y));
       else asm volatile("add.u32 %0, %0, %1;" : "+r"(z[i]) : "r"(y)));
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= lo[i] ^ hi[i] ^ z[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// one operand uniform (kernel parameter -> uniform register)
__global__ void k_wide_uniform(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t lo[ILP], hi[ILP], x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { lo[i] = i; hi[i] = 0; x[i] = (a0 ^ threadIdx.x) + i; }
  LOOP(asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo[i]), "+r"(hi[i]) : "r"(x[i]), "r"(b0)));
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= lo[i] ^ hi[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// the trailing-update tile shape: acc[a][b] += x[a] * y[b], 2 x 4, x[a] shared by 4 consecutive MACs
__global__ void k_wide_tile(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t lo[2][4], hi[2][4], x[2][8], y[8][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) { lo[a][b] = a + b; hi[a][b] = 0; }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    x[0][q] = (a0 ^ threadIdx.x) + q; x[1][q] = (a0 ^ threadIdx.x) * 3 + q;
#pragma unroll
    for (int b = 0; b < 4; ++b) y[q][b] = b0 + threadIdx.x * (b + 1) + q;
  }
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;"
                       : "+r"(lo[a][b]), "+r"(hi[a][b]) : "r"(x[a][q]), "r"(y[q][b]));
  }
  uint32_t s = 0;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) s ^= lo[a][b] ^ hi[a][b];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imadhi(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t v[ILP];
  const uint32_t y = b0 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = a0 + i;
  LOOP(asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(v[i]) : "r"(y)));
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imadlo(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t v[ILP];
  const uint32_t y = b0 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = a0 + i;
  LOOP(asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(v[i]) : "r"(y)));
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(uint32_t* out, uint32_t a0, uint32_t b0) {
  double v[ILP];
  const double y = 1.0 + 1e-9 * threadIdx.x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = a0 + i;
  LOOP(asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(v[i]) : "d"(y)));
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)s;
}

__global__ void k_ffma(uint32_t* out, uint32_t a0, uint32_t b0) {
  float v[ILP];
  const float y = 1.0f + 1e-7f * threadIdx.x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = a0 + i;
  LOOP(asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(v[i]) : "f"(y)));
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)s;
}

// IMAD.WIDE chains and DFMA chains interleaved 1:1
__global__ void k_mix(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t lo[ILP], hi[ILP];
  double v[ILP];
  const uint32_t x = a0 ^ threadIdx.x, y = b0 + threadIdx.x;
  const double yd = 1.0 + 1e-9 * threadIdx.x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) { lo[i] = i; hi[i] = 0; v[i] = a0 + i; }
  LOOP(asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo[i]), "+r"(hi[i]) : "r"(x + i), "r"(y));
       asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(v[i]) : "d"(yd)));
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= lo[i] ^ hi[i] ^ (uint32_t)v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// IMAD.WIDE chains and plain IADD3 (alu) interleaved 1:1
__global__ void k_mix_alu(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t lo[ILP], hi[ILP], z[ILP];
  const uint32_t x = a0 ^ threadIdx.x, y = b0 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < ILP; ++i) { lo[i] = i; hi[i] = 0; z[i] = i * 3; }
  LOOP(asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo[i]), "+r"(hi[i]) : "r"(x + i), "r"(y));
       asm volatile("add.u32 %0, %0, %1;" : "+r"(z[i]) : "r"(y)));
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= lo[i] ^ hi[i] ^ z[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  uint32_t* d;
  const int blocks = sms * 8, threads = 256;
  cudaMalloc(&d, sizeof(uint32_t) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern) {
    kern<<<blocks, threads>>>(d, 3u, 0x9e3779b9u);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(d, 3u, 0x9e3779b9u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double ops = (double)ITERS * ILP * blocks * threads;
    printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"ops_per_clk_sm\": %.2f}\n", name, best,
           ops / (best * 1e-3) / (sms * (double)khz * 1e3));
  };
  run("imad.wide (acc)", k_imadwide);
  run("imad.wide pure (loop-invariant operands)", k_imadwide_pure);
  run("imad.wide, one operand uniform", k_wide_uniform);
  run("imad.wide 2x4 tile pattern (x[a] shared by 4 MACs)", k_wide_tile);
  run("imad.wide + imad.hi pairs", k_wide_plus<0>);
  run("imad.wide + imad pairs", k_wide_plus<1>);
  run("imad.wide + iadd pairs (invariant operands)", k_wide_plus<2>);
  run("imad.hi", k_imadhi);
  run("imad.lo", k_imadlo);
  run("dfma", k_dfma);
  run("ffma", k_ffma);
  run("imad.wide + dfma pairs", k_mix);
  run("imad.wide + iadd pairs", k_mix_alu);
  printf("{\"sm_clock_khz\": %d, \"sms\": %d}\n", khz, sms);
  cudaFree(d);
  return 0;
}
