// Is the FP64 pipe a usable second multiplier next to IMAD.WIDE on B200?
// Exact integer products on the FP64 pipe: a (30-bit) split into 15-bit halves,
// a_h * b and a_l * b (< 2^45) accumulate exactly in doubles (< 2^53).
// Each kernel runs the trailing-update tile shape (operands re-read from shared
// memory every step, as in det_gj) and reports MACs per clock per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64mix fp64mix.cu && ./fp64mix
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 1024;

__device__ __forceinline__ uint64_t madw(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t r;
  asm("{\n\t.reg .u32 lo, hi;\n\tmov.b64 {lo, hi}, %3;\n\t"
      "mad.lo.cc.u32 lo, %1, %2, lo;\n\tmadc.hi.u32 hi, %1, %2, hi;\n\tmov.b64 %0, {lo, hi};\n\t}"
      : "=l"(r) : "r"(a), "r"(b), "l"(c));
  return r;
}

// integer tile TRxTC: acc[a][b] += x[a][q] * y[q][b]
template <int TR, int TC>
__global__ void k_int(uint32_t* out) {
  __shared__ uint32_t sx[64][8], sy[64][8];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) { sx[i / 8][i % 8] = i * 2654435761u >> 2; sy[i / 8][i % 8] = i * 40503u; }
  __syncthreads();
  uint64_t acc[TR][TC] = {};
  const int l = threadIdx.x & 31;
  for (int it = 0; it < ITERS; ++it) {
    const int row = (it + l) & 63;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t x[TR], y[TC];
#pragma unroll
      for (int a = 0; a < TR; ++a) x[a] = sx[(row + a * 8 + q) & 63][q];
#pragma unroll
      for (int b = 0; b < TC; ++b) y[b] = sy[(row + q) & 63][b];
#pragma unroll
      for (int a = 0; a < TR; ++a)
#pragma unroll
        for (int b = 0; b < TC; ++b) acc[a][b] = madw(x[a], y[b], acc[a][b]);
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) s ^= acc[a][b];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)s ^ (uint32_t)(s >> 32);
}

// FP64 tile: x split into halves (doubles in smem), y as doubles: 2 DFMA per MAC
template <int TR, int TC>
__global__ void k_fp(uint32_t* out) {
  __shared__ double sxh[64][8], sxl[64][8], sy[64][8];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    const uint32_t v = i * 2654435761u >> 2;
    sxh[i / 8][i % 8] = (double)(v >> 15); sxl[i / 8][i % 8] = (double)(v & 0x7fff); sy[i / 8][i % 8] = (double)(i * 40503u);
  }
  __syncthreads();
  double ah[TR][TC] = {}, al[TR][TC] = {};
  const int l = threadIdx.x & 31;
  for (int it = 0; it < ITERS; ++it) {
    const int row = (it + l) & 63;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      double xh[TR], xl[TR], y[TC];
#pragma unroll
      for (int a = 0; a < TR; ++a) { xh[a] = sxh[(row + a * 8 + q) & 63][q]; xl[a] = sxl[(row + a * 8 + q) & 63][q]; }
#pragma unroll
      for (int b = 0; b < TC; ++b) y[b] = sy[(row + q) & 63][b];
#pragma unroll
      for (int a = 0; a < TR; ++a)
#pragma unroll
        for (int b = 0; b < TC; ++b) { ah[a][b] = fma(xh[a], y[b], ah[a][b]); al[a][b] = fma(xl[a], y[b], al[a][b]); }
    }
    if ((it & 7) == 7) {   // keep the sums exact: fold every 8 steps (64 products < 2^51)
#pragma unroll
      for (int a = 0; a < TR; ++a)
#pragma unroll
        for (int b = 0; b < TC; ++b) { ah[a][b] = ah[a][b] * 0.5; al[a][b] = al[a][b] * 0.5; }
    }
  }
  double s = 0;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) s += ah[a][b] + al[a][b];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)(uint64_t)s;
}

// both: integer TRxTC tile and FP64 TRxTF tile in the same loop (different columns)
template <int TR, int TC, int TF>
__global__ void k_mix(uint32_t* out) {
  __shared__ uint32_t sx[64][8], sy[64][8];
  __shared__ double sxh[64][8], sxl[64][8], syd[64][8];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    const uint32_t v = i * 2654435761u >> 2;
    sx[i / 8][i % 8] = v; sy[i / 8][i % 8] = i * 40503u;
    sxh[i / 8][i % 8] = (double)(v >> 15); sxl[i / 8][i % 8] = (double)(v & 0x7fff); syd[i / 8][i % 8] = (double)(i * 40503u);
  }
  __syncthreads();
  uint64_t acc[TR][TC] = {};
  double ah[TR][TF] = {}, al[TR][TF] = {};
  const int l = threadIdx.x & 31;
  for (int it = 0; it < ITERS; ++it) {
    const int row = (it + l) & 63;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t x[TR], y[TC];
      double xh[TR], xl[TR], yd[TF];
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        x[a] = sx[(row + a * 8 + q) & 63][q];
        xh[a] = sxh[(row + a * 8 + q) & 63][q]; xl[a] = sxl[(row + a * 8 + q) & 63][q];
      }
#pragma unroll
      for (int b = 0; b < TC; ++b) y[b] = sy[(row + q) & 63][b];
#pragma unroll
      for (int b = 0; b < TF; ++b) yd[b] = syd[(row + q) & 63][b + 4];
#pragma unroll
      for (int a = 0; a < TR; ++a) {
#pragma unroll
        for (int b = 0; b < TC; ++b) acc[a][b] = madw(x[a], y[b], acc[a][b]);
#pragma unroll
        for (int b = 0; b < TF; ++b) { ah[a][b] = fma(xh[a], yd[b], ah[a][b]); al[a][b] = fma(xl[a], yd[b], al[a][b]); }
      }
    }
    if ((it & 7) == 7) {
#pragma unroll
      for (int a = 0; a < TR; ++a)
#pragma unroll
        for (int b = 0; b < TF; ++b) { ah[a][b] = ah[a][b] * 0.5; al[a][b] = al[a][b] * 0.5; }
    }
  }
  uint64_t s = 0;
  double d = 0;
#pragma unroll
  for (int a = 0; a < TR; ++a) {
#pragma unroll
    for (int b = 0; b < TC; ++b) s ^= acc[a][b];
#pragma unroll
    for (int b = 0; b < TF; ++b) d += ah[a][b] + al[a][b];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)s ^ (uint32_t)(s >> 32) ^ (uint32_t)(uint64_t)d;
}

// raw streams with loop-invariant operands: W IMAD.WIDE and F DFMA per step (8 chains each)
template <int W, int F>
__global__ void k_raw(uint32_t* out, uint32_t a0, uint32_t b0) {
  uint32_t lo[8], hi[8], x[8];
  double v[8];
  const uint32_t y = b0 + threadIdx.x;
  const double yd = 1.0 + 1e-9 * threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) { lo[i] = i; hi[i] = 0; x[i] = (a0 ^ threadIdx.x) + i; v[i] = a0 + i; }
  for (int it = 0; it < ITERS * 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int w = 0; w < W; ++w)
        asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo[i]), "+r"(hi[i]) : "r"(x[i]), "r"(y));
#pragma unroll
      for (int f = 0; f < F; ++f) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(v[i]) : "d"(yd));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= lo[i] ^ hi[i] ^ (uint32_t)v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  uint32_t* d;
  const int threads = 256;
  cudaMalloc(&d, sizeof(uint32_t) * sms * 8 * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, double macs_per_thread, int ctas_per_sm, auto kern, auto... args) {
    const int blocks = sms * ctas_per_sm;
    kern<<<blocks, threads>>>(d, args...);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("{\"kernel\": \"%s\", \"error\": \"%s\"}\n", name, cudaGetErrorString(e)); return; }
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(d, args...);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double ops = macs_per_thread * blocks * threads;
    printf("{\"kernel\": \"%s\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"mac_per_clk_sm\": %.2f}\n", name, ctas_per_sm, best,
           ops / (best * 1e-3) / (sms * (double)khz * 1e3));
  };
  const double T = (double)ITERS * 8;
  for (int c : {2, 4}) {
    run("int 2x4", T * 8, c, k_int<2, 4>);
    run("int 2x8", T * 16, c, k_int<2, 8>);
    run("fp64 2x4 (2 DFMA/MAC)", T * 8, c, k_fp<2, 4>);
    run("fp64 2x2", T * 4, c, k_fp<2, 2>);
    run("mix int 2x4 + fp64 2x2", T * 12, c, k_mix<2, 4, 2>);
    run("mix int 2x4 + fp64 2x4", T * 16, c, k_mix<2, 4, 4>);
    run("mix int 2x2 + fp64 2x2", T * 8, c, k_mix<2, 2, 2>);
    run("mix int 2x4 + fp64 2x1", T * 10, c, k_mix<2, 4, 1>);
  }
  const double R = (double)ITERS * 4 * 8;
  run("raw W1 F0 (IMAD.WIDE per clk)", R, 8, k_raw<1, 0>, 3u, 0x9e3779b9u);
  run("raw W0 F1 (DFMA per clk)", R, 8, k_raw<0, 1>, 3u, 0x9e3779b9u);
  run("raw W1 F1 (IMAD.WIDE per clk)", R, 8, k_raw<1, 1>, 3u, 0x9e3779b9u);
  run("raw W1 F2 (IMAD.WIDE per clk)", R, 8, k_raw<1, 2>, 3u, 0x9e3779b9u);
  run("raw W1 F3 (IMAD.WIDE per clk)", R, 8, k_raw<1, 3>, 3u, 0x9e3779b9u);
  run("raw W1 F4 (IMAD.WIDE per clk)", R, 8, k_raw<1, 4>, 3u, 0x9e3779b9u);
  run("raw W2 F2 (IMAD.WIDE/2 per clk)", R * 2, 8, k_raw<2, 2>, 3u, 0x9e3779b9u);
  printf("{\"sm_clock_khz\": %d, \"sms\": %d}\n", khz, sms);
  cudaFree(d);
  return 0;
}
