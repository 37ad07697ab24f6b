// Internal declarations shared by the CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <mutex>
#include <string>

#include "modarith.cuh"

#define PDB_MAX_DIMS 16
#define PDB_SMEM_NTT_MAX 8192   // longest axis transformed in shared memory
#define PDB_MAX_ORDER 128       // largest matrix order r
#define PDB_MAX_PRIMES 256      // most primes in one CRT call

namespace pdb {

// Per-length twiddle tables of one prime (device memory).
struct Twiddles {
  int N = 0;
  uint32_t* fwd = nullptr;    // w^j, j < N/2          (w = omega_N)
  uint32_t* fwd_s = nullptr;  // Shoup companions
  uint32_t* inv = nullptr;    // w^-j, j < N/2
  uint32_t* inv_s = nullptr;
  uint32_t* full = nullptr;   // w^c, c < N (node abscissae for fused evaluation)
  uint32_t* full_s = nullptr;
  uint32_t* inv_full_n = nullptr;   // w^-c N^-1, c < N (register-radix inverse twiddles)
  uint32_t* inv_full_ns = nullptr;
  uint32_t ninv = 1, ninv_s = 0;  // N^-1 and its companion
};

// Per-length tables of a wide prime (p >= 2^31): Montgomery forms (R = 2^64).
struct Twiddles64 {
  int N = 0;
  uint64_t* fwd = nullptr;   // w^j R, j < N/2
  uint64_t* inv = nullptr;   // w^-j R
  uint64_t ninv = 0;         // N^-1 R
};

struct PrimeCtx {
  uint64_t p = 0, omega = 0;
  int q = 0;
  bool wide = false;         // p >= 2^31: the u64 kernels (wide.cu)
  Mod32 m;
  Mod64 m64;
  Twiddles64 tw64[64];
  int device = 0;
  int sms = 148;
  Twiddles tw[32];
  std::mutex lock;
};

const Twiddles* ctx_twiddles(PrimeCtx* ctx, int N);
const Twiddles64* ctx_twiddles64(PrimeCtx* ctx, int N);

// ---- one axis of a batched row-major tensor (shared by the u32 and u64 NTTs) ----
struct AxisGeom {
  int64_t inner;           // product of dims after the axis
  int32_t nbox;            // number of box dims describing active outer lines
  int64_t box_ext[PDB_MAX_DIMS + 1];   // active extent per outer dim (slowest first)
  int64_t box_dim[PDB_MAX_DIMS + 1];   // full dim per outer dim
  int64_t active_outer;    // product of box_ext
};

__device__ __forceinline__ int64_t outer_offset(int64_t c, const AxisGeom& g) {
  // compact active index -> real outer line index (mixed radix)
  int64_t off = 0, mul = 1;
  for (int d = g.nbox - 1; d >= 0; --d) {
    int64_t e = g.box_ext[d];
    int64_t i = c % e;
    c /= e;
    off += i * mul;
    mul *= g.box_dim[d];
  }
  return off;
}

__device__ __forceinline__ uint32_t bitrev(uint32_t x, int bits) {
  return bits ? (__brev(x) >> (32 - bits)) : 0u;
}


void set_error(const char* fmt, ...);
int check_launch(const char* what);
// Counts kernel launches issued by this library (pdb_launch_count()).
void count_launch(long long n = 1);
// pdb_kernel_timing: CUDA events on the launch stream around a det_gj launch
// (ktimer_start returns -1 while timing is off).
int ktimer_start(cudaStream_t st);
void ktimer_stop(int slot, cudaStream_t st);

// kept (may be null): per axis, evaluate only the kept nodes u < kept[a] of a
// pruned node set (forward sparse passes; the other outputs are not written)
int ntt_axis(PrimeCtx* ctx, uint32_t* data, int64_t batch, int nd, const int64_t* dims,
             const int64_t* ext, int axis, bool inverse, cudaStream_t st, const int64_t* kept = nullptr);

// ---- pruned node sets ----------------------------------------------------------
// The determinant is a polynomial of degree <= D_a in variable a (the plan's
// degree bound), so on an axis of N >= 16 nodes only the nodes
//     {u + (N/8) v : u < U, v < 8},   U >= floor(D_a / 8) + 1,
// need a determinant: writing f(x) = sum_{l<8} x^l g_l(x^8), every g_l has
// degree <= floor(D_a/8) < U, so its values at the first U of the N/8 points
// (w^8)^u determine the rest (expand.cu).  A NodeMap enumerates the kept nodes
// of a grid in a compact row-major order: axis a has klen[a] = 8 U_a compact
// positions k = v U_a + u (or all N_a when u[a] == 0), and full() returns the
// node's position in the full row-major grid.  nd == 0 is the identity.
#define PDB_MAP_DIMS 8
struct NodeMap {
  int32_t nd = 0;
  int32_t u[PDB_MAP_DIMS] = {};          // kept u per axis, 0 = whole axis
  int64_t klen[PDB_MAP_DIMS] = {};       // compact extent per axis
  int64_t n8[PDB_MAP_DIMS] = {};         // N_a / 8
  int64_t stride[PDB_MAP_DIMS] = {};     // row-major stride of axis a in the full grid
  int32_t small = 0;                     // full grid < 2^32 nodes: 32-bit index arithmetic
  __host__ __device__ __forceinline__ int64_t full(int64_t c) const {
    if (nd == 0) return c;
    if (!small) return full_big(c);
    uint32_t cc = (uint32_t)c, off = 0;
    for (int a = nd - 1; a >= 0; --a) {
      const uint32_t kl = (uint32_t)klen[a];
      const uint32_t k = cc % kl;
      cc /= kl;
      const uint32_t ax = u[a] ? k % (uint32_t)u[a] + (uint32_t)n8[a] * (k / (uint32_t)u[a]) : k;
      off += ax * (uint32_t)stride[a];
    }
    return off;
  }
  // grids of 2^32 nodes or more (out of line: 64-bit division)
  __host__ __device__ __noinline__ int64_t full_big(int64_t c) const {
    int64_t off = 0;
    for (int a = nd - 1; a >= 0; --a) {
      const int64_t k = c % klen[a];
      c /= klen[a];
      const int64_t ax = u[a] ? k % u[a] + n8[a] * (k / u[a]) : k;
      off += ax * stride[a];
    }
    return off;
  }
};

// ---- entry sources for the determinant kernels ---------------------------------
// Kernels index nodes in the compact space of `map` (identity: the grid);
// node(c) is the full-grid node, at(e, node) the value of entry e there.
// Staged: materialised entry grids [k][stride] (node-major within an entry).
struct StagedSrc {
  const uint32_t* grids;
  int64_t stride;
  NodeMap map;
  __device__ __forceinline__ int64_t node(int64_t c) const { return map.full(c); }
  __device__ __forceinline__ uint32_t at(int e, int64_t node) const {
    return __ldg(grids + (int64_t)e * stride + node);
  }
};

// Fused: partially transformed entries [outer][E][k] (every axis but the last
// already evaluated; E coefficient planes along the last axis; the k unique
// entries innermost, so a CTA filling its matrices reads coalesced rows).
// The value of entry e at node = o * NL + c is the degree-(E-1) polynomial in
// x = w_NL^c with coefficients part[(o*E + l)*k + e].
struct FusedSrc {
  const uint32_t* part;
  int64_t outer;
  int E;
  int k;
  int NL;
  const uint32_t* xs;    // w^c, c < NL
  const uint32_t* xss;   // companions
  uint32_t p;
  NodeMap map;
  int ulast = 0;         // kept u of the last axis (NL / 8 when it is not pruned)
  int64_t orow0 = 0;     // the launch's first compact last-axis row (node_lo / (8 ulast))
  const int64_t* orow_full = nullptr;   // pruned map: full outer index of launch row j (det scratch)
  __device__ __forceinline__ int64_t node(int64_t c) const { return map.full(c); }
  __device__ __forceinline__ uint32_t at(int e, int64_t node) const {
    int64_t o = node / NL;
    int c = (int)(node - o * NL);
    const uint32_t* a = part + o * E * (int64_t)k + e;
    uint32_t x = __ldg(xs + c), xc = __ldg(xss + c);
    uint32_t v = __ldg(a + (int64_t)(E - 1) * k);
    for (int l = E - 2; l >= 0; --l) v = add_mod(shoup_mul(v, x, xc, p), __ldg(a + (int64_t)l * k), p);
    return v;
  }
};

}  // namespace pdb
