// extern "C" boundary of libpolydet_b200.so (declared in include/polydet_b200.h).
#include <atomic>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <vector>

#include "../../include/polydet_b200.h"
#include "pdb_internal.cuh"


struct pdb_prime_ctx : pdb::PrimeCtx {};

namespace pdb {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void count_launch(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ---- det kernel timing (pdb_kernel_timing): event pairs around det_gj launches ----
static std::mutex g_kt_lock;
static bool g_kt_on = false;
static std::vector<cudaEvent_t> g_kt_events;   // start, stop, start, stop, ...
static size_t g_kt_used = 0;

int ktimer_start(cudaStream_t st) {
  std::lock_guard<std::mutex> guard(g_kt_lock);
  if (!g_kt_on) return -1;
  while (g_kt_events.size() < g_kt_used + 2) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    g_kt_events.push_back(e);
  }
  const int slot = (int)g_kt_used;
  g_kt_used += 2;
  cudaEventRecord(g_kt_events[slot], st);
  return slot;
}

void ktimer_stop(int slot, cudaStream_t st) {
  if (slot < 0) return;
  std::lock_guard<std::mutex> guard(g_kt_lock);
  cudaEventRecord(g_kt_events[slot + 1], st);
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return -1;
  }
  return 0;
}

static uint64_t mulmod64(uint64_t a, uint64_t b, uint64_t p) {
  return (uint64_t)((unsigned __int128)a * b % p);
}

static uint64_t powmod64(uint64_t a, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  a %= p;
  while (e) {
    if (e & 1) r = mulmod64(r, a, p);
    a = mulmod64(a, a, p);
    e >>= 1;
  }
  return r;
}

const Twiddles* ctx_twiddles(PrimeCtx* ctx, int N) {
  if (N < 1 || (N & (N - 1))) {
    set_error("unsupported length: %d is not a power of two", N);
    return nullptr;
  }
  const int l = 31 - __builtin_clz((unsigned)N);
  if (l > ctx->q) {
    set_error("unsupported length: %d exceeds 2^%d for p=%llu", N, ctx->q, (unsigned long long)ctx->p);
    return nullptr;
  }
  std::lock_guard<std::mutex> guard(ctx->lock);
  Twiddles& T = ctx->tw[l];
  if (T.N == N) return &T;
  const uint64_t p = ctx->p;
  const uint64_t w = powmod64(ctx->omega, 1ull << (ctx->q - l), p);
  const uint64_t wi = powmod64(w, p - 2, p);
  const int half = N / 2 > 0 ? N / 2 : 1;
  std::vector<uint32_t> host((size_t)4 * half + 4 * (size_t)N);
  uint32_t* f = host.data();
  uint32_t* fs = f + half;
  uint32_t* iv = fs + half;
  uint32_t* is = iv + half;
  uint32_t* full = is + half;
  uint32_t* fulls = full + N;
  uint64_t a = 1, b = 1;
  for (int j = 0; j < half; ++j) {
    f[j] = (uint32_t)a;
    fs[j] = shoup_companion((uint32_t)a, (uint32_t)p);
    iv[j] = (uint32_t)b;
    is[j] = shoup_companion((uint32_t)b, (uint32_t)p);
    a = mulmod64(a, w, p);
    b = mulmod64(b, wi, p);
  }
  uint64_t c = 1;
  for (int j = 0; j < N; ++j) {
    full[j] = (uint32_t)c;
    fulls[j] = shoup_companion((uint32_t)c, (uint32_t)p);
    c = mulmod64(c, w, p);
  }
  // w^-j * N^-1, j < N (the register-radix inverse folds N^-1 into its twiddles)
  uint32_t* invn = fulls + N;
  uint32_t* invns = invn + N;
  const uint64_t ninv = powmod64((uint64_t)N % p, p - 2, p);
  uint64_t d = ninv;
  for (int j = 0; j < N; ++j) {
    invn[j] = (uint32_t)d;
    invns[j] = shoup_companion((uint32_t)d, (uint32_t)p);
    d = mulmod64(d, wi, p);
  }
  uint32_t* dev = nullptr;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaMalloc(&dev, host.size() * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemcpy(dev, host.data(), host.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("twiddle table allocation: %s", cudaGetErrorString(e));
    return nullptr;
  }
  T.fwd = dev;
  T.fwd_s = dev + half;
  T.inv = dev + 2 * half;
  T.inv_s = dev + 3 * half;
  T.full = dev + 4 * half;
  T.full_s = dev + 4 * half + N;
  T.inv_full_n = dev + 4 * half + 2 * N;
  T.inv_full_ns = dev + 4 * half + 3 * N;
  T.ninv = (uint32_t)powmod64((uint64_t)N % p, p - 2, p);
  T.ninv_s = shoup_companion(T.ninv, (uint32_t)p);
  T.N = N;
  return &T;
}

size_t det_scratch_bytes(int r, int64_t nodes);
template <class Src>
int det_run(PrimeCtx* ctx, Src src, const int32_t* ids, int r, int64_t node_lo, int64_t nodes,
            uint32_t* out, void* scratch, size_t scratch_bytes, cudaStream_t st);
int reduce_scatter(PrimeCtx* ctx, const uint32_t* mag, const uint8_t* neg, const int64_t* pos,
                   int64_t count, int Lc, uint32_t* dst, cudaStream_t st);
int condense_run(PrimeCtx* ctx, const uint32_t* mat, int r, uint32_t* trail_vals, int32_t* trail_cols,
                 uint32_t* det_out, void* scratch, size_t scratch_bytes, cudaStream_t st);
size_t crt_scratch_bytes(int P);
size_t crt_nonzero_scratch_bytes(int64_t n);
int crt_nonzero(const uint32_t* res, int P, int64_t n, int64_t stride, int64_t* index, int64_t* count,
                void* scratch, size_t scratch_bytes, cudaStream_t st);
int limbs_to_digits(const uint32_t* limbs, int64_t count, int width, int64_t ls, uint32_t* digits, int D,
                    uint8_t* ndig, int sms, cudaStream_t st);
int crt_mrc_sel(const uint32_t* res, int P, const int64_t* index, int64_t count, int64_t res_stride,
                const uint32_t* primes_host, uint32_t* limbs, int L, uint8_t* neg, int32_t* width, int sms,
                cudaStream_t st);
int crt_limbs(int P);
int grid_interpolate(PrimeCtx* ctx, uint32_t* compact, uint32_t* scratch, uint32_t* grid, const NodeMap& map,
                     const int64_t* dims, const int64_t* box, cudaStream_t st);
int grid_expand(PrimeCtx* ctx, const uint32_t* compact, uint32_t* grid, const NodeMap& map, const int64_t* dims,
                cudaStream_t st);
void expand_release(const PrimeCtx* ctx);

// C-ABI node map -> device NodeMap (validated); false + error text when invalid.
static bool make_node_map(const pdb_node_map* in, NodeMap* out, int64_t* size) {
  *out = NodeMap{};
  if (!in || in->ndim == 0) {
    *size = -1;   // identity: caller's node count
    return true;
  }
  if (in->ndim < 0 || in->ndim > PDB_MAP_DIMS) {
    set_error("node map rank %d outside 1..%d", in->ndim, PDB_MAP_DIMS);
    return false;
  }
  out->nd = in->ndim;
  int64_t stride = 1, n = 1;
  for (int a = in->ndim - 1; a >= 0; --a) {
    const int64_t N = in->dims[a];
    const int U = in->kept_u[a];
    if (N < 1 || (N & (N - 1))) {
      set_error("node map axis %d: %lld is not a power of two", a, (long long)N);
      return false;
    }
    if (U != 0 && (N < 16 || U < 1 || 8ll * U >= N)) {
      set_error("node map axis %d: kept u %d invalid for length %lld", a, U, (long long)N);
      return false;
    }
    out->u[a] = U;
    out->n8[a] = N / 8;
    out->klen[a] = U ? 8ll * U : N;
    out->stride[a] = stride;
    stride *= N;
    n *= out->klen[a];
  }
  out->small = stride < (1ll << 32);
  *size = n;
  return true;
}

int crt_mrc(const uint32_t* res, int P, int64_t n, int64_t res_stride, const uint32_t* primes_host,
            uint32_t* limbs, int L, uint8_t* neg, void* scratch, size_t scratch_bytes, int sms,
            cudaStream_t st);

// ---- peak microbenchmark kernels (same primitives as the det kernels) --------
__global__ void peak_shoup(uint32_t* out, uint32_t seed, uint32_t w, uint32_t ws, uint32_t p, int iters) {
  uint32_t a[8], x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = (seed + threadIdx.x * 8 + i) % p; x[i] = (seed * 3 + i) % p; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a[i] = sub_mod(a[i], shoup_mul(x[i], w, ws, p), p);   // a -= w * x   (mul-mod + sub-mod)
      x[i] ^= a[i] & 1;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void peak_delayed(uint32_t* out, uint32_t seed, Mod32 m, int iters) {
  uint32_t a[4], tau[8], np[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = (seed + threadIdx.x * 4 + i) % m.p;
#pragma unroll
  for (int q = 0; q < 8; ++q) { tau[q] = (seed * (q + 3)) % m.p; np[q] = (seed * (q + 7) + threadIdx.x) % m.p; }
  for (int it = 0; it < iters; ++it) {
    uint64_t acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = (uint64_t)a[i] * np[i];
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = mad_wide(tau[q], np[q] ^ i, acc[i]);
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = csub(csub(redc(acc[i], m), 2u * m.p), m.p);
    // the multipliers depend on this iteration's results, so no product can be
    // hoisted out of the loop (an earlier version let the compiler do exactly
    // that and over-stated the peak)
#pragma unroll
    for (int q = 0; q < 8; ++q) tau[q] = a[q & 3] ^ q;
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// The raw integer-multiplier ceiling: a stream of independent accumulating
// 32x32->64 IMAD.WIDE (8 chains per thread; the multiplier changes every
// iteration so no product can be hoisted).
__global__ void peak_imadwide(uint32_t* out, uint32_t seed, int iters) {
  uint64_t acc[8];
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i] = i; x[i] = seed * (i + 1) + threadIdx.x; }
  uint32_t y = seed ^ (threadIdx.x * 2654435761u);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = mad_wide(x[i], y, acc[i]);
    y += 0x9e3779b9u;
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)(s ^ (s >> 32));
}

}  // namespace pdb

using namespace pdb;

extern "C" {

const char* pdb_last_error(void) { return g_err; }
int32_t pdb_version(void) { return 1; }
int64_t pdb_launch_count(void) { return g_launches.load(); }

int32_t pdb_device_sm_count(int32_t device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    set_error("no CUDA device %d", device);
    return -1;
  }
  return v;
}

int32_t pdb_prime_ctx_create(uint64_t p, uint64_t omega, int32_t q, pdb_prime_ctx** out) {
  if (!out) { set_error("null output pointer"); return -2; }
  if (p < 2 || p >= (1ull << 62)) {
    set_error("modulus %llu outside the kernel range (p < 2^62)", (unsigned long long)p);
    return -2;
  }
  const bool wide = p >= (1ull << 31);
  if (wide && !(p & 1)) { set_error("wide modulus %llu must be odd", (unsigned long long)p); return -2; }
  if (q < 0 || q > (wide ? 62 : 30) || omega >= p) { set_error("invalid prime spec"); return -2; }
  auto* c = new pdb_prime_ctx();
  c->p = p;
  c->omega = omega;
  c->q = q;
  c->wide = wide;
  if (wide) c->m64 = make_mod64(p);
  else c->m = make_mod32((uint32_t)p);
  cudaGetDevice(&c->device);
  int sms = pdb_device_sm_count(c->device);
  c->sms = sms > 0 ? sms : 148;
  *out = c;
  return 0;
}

int32_t pdb_prime_ctx_create_wide(uint64_t p, uint64_t omega, int32_t q, pdb_prime_ctx** out) {
  // a u64-kernel context for any odd prime (mixed prime sets share one residue width)
  if (!out) { set_error("null output pointer"); return -2; }
  if (p < 3 || !(p & 1) || p >= (1ull << 62)) {
    set_error("wide context needs an odd modulus 3 <= p < 2^62, got %llu", (unsigned long long)p);
    return -2;
  }
  if (q < 0 || q > 62 || omega >= p) { set_error("invalid prime spec"); return -2; }
  auto* c = new pdb_prime_ctx();
  c->p = p;
  c->omega = omega;
  c->q = q;
  c->wide = true;
  c->m64 = make_mod64(p);
  cudaGetDevice(&c->device);
  int sms = pdb_device_sm_count(c->device);
  c->sms = sms > 0 ? sms : 148;
  *out = c;
  return 0;
}

int32_t pdb_prime_ctx_destroy(pdb_prime_ctx* ctx) {
  if (!ctx) return 0;
  expand_release(ctx);
  for (auto& T : ctx->tw)
    if (T.fwd) cudaFree(T.fwd);
  for (auto& T : ctx->tw64)
    if (T.fwd) cudaFree(T.fwd);
  delete ctx;
  return 0;
}

int32_t pdb_prime_ctx_prepare(pdb_prime_ctx* ctx, int64_t n) {
  if (!ctx) { set_error("null context"); return -2; }
  if (ctx->wide) return ctx_twiddles64(ctx, (int)n) ? 0 : -2;
  return ctx_twiddles(ctx, (int)n) ? 0 : -2;
}

// the u32 entry points take contexts of primes < 2^31 only
static bool narrow_ctx(const pdb_prime_ctx* ctx) {
  if (!ctx) { set_error("null context"); return false; }
  if (ctx->wide) { set_error("context holds a prime >= 2^31: use the _u64 entry points"); return false; }
  return true;
}

int32_t pdb_ntt_multi_u32(pdb_prime_ctx* ctx, uint32_t* data, int64_t batch, int32_t ndim,
                          const int64_t* dims, const int64_t* extents, uint32_t axis_mask,
                          int32_t inverse, void* stream) {
  if (!narrow_ctx(ctx)) return -2;
  if (ndim < 0 || ndim > PDB_MAX_DIMS || batch < 0) { set_error("invalid NTT arguments"); return -2; }
  for (int a = 0; a < ndim; ++a)
    if ((axis_mask >> a) & 1)
      if (!ctx_twiddles(ctx, (int)dims[a])) return -2;
  if (batch == 0) return 0;
  for (int a = ndim - 1; a >= 0; --a) {
    if (!((axis_mask >> a) & 1)) continue;
    int rc = ntt_axis(ctx, data, batch, ndim, dims, extents, a, inverse != 0, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return 0;
}

int32_t pdb_ntt_forward_kept_u32(pdb_prime_ctx* ctx, uint32_t* data, int64_t batch, int32_t ndim,
                                 const int64_t* dims, const int64_t* extents, const int64_t* kept_u,
                                 uint32_t axis_mask, void* stream) {
  if (!narrow_ctx(ctx)) return -2;
  if (ndim < 0 || ndim > PDB_MAX_DIMS || batch < 0 || !kept_u) { set_error("invalid NTT arguments"); return -2; }
  for (int a = 0; a < ndim; ++a) {
    if (kept_u[a] < 0 || (kept_u[a] > 0 && (dims[a] < 16 || 8 * kept_u[a] >= dims[a]))) {
      set_error("kept u %lld invalid for axis %d of length %lld", (long long)kept_u[a], a, (long long)dims[a]);
      return -2;
    }
    if ((axis_mask >> a) & 1)
      if (!ctx_twiddles(ctx, (int)dims[a])) return -2;
  }
  if (batch == 0) return 0;
  for (int a = ndim - 1; a >= 0; --a) {
    if (!((axis_mask >> a) & 1)) continue;
    int rc = ntt_axis(ctx, data, batch, ndim, dims, extents, a, false, (cudaStream_t)stream, kept_u);
    if (rc) return rc;
  }
  return 0;
}

int32_t pdb_reduce_scatter_u32(pdb_prime_ctx* ctx, const uint32_t* mag, const uint8_t* neg,
                               const int64_t* pos, int64_t count, int32_t limbs, uint32_t* dst,
                               void* stream) {
  if (!narrow_ctx(ctx)) return -2;
  if (limbs < 1) { set_error("invalid reduce arguments"); return -2; }
  return reduce_scatter(ctx, mag, neg, pos, count, limbs, dst, (cudaStream_t)stream);
}

size_t pdb_det_scratch_bytes(int32_t r, int64_t nodes) { return det_scratch_bytes(r, nodes); }

int32_t pdb_det_batch_u32(pdb_prime_ctx* ctx, const uint32_t* grids, int64_t grid_stride,
                          const int32_t* entry_ids, int32_t r, int64_t node_lo, int64_t nodes,
                          uint32_t* out, void* scratch, size_t scratch_bytes, void* stream) {
  if (!narrow_ctx(ctx)) return -2;
  StagedSrc src{grids, grid_stride};
  return det_run(ctx, src, entry_ids, r, node_lo, nodes, out, scratch, scratch_bytes, (cudaStream_t)stream);
}

int32_t pdb_eval_det_fused_u32(pdb_prime_ctx* ctx, const uint32_t* partial, int64_t outer,
                               int32_t ncoef, int32_t entries, int32_t n_last, const int32_t* entry_ids, int32_t r,
                               int64_t node_lo, int64_t nodes, uint32_t* out, void* scratch,
                               size_t scratch_bytes, void* stream) {
  if (!narrow_ctx(ctx)) return -2;
  if (ncoef < 1 || entries < 1) { set_error("invalid fused arguments"); return -2; }
  const Twiddles* T = ctx_twiddles(ctx, n_last);
  if (!T) return -2;
  FusedSrc src{partial, outer, ncoef, entries, n_last, T->full, T->full_s, ctx->m.p};
  src.ulast = n_last / 8;
  if (src.ulast > 0) src.orow0 = node_lo / (8 * (int64_t)src.ulast);
  return det_run(ctx, src, entry_ids, r, node_lo, nodes, out, scratch, scratch_bytes, (cudaStream_t)stream);
}

int64_t pdb_node_map_size(const pdb_node_map* map) {
  NodeMap nm;
  int64_t n = 0;
  if (!map) { set_error("null node map"); return -2; }
  if (!make_node_map(map, &nm, &n)) return -2;
  if (n < 0) {
    n = 1;
    for (int a = 0; a < map->ndim; ++a) n *= map->dims[a];
  }
  return n;
}

int32_t pdb_det_batch_map_u32(pdb_prime_ctx* ctx, const uint32_t* grids, int64_t grid_stride,
                              const int32_t* entry_ids, int32_t r, const pdb_node_map* map,
                              int64_t node_lo, int64_t nodes, uint32_t* out, void* scratch,
                              size_t scratch_bytes, void* stream) {
  if (!narrow_ctx(ctx)) return -2;
  StagedSrc src{grids, grid_stride};
  int64_t n = 0;
  if (!make_node_map(map, &src.map, &n)) return -2;
  if (n >= 0 && (node_lo < 0 || node_lo + nodes > n)) { set_error("node range outside the node map"); return -2; }
  return det_run(ctx, src, entry_ids, r, node_lo, nodes, out, scratch, scratch_bytes, (cudaStream_t)stream);
}

int32_t pdb_eval_det_fused_map_u32(pdb_prime_ctx* ctx, const uint32_t* partial, int64_t outer,
                                   int32_t ncoef, int32_t entries, int32_t n_last,
                                   const int32_t* entry_ids, int32_t r, const pdb_node_map* map,
                                   int64_t node_lo, int64_t nodes, uint32_t* out, void* scratch,
                                   size_t scratch_bytes, void* stream) {
  if (!narrow_ctx(ctx)) return -2;
  if (ncoef < 1 || entries < 1) { set_error("invalid fused arguments"); return -2; }
  const Twiddles* T = ctx_twiddles(ctx, n_last);
  if (!T) return -2;
  FusedSrc src{partial, outer, ncoef, entries, n_last, T->full, T->full_s, ctx->m.p};
  int64_t n = 0;
  if (!make_node_map(map, &src.map, &n)) return -2;
  src.ulast = n_last / 8;
  if (n >= 0) {
    int64_t full = 1;
    for (int a = 0; a < map->ndim; ++a) full *= map->dims[a];
    if (full != outer * n_last || map->dims[map->ndim - 1] != n_last) {
      set_error("node map shape does not match outer x n_last");
      return -2;
    }
    if (node_lo < 0 || node_lo + nodes > n) { set_error("node range outside the node map"); return -2; }
    if (src.map.u[map->ndim - 1]) src.ulast = src.map.u[map->ndim - 1];
  }
  if (src.ulast > 0) src.orow0 = node_lo / (8 * (int64_t)src.ulast);
  return det_run(ctx, src, entry_ids, r, node_lo, nodes, out, scratch, scratch_bytes, (cudaStream_t)stream);
}

int32_t pdb_grid_interpolate_u32(pdb_prime_ctx* ctx, uint32_t* compact, uint32_t* scratch, uint32_t* grid,
                                 const pdb_node_map* map, const int64_t* box, void* stream) {
  if (!narrow_ctx(ctx)) return -2;
  NodeMap nm;
  int64_t n = 0;
  if (!map || map->ndim == 0 || !box) { set_error("grid_interpolate needs a pruned node map and a box"); return -2; }
  if (!make_node_map(map, &nm, &n)) return -2;
  return grid_interpolate(ctx, compact, scratch, grid, nm, map->dims, box, (cudaStream_t)stream);
}

int32_t pdb_grid_expand_u32(pdb_prime_ctx* ctx, const uint32_t* compact, uint32_t* grid,
                            const pdb_node_map* map, void* stream) {
  if (!narrow_ctx(ctx)) return -2;
  NodeMap nm;
  int64_t n = 0;
  if (!map || map->ndim == 0) { set_error("grid_expand needs a pruned node map"); return -2; }
  if (!make_node_map(map, &nm, &n)) return -2;
  for (int a = 0; a < map->ndim; ++a)
    if (map->kept_u[a] && !ctx_twiddles(ctx, (int)map->dims[a])) return -2;
  return grid_expand(ctx, compact, grid, nm, map->dims, (cudaStream_t)stream);
}

int32_t pdb_condense_u32(pdb_prime_ctx* ctx, const uint32_t* mat, int32_t r, uint32_t* trail_vals,
                         int32_t* trail_cols, uint32_t* det_out, void* scratch, size_t scratch_bytes,
                         void* stream) {
  if (!narrow_ctx(ctx)) return -2;
  return condense_run(ctx, mat, r, trail_vals, trail_cols, det_out, scratch, scratch_bytes,
                      (cudaStream_t)stream);
}

int32_t pdb_crt_limbs(int32_t nprimes) { return crt_limbs(nprimes); }
size_t pdb_crt_scratch_bytes(int32_t nprimes) { return crt_scratch_bytes(nprimes); }

int32_t pdb_crt_mrc_u32(const uint32_t* residues, int32_t nprimes, int64_t n, int64_t stride,
                        const uint32_t* primes, uint32_t* limbs, int32_t L, uint8_t* neg,
                        void* scratch, size_t scratch_bytes, void* stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = pdb_device_sm_count(dev);
  return crt_mrc(residues, nprimes, n, stride, primes, limbs, L, neg, scratch, scratch_bytes,
                 sms > 0 ? sms : 148, (cudaStream_t)stream);
}

size_t pdb_crt_nonzero_scratch_bytes(int64_t n) { return crt_nonzero_scratch_bytes(n); }

int32_t pdb_crt_nonzero_u32(const uint32_t* residues, int32_t nprimes, int64_t n, int64_t stride,
                            int64_t* index, int64_t* count, void* scratch, size_t scratch_bytes,
                            void* stream) {
  return crt_nonzero(residues, nprimes, n, stride, index, count, scratch, scratch_bytes, (cudaStream_t)stream);
}

int32_t pdb_crt_mrc_sel_u32(const uint32_t* residues, int32_t nprimes, int64_t stride,
                            const uint32_t* primes, const int64_t* index, int64_t count, uint32_t* limbs,
                            int32_t L, uint8_t* neg, int32_t* width, void* stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = pdb_device_sm_count(dev);
  return crt_mrc_sel(residues, nprimes, index, count, stride, primes, limbs, L, neg, width, sms > 0 ? sms : 148,
                     (cudaStream_t)stream);
}

int32_t pdb_limbs_to_digits30(const uint32_t* limbs, int64_t count, int32_t width, int64_t stride,
                              uint32_t* digits, int32_t ndigits, uint8_t* digit_count, void* stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = pdb_device_sm_count(dev);
  return limbs_to_digits(limbs, count, width, stride, digits, ndigits, digit_count, sms > 0 ? sms : 148,
                         (cudaStream_t)stream);
}

int32_t pdb_kernel_timing(int32_t enable) {
  std::lock_guard<std::mutex> guard(g_kt_lock);
  g_kt_on = enable != 0;
  g_kt_used = 0;
  return 0;
}

int32_t pdb_kernel_timing_read(double* ms, int64_t* launches) {
  if (!ms || !launches) { set_error("null output pointer"); return -2; }
  std::lock_guard<std::mutex> guard(g_kt_lock);
  double total = 0;
  for (size_t i = 0; i + 1 < g_kt_used; i += 2) {
    if (cudaEventSynchronize(g_kt_events[i + 1]) != cudaSuccess) return check_launch("kernel timing");
    float t = 0;
    cudaEventElapsedTime(&t, g_kt_events[i], g_kt_events[i + 1]);
    total += t;
  }
  *ms = total;
  *launches = (int64_t)(g_kt_used / 2);
  return 0;
}

int32_t pdb_mulmod_peak(uint32_t p, int32_t variant, double* ups, void* stream) {
  if (p < 3 || p >= (1u << 30) || !ups) { set_error("peak needs 2 < p < 2^30"); return -2; }
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = pdb_device_sm_count(dev);
  const int threads = 256, blocks = sms * 8, iters = 4096;
  uint32_t* d = nullptr;
  if (cudaMalloc(&d, sizeof(uint32_t) * threads * blocks) != cudaSuccess) return check_launch("peak alloc");
  Mod32 m = make_mod32(p);
  const uint32_t w = 123456789u % p, ws = shoup_companion(w, p);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, st);
    if (variant == 0) peak_shoup<<<blocks, threads, 0, st>>>(d, 12345u + rep, w, ws, p, iters);
    else if (variant == 1) peak_delayed<<<blocks, threads, 0, st>>>(d, 12345u + rep, m, iters / 8);
    else peak_imadwide<<<blocks, threads, 0, st>>>(d, 12345u + rep, iters);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double per_thread = variant == 0 ? 8.0 * iters : (variant == 1 ? 4.0 * 9 * (iters / 8) : 8.0 * iters);
  *ups = per_thread * threads * blocks / (best * 1e-3);
  return check_launch("peak");
}

}  // extern "C"
