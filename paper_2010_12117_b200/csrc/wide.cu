// The wide path: primes 2^31 <= p < 2^62.
//
// The reference serves these with int64 arrays up to 3.04e9 and Python
// object arrays up to 2^62 (tensor.py:152-154, modular.py:15-19); its tests
// run whole pipelines, workspaces, NTTs, determinants and CRTs at
// prime_start = 2^61 (test_pipeline.py:149-153, test_workspace.py:179-189,
// test_transform.py:221-230, test_determinant.py:105-114, test_crt.py:147-153).
// Here they are u64 residues on the GPU with Montgomery arithmetic (R = 2^64,
// modarith.cuh:mont64); there is no CPU fallback.  These kernels are simple
// (global-memory radix-2 NTT, one warp per matrix elimination in shared memory
// with the reference's pivot rule, one thread per coefficient CRT): the wide
// path is for exactness at large moduli, not the throughput configuration.
#include <vector>

#include "../../include/polydet_b200.h"
#include "pdb_internal.cuh"

struct pdb_prime_ctx : pdb::PrimeCtx {};

namespace pdb {

static uint64_t hmul(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)((unsigned __int128)a * b % p); }
static uint64_t hpow(uint64_t a, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  a %= p;
  while (e) {
    if (e & 1) r = hmul(r, a, p);
    a = hmul(a, a, p);
    e >>= 1;
  }
  return r;
}
static uint64_t hmont(uint64_t x, uint64_t p) { return (uint64_t)(((unsigned __int128)x << 64) % p); }

const Twiddles64* ctx_twiddles64(PrimeCtx* ctx, int N) {
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
  Twiddles64& T = ctx->tw64[l];
  if (T.N == N) return &T;
  const uint64_t p = ctx->p;
  const uint64_t w = hpow(ctx->omega, 1ull << (ctx->q - l), p);
  const uint64_t wi = hpow(w, p - 2, p);
  const int half = N / 2 > 0 ? N / 2 : 1;
  std::vector<uint64_t> host(2 * (size_t)half);
  uint64_t a = 1, b = 1;
  for (int j = 0; j < half; ++j) {
    host[j] = hmont(a, p);
    host[half + j] = hmont(b, p);
    a = hmul(a, w, p);
    b = hmul(b, wi, p);
  }
  uint64_t* dev = nullptr;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaMalloc(&dev, host.size() * sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMemcpy(dev, host.data(), host.size() * sizeof(uint64_t), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("twiddle table allocation: %s", cudaGetErrorString(e));
    return nullptr;
  }
  T.fwd = dev;
  T.inv = dev + half;
  T.ninv = hmont(hpow((uint64_t)N % p, p - 2, p), p);
  T.N = N;
  return &T;
}

// ---- NTT: bit reversal + log2 N radix-2 stages in global memory -------------
__global__ void ntt64_bitrev(uint64_t* __restrict__ data, AxisGeom g, int N, int logN) {
  const int64_t total = g.active_outer * g.inner * (int64_t)N;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t line = w / N;
    const int n = (int)(w % N);
    const int rn = (int)bitrev((uint32_t)n, logN);
    if (rn <= n) continue;
    const int64_t oc = line / g.inner, t = line % g.inner;
    const int64_t base = outer_offset(oc, g) * (int64_t)N * g.inner + t;
    const uint64_t a = data[base + (int64_t)n * g.inner];
    data[base + (int64_t)n * g.inner] = data[base + (int64_t)rn * g.inner];
    data[base + (int64_t)rn * g.inner] = a;
  }
}

__global__ void ntt64_stage(uint64_t* __restrict__ data, AxisGeom g, int N, int h, const uint64_t* __restrict__ tw,
                            Mod64 m, int scale, uint64_t ninv) {
  const int64_t total = g.active_outer * g.inner * (int64_t)(N / 2);
  const int stride = N / (2 * h);
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t line = w / (N / 2);
    const int j = (int)(w % (N / 2));
    const int64_t oc = line / g.inner, t = line % g.inner;
    const int64_t base = outer_offset(oc, g) * (int64_t)N * g.inner + t;
    const int q = j & (h - 1);
    const int a = ((j - q) << 1) + q;
    const int64_t ia = base + (int64_t)a * g.inner, ib = ia + (int64_t)h * g.inner;
    const uint64_t u = data[ia];
    const uint64_t v = mont64(data[ib], tw[q * stride], m);   // x * w^q (w in Montgomery form)
    uint64_t ra = add_mod64(u, v, m.p), rb = sub_mod64(u, v, m.p);
    if (scale) {
      ra = mont64(ra, ninv, m);
      rb = mont64(rb, ninv, m);
    }
    data[ia] = ra;
    data[ib] = rb;
  }
}

static int ntt64_axis(PrimeCtx* ctx, uint64_t* data, int64_t batch, int nd, const int64_t* dims,
                      const int64_t* ext, int axis, bool inverse, cudaStream_t st) {
  const int N = (int)dims[axis];
  if (N == 1) return 0;
  const Twiddles64* T = ctx_twiddles64(ctx, N);
  if (!T) return -2;
  AxisGeom g;
  g.inner = 1;
  for (int d = axis + 1; d < nd; ++d) g.inner *= dims[d];
  g.nbox = axis + 1;
  g.box_dim[0] = batch;
  g.box_ext[0] = batch;
  for (int d = 0; d < axis; ++d) {
    g.box_dim[d + 1] = dims[d];
    g.box_ext[d + 1] = ext ? ext[d] : dims[d];
  }
  g.active_outer = 1;
  for (int d = 0; d < g.nbox; ++d) g.active_outer *= g.box_ext[d];
  if (g.active_outer == 0 || g.inner == 0) return 0;
  const int logN = 31 - __builtin_clz((unsigned)N);
  const int64_t total = g.active_outer * g.inner * (int64_t)N;
  int grid = (int)((total / 2 + 255) / 256);
  if (grid > ctx->sms * 32) grid = ctx->sms * 32;
  if (grid < 1) grid = 1;
  ntt64_bitrev<<<grid, 256, 0, st>>>(data, g, N, logN);
  for (int h = 1; h < N; h <<= 1)
    ntt64_stage<<<grid, 256, 0, st>>>(data, g, N, h, inverse ? T->inv : T->fwd, ctx->m64,
                                      inverse && h == N / 2, T->ninv);
  count_launch(1 + logN);
  return check_launch("ntt64");
}

// ---- coefficients -> residues ----------------------------------------------
__global__ void reduce_scatter64_kernel(const uint32_t* __restrict__ mag, const uint8_t* __restrict__ negs,
                                        const int64_t* __restrict__ pos, int64_t count, int Lc,
                                        uint64_t* __restrict__ dst, Mod64 m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t v = 0;   // Horner over the 32-bit limbs, plain residues: v <- v * 2^32 + limb
    for (int l = Lc - 1; l >= 0; --l) v = add_mod64(mont64(v, m.r96, m), mag[i * Lc + l] % m.p, m.p);
    if (negs[i] && v) v = m.p - v;
    dst[pos[i]] = v;
  }
}

// ---- determinants: the reference's exact rule (determinant.py:136-169) ------
// One warp per matrix in shared memory (Montgomery forms): row i's pivot is its
// first nonzero column (ballots), the rows below get the division-free update
// z*row_k - t*row_i in parallel over (row, column) pairs with the multiplier
// column saved first; det = prod z / prod z^(r-1-i) * (-1)^(inversions).
struct Staged64 {
  const uint64_t* grids;
  int64_t stride;
};

constexpr int DET64_WARPS = 4;

__global__ void __launch_bounds__(32 * DET64_WARPS)
det64_kernel(Staged64 src, const int32_t* __restrict__ ids, int r, int64_t node_lo, int64_t nodes,
             uint64_t* __restrict__ out, Mod64 m, uint64_t* __restrict__ trail_vals, int32_t* __restrict__ trail_cols) {
  extern __shared__ uint64_t wsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* A = wsm + (size_t)warp * (r * r + r);
  uint64_t* T = A + r * r;
  const uint64_t p = m.p;
  const int wpc = blockDim.x >> 5;
  const int64_t wstride = (int64_t)gridDim.x * wpc;
  for (int64_t idx = blockIdx.x * (int64_t)wpc + warp; idx < nodes; idx += wstride) {
    const int64_t node = node_lo + idx;
    for (int e = lane; e < r * r; e += 32) A[e] = to_mont64(src.grids[(int64_t)ids[e] * src.stride + node] % p, m);
    __syncwarp();
    uint64_t pre = m.r1, infl = m.r1;
    uint64_t used0 = 0, used1 = 0;   // pivot columns so far (r <= 128)
    int parity = 0;
    bool alive = true;
    for (int i = 0; i < r; ++i) {
      const uint64_t* row = A + i * r;
      int c = -1;
      for (int j0 = 0; j0 < r && c < 0; j0 += 32) {
        const unsigned nz = __ballot_sync(0xffffffffu, j0 + lane < r && row[j0 + lane] != 0);
        if (nz) c = j0 + __ffs(nz) - 1;
      }
      if (c < 0) { alive = false; break; }
      const uint64_t z = row[c];
      if (trail_vals && lane == 0) { trail_vals[i] = from_mont64(z, m); trail_cols[i] = c; }
      // earlier pivot columns to the right of c flip the permutation sign
      parity ^= (c < 64 ? __popcll(used0 >> c) + __popcll(used1) : __popcll(used1 >> (c - 64))) & 1;
      if (c < 64) used0 |= 1ull << c;
      else used1 |= 1ull << (c - 64);
      pre = mont64(pre, z, m);
      if (i + 1 < r) infl = mont64(infl, pre, m);
      const int rows = r - 1 - i;
      for (int k = lane; k < rows; k += 32) T[k] = A[(i + 1 + k) * r + c];
      __syncwarp();
      for (int w = lane; w < rows * r; w += 32) {
        const int kk = w / r, j = w - (w / r) * r;
        uint64_t* a = A + (i + 1 + kk) * r + j;
        *a = sub_mod64(mont64(z, *a, m), mont64(T[kk], row[j], m), p);
      }
      __syncwarp();
    }
    if (lane == 0) {
      uint64_t det = 0;
      if (alive) {
        det = from_mont64(mont64(pre, mont_pow64(infl, p - 2, m), m), m);
        if (parity && det) det = p - det;
      }
      out[idx] = det;
    }
    __syncwarp();
  }
}

// ---- CRT over up to PDB_MAX_PRIMES primes < 2^62 ------------------------------
struct Crt64Prime {
  Mod64 m;
  uint64_t cR;   // c_i = (m_i mod p_i)^-1, Montgomery form
};

__global__ void __launch_bounds__(64)
crt64_kernel(const uint64_t* __restrict__ res, int P, int64_t n, int64_t stride, const Crt64Prime* __restrict__ primes,
             const uint64_t* __restrict__ wR, const uint64_t* __restrict__ prod, int L64, int L,
             uint32_t* __restrict__ limbs, uint8_t* __restrict__ neg) {
  uint64_t alpha[PDB_MAX_PRIMES];
  uint64_t acc[PDB_MAX_PRIMES + 1];
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < n; pos += (int64_t)gridDim.x * blockDim.x) {
    for (int i = 0; i < P; ++i) {
      const Mod64 m = primes[i].m;
      uint64_t x = res[(int64_t)i * stride + pos];
      for (int j = 0; j < i; ++j) x = sub_mod64(x, mont64(alpha[j], wR[i * P + j], m), m.p);
      alpha[i] = i ? mont64(x, primes[i].cR, m) : x;
    }
    int len = 1;   // X in base 2^64 limbs
    acc[0] = alpha[P - 1];
    for (int i = P - 2; i >= 0; --i) {
      const uint64_t p = primes[i].m.p;
      uint64_t carry = alpha[i];
      for (int l = 0; l < len; ++l) {
        const uint64_t lo = acc[l] * p, hi = __umul64hi(acc[l], p);
        const uint64_t s = lo + carry;
        acc[l] = s;
        carry = hi + (s < lo);
      }
      if (carry) acc[len++] = carry;
    }
    for (int l = len; l < L64; ++l) acc[l] = 0;
    // D = P - X; negative iff X > D
    uint64_t d[PDB_MAX_PRIMES + 1];
    uint64_t borrow = 0;
    for (int l = 0; l < L64; ++l) {
      const uint64_t t = prod[l] - acc[l];
      const uint64_t b1 = prod[l] < acc[l];
      d[l] = t - borrow;
      borrow = b1 | (t < borrow);
    }
    int cmp = 0;
    for (int l = L64 - 1; l >= 0 && cmp == 0; --l) cmp = (acc[l] > d[l]) - (acc[l] < d[l]);
    const bool negative = cmp > 0;
    uint32_t* o = limbs + pos * (int64_t)L;
    for (int l = 0; l < L; ++l) {
      const uint64_t w = negative ? d[l >> 1] : acc[l >> 1];
      o[l] = (l >> 1) < L64 ? (uint32_t)(w >> (32 * (l & 1))) : 0u;
    }
    neg[pos] = negative;
  }
}

static int crt64_limbs64(int P) { return (62 * P + 63) / 64 + 1; }

}  // namespace pdb

using namespace pdb;

extern "C" {

int32_t pdb_ntt_multi_u64(pdb_prime_ctx* ctx, uint64_t* data, int64_t batch, int32_t ndim, const int64_t* dims,
                          const int64_t* extents, uint32_t axis_mask, int32_t inverse, void* stream) {
  if (!ctx || !ctx->wide || ndim < 0 || ndim > PDB_MAX_DIMS || batch < 0) {
    set_error("invalid u64 NTT arguments (context must hold a prime >= 2^31)");
    return -2;
  }
  for (int a = 0; a < ndim; ++a)
    if ((axis_mask >> a) & 1)
      if (!ctx_twiddles64(ctx, (int)dims[a])) return -2;
  if (batch == 0) return 0;
  for (int a = ndim - 1; a >= 0; --a) {
    if (!((axis_mask >> a) & 1)) continue;
    int rc = ntt64_axis(ctx, data, batch, ndim, dims, extents, a, inverse != 0, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return 0;
}

int32_t pdb_reduce_scatter_u64(pdb_prime_ctx* ctx, const uint32_t* mag, const uint8_t* neg, const int64_t* pos,
                               int64_t count, int32_t limbs, uint64_t* dst, void* stream) {
  if (!ctx || !ctx->wide || limbs < 1) { set_error("invalid u64 reduce arguments"); return -2; }
  if (count == 0) return 0;
  int64_t blocks = (count + 255) / 256;
  int grid = (int)(blocks < (int64_t)ctx->sms * 8 ? blocks : (int64_t)ctx->sms * 8);
  reduce_scatter64_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(mag, neg, pos, count, limbs, dst, ctx->m64);
  count_launch();
  return check_launch("reduce_scatter64");
}

size_t pdb_det_scratch_bytes_u64(int32_t, int64_t) { return 256; }

static int det64_launch(pdb_prime_ctx* ctx, Staged64 src, const int32_t* ids, int r, int64_t node_lo, int64_t nodes,
                        uint64_t* out, void* scratch, size_t scratch_bytes, uint64_t* tv, int32_t* tc,
                        cudaStream_t st) {
  (void)scratch;
  if (r < 1 || r > PDB_MAX_ORDER) { set_error("unsupported matrix order %d (1..%d)", r, PDB_MAX_ORDER); return -2; }
  if (nodes == 0) return 0;
  if (scratch_bytes < pdb_det_scratch_bytes_u64(r, nodes)) { set_error("det scratch too small"); return -2; }
  const size_t per_warp = sizeof(uint64_t) * (size_t)(r * r + r);
  int warps = (int)((200u * 1024u) / per_warp);
  warps = warps < 1 ? 1 : (warps > DET64_WARPS ? DET64_WARPS : warps);
  const size_t smem = per_warp * warps;
  if (cudaFuncSetAttribute(det64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("det64 attribute");
  const int64_t want = (nodes + warps - 1) / warps;
  const int64_t cap = (int64_t)ctx->sms * 8;
  const int grid = (int)(want < cap ? want : cap);
  det64_kernel<<<grid, 32 * warps, smem, st>>>(src, ids, r, node_lo, nodes, out, ctx->m64, tv, tc);
  count_launch();
  return check_launch("det64");
}

int32_t pdb_det_batch_u64(pdb_prime_ctx* ctx, const uint64_t* grids, int64_t grid_stride, const int32_t* entry_ids,
                          int32_t r, int64_t node_lo, int64_t nodes, uint64_t* out, void* scratch,
                          size_t scratch_bytes, void* stream) {
  if (!ctx || !ctx->wide) { set_error("u64 determinants need a context with p >= 2^31"); return -2; }
  return det64_launch(ctx, Staged64{grids, grid_stride}, entry_ids, r, node_lo, nodes, out, scratch, scratch_bytes,
                      nullptr, nullptr, (cudaStream_t)stream);
}

int32_t pdb_condense_u64(pdb_prime_ctx* ctx, const uint64_t* mat, int32_t r, uint64_t* trail_vals,
                         int32_t* trail_cols, uint64_t* det_out, void* scratch, size_t scratch_bytes, void* stream) {
  if (!ctx || !ctx->wide) { set_error("u64 condense needs a context with p >= 2^31"); return -2; }
  if (r < 1 || r > PDB_MAX_ORDER) { set_error("unsupported matrix order %d (1..%d)", r, PDB_MAX_ORDER); return -2; }
  const size_t ids_bytes = ((sizeof(int32_t) * r * r + 255) & ~size_t(255));
  if (scratch_bytes < ids_bytes + pdb_det_scratch_bytes_u64(r, 1)) { set_error("condense scratch too small"); return -2; }
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int32_t> ids(r * r);
  for (int e = 0; e < r * r; ++e) ids[e] = e;
  int32_t* d_ids = static_cast<int32_t*>(scratch);
  cudaMemcpyAsync(d_ids, ids.data(), sizeof(int32_t) * r * r, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(trail_cols, 0xff, sizeof(int32_t) * r, st);
  cudaStreamSynchronize(st);
  return det64_launch(ctx, Staged64{mat, 1}, d_ids, r, 0, 1, det_out, static_cast<char*>(scratch) + ids_bytes,
                      scratch_bytes - ids_bytes, trail_vals, trail_cols, st);
}

int32_t pdb_crt_limbs_u64(int32_t nprimes) { return 2 * crt64_limbs64(nprimes); }

size_t pdb_crt_scratch_bytes_u64(int32_t nprimes) {
  const int P = nprimes;
  return sizeof(Crt64Prime) * P + sizeof(uint64_t) * ((size_t)P * P + crt64_limbs64(P)) + 1024;
}

int32_t pdb_crt_mrc_u64(const uint64_t* residues, int32_t nprimes, int64_t n, int64_t stride, const uint64_t* primes_host,
                        uint32_t* limbs, int32_t L, uint8_t* neg, void* scratch, size_t scratch_bytes, void* stream) {
  const int P = nprimes;
  if (P < 1 || P > PDB_MAX_PRIMES) { set_error("need 1..%d primes, got %d", PDB_MAX_PRIMES, P); return -2; }
  if (L < pdb_crt_limbs_u64(P)) { set_error("limb count %d too small for %d primes", L, P); return -2; }
  if (scratch_bytes < pdb_crt_scratch_bytes_u64(P)) { set_error("crt scratch too small"); return -2; }
  for (int i = 0; i < P; ++i) {
    const uint64_t p = primes_host[i];
    if (p < 3 || !(p & 1) || p >= (1ull << 62)) { set_error("u64 CRT needs odd primes 3 <= p < 2^62"); return -2; }
    for (int j = 0; j < i; ++j)
      if (primes_host[j] == p) { set_error("duplicate prime %llu", (unsigned long long)p); return -2; }
  }
  std::vector<Crt64Prime> cp(P);
  std::vector<uint64_t> wR((size_t)P * P, 0);
  const int L64 = crt64_limbs64(P);
  std::vector<uint64_t> prod(L64, 0);
  prod[0] = 1;
  for (int i = 0; i < P; ++i) {
    const uint64_t p = primes_host[i];
    cp[i].m = make_mod64(p);
    // m_j mod p_i for j < i (m_j = p_0 ... p_{j-1}); c_i = (m_i mod p_i)^-1
    uint64_t mj = 1 % p;
    for (int j = 0; j < i; ++j) {
      wR[(size_t)i * P + j] = hmont(mj, p);
      mj = hmul(mj, primes_host[j] % p, p);
    }
    cp[i].cR = hmont(i ? hpow(mj, p - 2, p) : 1, p);
    // prod *= p
    unsigned __int128 carry = 0;
    for (int l = 0; l < L64; ++l) {
      unsigned __int128 t = (unsigned __int128)prod[l] * p + carry;
      prod[l] = (uint64_t)t;
      carry = t >> 64;
    }
  }
  char* base = static_cast<char*>(scratch);
  Crt64Prime* d_cp = reinterpret_cast<Crt64Prime*>(base);
  uint64_t* d_w = reinterpret_cast<uint64_t*>(base + sizeof(Crt64Prime) * P);
  uint64_t* d_prod = d_w + (size_t)P * P;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(d_cp, cp.data(), sizeof(Crt64Prime) * P, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_w, wR.data(), sizeof(uint64_t) * P * P, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_prod, prod.data(), sizeof(uint64_t) * L64, cudaMemcpyHostToDevice, st);
  if (n == 0) return check_launch("crt64 tables");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (n + 63) / 64;
  int grid = (int)(blocks < (int64_t)sms * 16 ? blocks : (int64_t)sms * 16);
  crt64_kernel<<<grid, 64, 0, st>>>(residues, P, n, stride, d_cp, d_w, d_prod, L64, L, limbs, neg);
  count_launch();
  // host tables must outlive the async copies
  cudaStreamSynchronize(st);
  return check_launch("crt64");
}

}  // extern "C"
