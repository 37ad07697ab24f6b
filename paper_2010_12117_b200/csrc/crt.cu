// Mixed-radix CRT lift and coefficient reduction.
//
// crt_mrc: one thread per coefficient position (reference crt.py:94-130 does
// the digits vectorised in numpy and the Horner lift in a Python loop; the
// paper's CrtOnGPU, does only the digits on the GPU).  Here
// the whole lift runs on the device:
//   a_0 = x_0,  a_i = (x_i - sum_{j<i} a_j * (m_j mod p_i)) * c_i  (mod p_i)
//   X   = a_{P-1}; X = X * p_i + a_i for i = P-2..0      (multi-limb Horner)
//   out = X if 2X <= P else -(P - X)                     (symmetric lift)
// and writes |out| as little-endian 32-bit limbs plus a sign byte, so the host
// only does `int.from_bytes` (or nothing, for coefficients that are zero).
//
// reduce_scatter: signed multi-limb integer coefficients -> residues mod p,
// written straight into their padded grid positions (reference
// tensor.py:214-237: reduce_mod + pad_to).
#include <map>
#include <vector>
#include "pdb_internal.cuh"

namespace pdb {

struct CrtPrime {
  Mod32 m;
  uint32_t c, cs;   // c_i = (m_i mod p_i)^-1 and companion
};

// Device tables of one CRT basis: primes, the weight residues m_j mod p_i
// (+ Shoup companions, [i][j] row-major) and P = prod p_i as L limbs.
struct CrtTables {
  int P = 0, L = 0;
  CrtPrime* primes = nullptr;
  uint32_t* wres = nullptr;
  uint32_t* wres_s = nullptr;
  uint32_t* prod = nullptr;
};

// The mixed-radix digits, the Horner lift and the symmetric lift of one
// coefficient.  PB >= P is a compile-time bound: every array index is static,
// so the digits and the limbs live in registers (the first version indexed
// PDB_MAX_PRIMES-sized local arrays: a 3 KB stack frame per thread).  PB = 0
// is the generic build for P > 64 (local memory).
template <int PB>
__device__ __forceinline__ int crt_one(const uint32_t* __restrict__ res, int P, int64_t pos, int64_t res_stride,
                                       const CrtTables& T, int L, uint32_t* __restrict__ o, uint8_t* neg) {
  constexpr int NA = PB ? PB : PDB_MAX_PRIMES;
  uint32_t alpha[NA];
  if constexpr (PB == 0) {   // generic: plain loops over local arrays
    for (int i = 0; i < P; ++i) {
      const CrtPrime cp = T.primes[i];
      const uint32_t p = cp.m.p;
      uint32_t x = __ldg(res + (int64_t)i * res_stride + pos);
      for (int j = 0; j < i; ++j) {
        const int w = i * P + j;
        x = sub_mod(x, shoup_mul(alpha[j], __ldg(T.wres + w), __ldg(T.wres_s + w), p), p);
      }
      alpha[i] = i ? shoup_mul(x, cp.c, cp.cs, p) : x;
    }
    uint32_t acc[NA + 2];
    int len = 1;
    acc[0] = alpha[P - 1];
    for (int i = P - 2; i >= 0; --i) {
      const uint32_t p = T.primes[i].m.p;
      uint64_t carry = alpha[i];
      for (int l = 0; l < len; ++l) {
        const uint64_t t = mad_wide(acc[l], p, carry);
        acc[l] = (uint32_t)t;
        carry = t >> 32;
      }
      if (carry) acc[len++] = (uint32_t)carry;
    }
    for (int l = len; l < L; ++l) acc[l] = 0;
    uint32_t d[NA + 2];
    uint32_t borrow = 0;
    for (int l = 0; l < L; ++l) {
      const uint64_t t = (uint64_t)__ldg(T.prod + l) - acc[l] - borrow;
      d[l] = (uint32_t)t;
      borrow = (uint32_t)(t >> 63);
    }
    int cmp = 0;
    for (int l = L - 1; l >= 0 && cmp == 0; --l) cmp = (acc[l] > d[l]) - (acc[l] < d[l]);
    const bool negative = cmp > 0;
    int used = 0;
    for (int l = 0; l < L; ++l) {
      const uint32_t v = negative ? d[l] : acc[l];
      o[l] = v;
      if (v) used = l + 1;
    }
    *neg = negative;
    return used;
  }
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    if (i < P) {
      const CrtPrime cp = T.primes[i];
      const uint32_t p = cp.m.p;
      uint32_t x = __ldg(res + (int64_t)i * res_stride + pos);
#pragma unroll
      for (int j = 0; j < i; ++j) {
        const int w = i * P + j;
        x = sub_mod(x, shoup_mul(alpha[j], __ldg(T.wres + w), __ldg(T.wres_s + w), p), p);
      }
      alpha[i] = i ? shoup_mul(x, cp.c, cp.cs, p) : x;
    }
  }
  // Horner in base 2^32: after the digits of primes i..P-1 the value is below
  // p_i ... p_{P-1} < 2^(31 (P - i)), i.e. at most P - i limbs
  uint32_t acc[NA + 2];
#pragma unroll
  for (int l = 0; l < NA + 2; ++l) acc[l] = 0;
#pragma unroll
  for (int i = NA - 1; i >= 0; --i) {
    if (i < P) {
      if (i == P - 1) {
        acc[0] = alpha[i];
      } else {
        const uint32_t p = T.primes[i].m.p;
        uint64_t carry = alpha[i];
#pragma unroll
        for (int l = 0; l < NA + 1 - i; ++l) {
          const uint64_t t = mad_wide(acc[l], p, carry);
          acc[l] = (uint32_t)t;
          carry = t >> 32;
        }
      }
    }
  }
  // D = P - X; the result is X if X <= D, else -D
  uint32_t d[NA + 2];
  uint32_t borrow = 0;
#pragma unroll
  for (int l = 0; l < NA + 2; ++l) {
    if (l < L) {
      const uint64_t t = (uint64_t)__ldg(T.prod + l) - acc[l] - borrow;
      d[l] = (uint32_t)t;
      borrow = (uint32_t)(t >> 63);
    }
  }
  int cmp = 0;   // X vs D from the top limb
#pragma unroll
  for (int l = NA + 1; l >= 0; --l)
    if (l < L && cmp == 0) cmp = (acc[l] > d[l]) - (acc[l] < d[l]);
  const bool negative = cmp > 0;
  int used = 0;
#pragma unroll
  for (int l = 0; l < NA + 2; ++l) {
    if (l < L) {
      const uint32_t v = negative ? d[l] : acc[l];
      o[l] = v;
      if (v) used = l + 1;
    }
  }
  *neg = negative;
  return used;
}

// index == nullptr: positions 0..count-1; else positions index[0..count).
// width (may be null): max over the coefficients of the limbs actually used.
template <int PB>
__global__ void __launch_bounds__(128)
crt_mrc_kernel(const uint32_t* __restrict__ res, int P, const int64_t* __restrict__ index, int64_t count,
               int64_t res_stride, CrtTables T, int L, uint32_t* __restrict__ limbs, uint8_t* __restrict__ neg,
               int32_t* __restrict__ width) {
  int wmax = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = index ? index[j] : j;
    const int used = crt_one<PB>(res, P, pos, res_stride, T, L, limbs + j * (int64_t)L, neg + j);
    wmax = used > wmax ? used : wmax;
  }
  if (width) {
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      const int o = __shfl_xor_sync(0xffffffffu, wmax, d);
      wmax = o > wmax ? o : wmax;
    }
    if ((threadIdx.x & 31) == 0 && wmax) atomicMax(width, wmax);
  }
}

// ---- nonzero compaction: a coefficient is 0 iff every residue is 0 (0 <= X < P) ----
constexpr int NZ_TILE = 1024;   // positions per block (256 threads x 4)

__global__ void __launch_bounds__(256)
nz_count(const uint32_t* __restrict__ res, int P, int64_t n, int64_t stride, uint8_t* __restrict__ flags,
         int64_t* __restrict__ block_counts) {
  __shared__ int wsum[8];
  const int64_t base = (int64_t)blockIdx.x * NZ_TILE;
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t pos = base + k * 256 + threadIdx.x;
    uint8_t f = 0;
    if (pos < n) {
      uint32_t any = 0;
      for (int i = 0; i < P; ++i) any |= __ldg(res + (int64_t)i * stride + pos);
      f = any != 0;
      flags[pos] = f;
    }
    cnt += f;
  }
  for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < 8; ++w) t += wsum[w];
    block_counts[blockIdx.x] = t;
  }
}

// exclusive scan of the block counts in place (one CTA), total -> *count
__global__ void __launch_bounds__(1024)
nz_scan(int64_t* __restrict__ block_counts, int64_t nblocks, int64_t* __restrict__ count) {
  __shared__ int64_t part[1024];
  const int64_t per = (nblocks + 1023) / 1024;
  const int64_t lo = threadIdx.x * per, hi = lo + per < nblocks ? lo + per : nblocks;
  int64_t s = 0;
  for (int64_t b = lo; b < hi; ++b) s += block_counts[b];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {
    const int64_t v = threadIdx.x >= d ? part[threadIdx.x - d] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t b = lo; b < hi; ++b) {
    const int64_t c = block_counts[b];
    block_counts[b] = run;
    run += c;
  }
  if (threadIdx.x == 1023) *count = part[1023];
}

__global__ void __launch_bounds__(256)
nz_write(const uint8_t* __restrict__ flags, int64_t n, const int64_t* __restrict__ offsets,
         int64_t* __restrict__ index) {
  __shared__ int wsum[8 * 4];
  const int64_t base = (int64_t)blockIdx.x * NZ_TILE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // positions in order: chunk k of 256, warp w, lane -> base + k*256 + w*32 + lane
  bool f[4];
  int wc[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t pos = base + k * 256 + threadIdx.x;
    f[k] = pos < n && flags[pos];
    wc[k] = __popc(__ballot_sync(0xffffffffu, f[k]));
    if (lane == 0) wsum[k * 8 + warp] = wc[k];
  }
  __syncthreads();
  int64_t off = offsets[blockIdx.x];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int before = 0;
    for (int w = 0; w < k * 8 + warp; ++w) before += wsum[w];
    const unsigned m = __ballot_sync(0xffffffffu, f[k]);
    if (f[k]) index[off + before + __popc(m & ((1u << lane) - 1))] = base + k * 256 + threadIdx.x;
  }
}

__global__ void __launch_bounds__(256)
reduce_scatter_kernel(const uint32_t* __restrict__ mag, const uint8_t* __restrict__ negs,
                      const int64_t* __restrict__ pos, int64_t count, int Lc,
                      uint32_t* __restrict__ dst, Mod32 m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (int l = Lc - 1; l >= 0; --l) {
      v = add_mod(shoup_mul(v, m.r1, m.r1s, m.p), canon32(mag[i * Lc + l], m), m.p);
    }
    if (negs[i] && v) v = m.p - v;
    dst[pos[i]] = v;
  }
}

int reduce_scatter(PrimeCtx* ctx, const uint32_t* mag, const uint8_t* neg, const int64_t* pos,
                   int64_t count, int Lc, uint32_t* dst, cudaStream_t st) {
  if (count == 0) return 0;
  int64_t blocks = (count + 255) / 256;
  int grid = (int)(blocks < (int64_t)ctx->sms * 8 ? blocks : (int64_t)ctx->sms * 8);
  reduce_scatter_kernel<<<grid, 256, 0, st>>>(mag, neg, pos, count, Lc, dst, ctx->m);
  count_launch();
  return check_launch("reduce_scatter");
}

// Host-side CRT tables (device copies owned by the caller-provided scratch).
static void mul_small(std::vector<uint32_t>& a, uint32_t m) {
  uint64_t carry = 0;
  for (auto& x : a) {
    uint64_t t = (uint64_t)x * m + carry;
    x = (uint32_t)t;
    carry = t >> 32;
  }
  if (carry) a.push_back((uint32_t)carry);
}

size_t crt_scratch_bytes(int P) {
  (void)P;   // the tables live in a per-basis cache; nothing per call
  return 256;
}

int crt_limbs(int P) {
  // P primes < 2^31 -> product < 2^(31 P); plus one limb of headroom
  return (31 * P + 31) / 32 + 1;
}

// Tables per prime basis, built once (synchronous upload, outside the hot
// calls) and kept for the process: crt_mrc itself never synchronises.
static std::mutex g_crt_lock;
static std::map<std::pair<int, std::vector<uint32_t>>, CrtTables> g_crt_tables;

static const CrtTables* crt_tables(const uint32_t* primes_host, int P, int L) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<uint32_t> key(primes_host, primes_host + P);
  std::lock_guard<std::mutex> guard(g_crt_lock);
  auto it = g_crt_tables.find({dev, key});
  if (it != g_crt_tables.end() && it->second.L >= L) return &it->second;
  std::vector<CrtPrime> cp(P);
  std::vector<uint32_t> w((size_t)P * P, 0), ws((size_t)P * P, 0);
  for (int i = 0; i < P; ++i) {
    const uint32_t p = primes_host[i];
    if (p >= (1u << 31) || p < 2) {
      set_error("prime %u outside the 32-bit kernel range", p);
      return nullptr;
    }
    for (int j = 0; j < i; ++j)
      if (primes_host[j] == p) {
        set_error("duplicate primes in CRT basis");
        return nullptr;
      }
    cp[i].m = make_mod32(p);
    // m_j mod p_i for j <= i (m_0 = 1), c_i = (m_i mod p_i)^-1
    uint64_t mj = 1 % p;
    for (int j = 0; j < i; ++j) {
      w[(size_t)i * P + j] = (uint32_t)mj;
      ws[(size_t)i * P + j] = shoup_companion((uint32_t)mj, p);
      mj = mj * (primes_host[j] % p) % p;
    }
    const uint32_t c = i ? inv_mod((uint32_t)mj, cp[i].m) : 1u % p;
    cp[i].c = c;
    cp[i].cs = shoup_companion(c, p);
  }
  std::vector<uint32_t> prod{1};
  for (int i = 0; i < P; ++i) mul_small(prod, primes_host[i]);
  prod.resize(L, 0);
  const size_t head = (sizeof(CrtPrime) * P + 255) & ~size_t(255);
  const size_t bytes = head + sizeof(uint32_t) * (2 * (size_t)P * P + L);
  char* dbuf = nullptr;
  if (cudaMalloc(&dbuf, bytes) != cudaSuccess) {
    set_error("crt table allocation failed");
    return nullptr;
  }
  CrtTables T;
  T.P = P;
  T.L = L;
  T.primes = reinterpret_cast<CrtPrime*>(dbuf);
  T.wres = reinterpret_cast<uint32_t*>(dbuf + head);
  T.wres_s = T.wres + (size_t)P * P;
  T.prod = T.wres_s + (size_t)P * P;
  cudaError_t e = cudaMemcpy(T.primes, cp.data(), sizeof(CrtPrime) * P, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(T.wres, w.data(), sizeof(uint32_t) * P * P, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(T.wres_s, ws.data(), sizeof(uint32_t) * P * P, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(T.prod, prod.data(), sizeof(uint32_t) * L, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    set_error("crt table upload: %s", cudaGetErrorString(e));
    cudaFree(dbuf);
    return nullptr;
  }
  if (it != g_crt_tables.end()) cudaFree(it->second.primes);   // a narrower table of the same basis
  return &(g_crt_tables[{dev, key}] = T);
}

int crt_mrc_sel(const uint32_t* res, int P, const int64_t* index, int64_t count, int64_t res_stride,
                const uint32_t* primes_host, uint32_t* limbs, int L, uint8_t* neg, int32_t* width, int sms,
                cudaStream_t st) {
  if (P < 1 || P > PDB_MAX_PRIMES) {
    set_error("unsupported prime count %d (1..%d)", P, PDB_MAX_PRIMES);
    return -2;
  }
  if (L < crt_limbs(P)) {
    set_error("limb count %d too small for %d primes (need %d)", L, P, crt_limbs(P));
    return -2;
  }
  const CrtTables* T = crt_tables(primes_host, P, L);
  if (!T) return -2;
  if (width) cudaMemsetAsync(width, 0, sizeof(int32_t), st);
  if (count <= 0) return check_launch("crt_mrc");
  const int64_t blocks = (count + 127) / 128;
  const int grid = (int)(blocks < (int64_t)sms * 16 ? blocks : (int64_t)sms * 16);
#define PDB_CRT(PB) crt_mrc_kernel<PB><<<grid, 128, 0, st>>>(res, P, index, count, res_stride, *T, L, limbs, neg, width)
  if (P <= 8) PDB_CRT(8);
  else if (P <= 16) PDB_CRT(16);
  else if (P <= 24) PDB_CRT(24);
  else if (P <= 32) PDB_CRT(32);
  else if (P <= 64) PDB_CRT(64);
  else PDB_CRT(0);
#undef PDB_CRT
  count_launch();
  return check_launch("crt_mrc");
}

int crt_mrc(const uint32_t* res, int P, int64_t n, int64_t res_stride, const uint32_t* primes_host,
            uint32_t* limbs, int L, uint8_t* neg, void* scratch, size_t scratch_bytes, int sms,
            cudaStream_t st) {
  (void)scratch;
  (void)scratch_bytes;
  return crt_mrc_sel(res, P, nullptr, n, res_stride, primes_host, limbs, L, neg, nullptr, sms, st);
}

// |X| as u32 limb rows [count][width] (stride ls words) -> CPython's 30-bit
// digits [count][D] (D = ceil(32 width / 30)) and the significant digit count,
// so the host builds each int with one allocation and one copy.
__global__ void __launch_bounds__(256)
limbs_to_digits30(const uint32_t* __restrict__ limbs, int64_t count, int width, int64_t ls,
                  uint32_t* __restrict__ digits, int D, uint8_t* __restrict__ ndig) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* row = limbs + j * ls;
    uint32_t* out = digits + j * (int64_t)D;
    int nd = 0, used = 0, bits = 0;
    uint64_t acc = 0;
    for (int w = 0; w < width; ++w) {
      acc |= (uint64_t)__ldg(row + w) << bits;
      bits += 32;
      while (bits >= 30) {
        const uint32_t d = (uint32_t)acc & 0x3fffffffu;
        out[nd++] = d;
        if (d) used = nd;
        acc >>= 30;
        bits -= 30;
      }
    }
    if (bits > 0) {
      const uint32_t d = (uint32_t)acc;
      out[nd++] = d;
      if (d) used = nd;
    }
    for (; nd < D; ++nd) out[nd] = 0u;
    ndig[j] = (uint8_t)used;
  }
}

int limbs_to_digits(const uint32_t* limbs, int64_t count, int width, int64_t ls, uint32_t* digits, int D,
                    uint8_t* ndig, int sms, cudaStream_t st) {
  if (width < 1 || D < (32 * width + 29) / 30 || D > 255 || ls < width) {
    set_error("limbs_to_digits: width %d, digit rows %d, stride %lld", width, D, (long long)ls);
    return -2;
  }
  if (count <= 0) return 0;
  const int64_t blocks = (count + 255) / 256;
  const int grid = (int)(blocks < (int64_t)sms * 8 ? blocks : (int64_t)sms * 8);
  limbs_to_digits30<<<grid, 256, 0, st>>>(limbs, count, width, ls, digits, D, ndig);
  count_launch();
  return check_launch("limbs_to_digits");
}

size_t crt_nonzero_scratch_bytes(int64_t n) {
  const int64_t nb = (n + NZ_TILE - 1) / NZ_TILE;
  return 256 + sizeof(int64_t) * (size_t)nb + (size_t)n;
}

int crt_nonzero(const uint32_t* res, int P, int64_t n, int64_t stride, int64_t* index, int64_t* count,
                void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (P < 1 || n < 0) { set_error("invalid nonzero arguments"); return -2; }
  if (scratch_bytes < crt_nonzero_scratch_bytes(n)) { set_error("nonzero scratch too small"); return -2; }
  if (n == 0) {
    cudaMemsetAsync(count, 0, sizeof(int64_t), st);
    return check_launch("crt_nonzero");
  }
  const int64_t nb = (n + NZ_TILE - 1) / NZ_TILE;
  int64_t* bc = reinterpret_cast<int64_t*>(static_cast<char*>(scratch) + 256);
  uint8_t* flags = reinterpret_cast<uint8_t*>(bc + nb);
  nz_count<<<(unsigned)nb, 256, 0, st>>>(res, P, n, stride, flags, bc);
  nz_scan<<<1, 1024, 0, st>>>(bc, nb, count);
  nz_write<<<(unsigned)nb, 256, 0, st>>>(flags, n, bc, index);
  count_launch(3);
  return check_launch("crt_nonzero");
}

}  // namespace pdb
