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
#include <vector>
#include "pdb_internal.cuh"

namespace pdb {

struct CrtPrime {
  Mod32 m;
  uint32_t c, cs;   // c_i = (m_i mod p_i)^-1 and companion
};

__global__ void __launch_bounds__(128)
crt_mrc_kernel(const uint32_t* __restrict__ res, int P, int64_t n, int64_t res_stride,
               const CrtPrime* __restrict__ primes, const uint32_t* __restrict__ wres,
               const uint32_t* __restrict__ wres_s, const uint32_t* __restrict__ prod_limbs,
               int L, uint32_t* __restrict__ limbs, uint8_t* __restrict__ neg) {
  uint32_t alpha[PDB_MAX_PRIMES];
  uint32_t acc[PDB_MAX_PRIMES + 2];
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < n;
       pos += (int64_t)gridDim.x * blockDim.x) {
    for (int i = 0; i < P; ++i) {
      const CrtPrime cp = primes[i];
      const uint32_t p = cp.m.p;
      uint32_t x = res[(int64_t)i * res_stride + pos];
      for (int j = 0; j < i; ++j) {
        const int w = i * P + j;
        x = sub_mod(x, shoup_mul(alpha[j], wres[w], wres_s[w], p), p);
      }
      alpha[i] = i ? shoup_mul(x, cp.c, cp.cs, p) : x;
    }
    // Horner in base 2^32 limbs
    int len = 1;
    acc[0] = alpha[P - 1];
    for (int i = P - 2; i >= 0; --i) {
      const uint32_t p = primes[i].m.p;
      uint64_t carry = alpha[i];
      for (int l = 0; l < len; ++l) {
        uint64_t t = (uint64_t)acc[l] * p + carry;
        acc[l] = (uint32_t)t;
        carry = t >> 32;
      }
      if (carry) acc[len++] = (uint32_t)carry;
    }
    for (int l = len; l < L; ++l) acc[l] = 0;
    // D = P - X; choose X if X <= D else D (negative)
    uint32_t d[PDB_MAX_PRIMES + 2];
    int64_t borrow = 0;
    for (int l = 0; l < L; ++l) {
      int64_t t = (int64_t)prod_limbs[l] - acc[l] - borrow;
      borrow = t < 0;
      d[l] = (uint32_t)(t + (borrow << 32));
    }
    int cmp = 0;  // compare X with D from the top limb
    for (int l = L - 1; l >= 0 && cmp == 0; --l) cmp = (acc[l] > d[l]) - (acc[l] < d[l]);
    const bool negative = cmp > 0;
    uint32_t* o = limbs + pos * (int64_t)L;
    for (int l = 0; l < L; ++l) o[l] = negative ? d[l] : acc[l];
    neg[pos] = negative;
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
  return sizeof(CrtPrime) * P + 2 * sizeof(uint32_t) * (size_t)P * P +
         sizeof(uint32_t) * (size_t)(P + 2) + 1024;
}

int crt_limbs(int P) {
  // P primes < 2^31 -> product < 2^(31 P); plus one limb of headroom
  return (31 * P + 31) / 32 + 1;
}

int crt_mrc(const uint32_t* res, int P, int64_t n, int64_t res_stride, const uint32_t* primes_host,
            uint32_t* limbs, int L, uint8_t* neg, void* scratch, size_t scratch_bytes, int sms,
            cudaStream_t st) {
  if (P < 1 || P > PDB_MAX_PRIMES) {
    set_error("unsupported prime count %d (1..%d)", P, PDB_MAX_PRIMES);
    return -2;
  }
  if (L < crt_limbs(P)) {
    set_error("limb count %d too small for %d primes (need %d)", L, P, crt_limbs(P));
    return -2;
  }
  if (scratch_bytes < crt_scratch_bytes(P)) {
    set_error("crt scratch too small");
    return -2;
  }
  std::vector<CrtPrime> cp(P);
  std::vector<uint32_t> w((size_t)P * P, 0), ws((size_t)P * P, 0);
  for (int i = 0; i < P; ++i) {
    const uint32_t p = primes_host[i];
    if (p >= (1u << 31) || p < 2) {
      set_error("prime %u outside the 32-bit kernel range", p);
      return -2;
    }
    for (int j = 0; j < i; ++j)
      if (primes_host[j] == p) {
        set_error("duplicate primes in CRT basis");
        return -2;
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
  char* base = static_cast<char*>(scratch);
  CrtPrime* d_cp = reinterpret_cast<CrtPrime*>(base);
  uint32_t* d_w = reinterpret_cast<uint32_t*>(base + ((sizeof(CrtPrime) * P + 255) & ~size_t(255)));
  uint32_t* d_ws = d_w + (size_t)P * P;
  uint32_t* d_prod = d_ws + (size_t)P * P;
  if (scratch_bytes < (size_t)((char*)(d_prod + L) - base)) {
    set_error("crt scratch too small for limbs");
    return -2;
  }
  cudaMemcpyAsync(d_cp, cp.data(), sizeof(CrtPrime) * P, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_w, w.data(), sizeof(uint32_t) * P * P, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_ws, ws.data(), sizeof(uint32_t) * P * P, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_prod, prod.data(), sizeof(uint32_t) * L, cudaMemcpyHostToDevice, st);
  // the host vectors must outlive the async copies
  cudaStreamSynchronize(st);
  if (n > 0) {
    int64_t blocks = (n + 127) / 128;
    int grid = (int)(blocks < (int64_t)sms * 16 ? blocks : (int64_t)sms * 16);
    crt_mrc_kernel<<<grid, 128, 0, st>>>(res, P, n, res_stride, d_cp, d_w, d_ws, d_prod, L, limbs, neg);
    count_launch();
  }
  return check_launch("crt_mrc");
}

}  // namespace pdb
