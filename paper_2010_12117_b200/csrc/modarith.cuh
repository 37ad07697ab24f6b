// Word-size modular arithmetic for the sm_100a kernels.
//
// All moduli on the 32-bit path satisfy p < 2^31 (so 2p < 2^32); the fast
// elimination kernels additionally require p < 2^30 (see Mod32::fast()).
//
// Primitives (cost in fma-heavy issue slots, measured on B200: IMAD = 1,
// IMAD.HI = IMAD.WIDE = 2; see profiles/intpipe_r01.json):
//   shoup_mul(x, w, w')  x*w mod p in [0, 2p) for a constant w          (2 IMAD + 1 IMAD.HI)
//   mul(a, b)            a*b mod p for two variables (Barrett, 64-bit)  (~6 IMAD-class)
//   redc(acc)            acc * 2^-32 mod p in [0, 2^32) for acc < (2^32-p-1) 2^32
//   canon32(v)           v mod p for any 32-bit v                       (IMAD.HI + IMAD + 1 ALU)
#pragma once
#include <cstdint>

#define PDB_HD __host__ __device__ __forceinline__

struct Mod32 {
  uint32_t p;        // the prime
  uint32_t qinv;     // p^-1 mod 2^32 (Montgomery, subtractive form)
  uint32_t mu;       // floor(2^32 / p)   (canon32)
  uint32_t r2;       // 2^64 mod p        (to_mont)
  uint32_t r1;       // 2^32 mod p
  uint32_t r1s;      // Shoup companion of r1
  uint64_t m64;      // floor(2^64 / p)   (Barrett for 64-bit products)

  PDB_HD bool fast() const { return p < (1u << 30) && (p & 1u); }   // Montgomery needs odd p
  PDB_HD bool odd() const { return (p & 1u) != 0; }
};

PDB_HD uint32_t umulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

PDB_HD uint64_t umulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// min(x, x - m) as unsigned: subtracts m once if x >= m (x < 2m).
PDB_HD uint32_t csub(uint32_t x, uint32_t m) {
  uint32_t y = x - m;
  return y < x ? y : x;
}

PDB_HD uint32_t add_mod(uint32_t a, uint32_t b, uint32_t p) { return csub(a + b, p); }
PDB_HD uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t p) { return csub(a + p - b, p); }

// Shoup companion floor(w * 2^32 / p) for w < p (host or device; slow path).
PDB_HD uint32_t shoup_companion(uint32_t w, uint32_t p) {
  return (uint32_t)(((uint64_t)w << 32) / p);
}

// Shoup companion via the precomputed floor(2^64/p): q = floor(w*2^32/p) exactly.
// q_est = floor(w * m64 / 2^32) = w*m_hi + hi(w*m_lo) is the exact quotient or
// one below it; the remainder w*2^32 - q*p < 2p fits 32 bits, so it is
// computed mod 2^32 as -q*p.
PDB_HD uint32_t shoup_companion_fast(uint32_t w, const Mod32& m) {
  uint32_t q = w * (uint32_t)(m.m64 >> 32) + umulhi32(w, (uint32_t)m.m64);
  uint32_t r = 0u - q * m.p;
  return r >= m.p ? q + 1 : q;
}

// x*w mod p, result in [0, 2p). Valid for any 32-bit x, w < p, ws = companion.
PDB_HD uint32_t shoup_lazy(uint32_t x, uint32_t w, uint32_t ws, uint32_t p) {
  uint32_t q = umulhi32(x, ws);
  return x * w - q * p;
}

PDB_HD uint32_t shoup_mul(uint32_t x, uint32_t w, uint32_t ws, uint32_t p) {
  return csub(shoup_lazy(x, w, ws, p), p);
}

// a*b mod p for variables a, b < 2^31 (p < 2^31): Barrett on the 62-bit product.
PDB_HD uint32_t mul_mod(uint32_t a, uint32_t b, const Mod32& m) {
  uint64_t t = (uint64_t)a * b;
  uint64_t q = umulhi64(t, m.m64);
  uint64_t r = t - q * m.p;          // in [0, 2p)
  return csub((uint32_t)r, m.p);
}

// c + a*b as one IMAD.WIDE.U32 (64-bit accumulate of a 32x32 product).  Written
// as a carry chain on the 32-bit halves: ptxas fuses mad.lo.cc + madc.hi into a
// single accumulating IMAD.WIDE.U32, whereas mad.wide.u32 with a 64-bit addend
// is split into IMAD.WIDE + IADD3 + IADD3.X (tools/microbench/mac.cu).
PDB_HD uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) {
#ifdef __CUDA_ARCH__
  uint32_t lo = (uint32_t)c, hi = (uint32_t)(c >> 32);
  asm("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo), "+r"(hi) : "r"(a), "r"(b));
  return ((uint64_t)hi << 32) | lo;
#else
  return c + (uint64_t)a * b;
#endif
}

// Montgomery reduction, subtractive form: with mq = lo(acc) * p^-1 mod 2^32,
// lo(mq * p) == lo(acc), so acc - mq*p = (hi(acc) - hi(mq*p)) * 2^32 exactly and
//   v = hi(acc) + p - hi(mq*p) == acc * 2^-32 (mod p),  0 < v <= hi(acc) + p.
// Three instructions (IMAD, IMAD.HI, IADD3); valid whenever hi(acc) + p < 2^32,
// e.g. up to 12 products of residues when p < 2^30.
PDB_HD uint32_t redc(uint64_t acc, const Mod32& m) {
  const uint32_t mq = (uint32_t)acc * m.qinv;
  return (uint32_t)(acc >> 32) + m.p - umulhi32(mq, m.p);
}

// The same reduction in additive form: with nq = -lo(acc) * p^-1 mod 2^32,
// acc + nq*p == 0 (mod 2^32) and v = hi(acc + nq*p) = acc * 2^-32 (mod p),
// v <= hi(acc) + p.  The 64-bit sum is one accumulating IMAD.WIDE (no IMAD.HI,
// no IADD3); valid whenever acc + (2^32 - 1) p < 2^64 (e.g. 9 products of
// residues for p < 2^30, 2 for p < 2^31).
PDB_HD uint32_t redc_add(uint64_t acc, const Mod32& m) {
  const uint32_t nq = (uint32_t)acc * (0u - m.qinv);
#ifdef __CUDA_ARCH__
  uint32_t lo = (uint32_t)acc, hi = (uint32_t)(acc >> 32);
  asm("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo), "+r"(hi) : "r"(nq), "r"(m.p));
  return hi;
#else
  return (uint32_t)((acc + (uint64_t)nq * m.p) >> 32);
#endif
}

// Any 32-bit v -> [0, p).
PDB_HD uint32_t canon32(uint32_t v, const Mod32& m) {
  uint32_t q = umulhi32(v, m.mu);
  return csub(v - q * m.p, m.p);
}

// Montgomery product a * b * 2^-32 mod p, canonical (a, b < 2^32, a*b < (2^32-p-1) 2^32).
// With b = x*R mod p ("Montgomery form") this is the plain product a*x.
PDB_HD uint32_t mont(uint32_t a, uint32_t b, const Mod32& m) {
  return canon32(redc(mad_wide(a, b, 0ull), m), m);
}

// x -> x*R mod p (R = 2^32), canonical.
PDB_HD uint32_t to_mont(uint32_t x, const Mod32& m) { return shoup_mul(x, m.r1, m.r1s, m.p); }

// (a*R)^e * R mod p for aR in Montgomery form (square and multiply).
PDB_HD uint32_t mont_pow(uint32_t aR, uint64_t e, const Mod32& m) {
  uint32_t r = m.r1, b = aR;
  while (e) {
    if (e & 1) r = mont(r, b, m);
    b = mont(b, b, m);
    e >>= 1;
  }
  return r;
}

PDB_HD uint32_t pow_mod(uint32_t a, uint64_t e, const Mod32& m) {
  uint32_t r = 1 % m.p, b = a;
  while (e) {
    if (e & 1) r = mul_mod(r, b, m);
    b = mul_mod(b, b, m);
    e >>= 1;
  }
  return r;
}

PDB_HD uint32_t inv_mod(uint32_t a, const Mod32& m) { return pow_mod(a, m.p - 2, m); }

// Host-side construction of the constants.
inline Mod32 make_mod32(uint32_t p) {
  Mod32 m;
  m.p = p;
  uint32_t inv = 1;  // Newton iteration for p^-1 mod 2^32
  for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
  m.qinv = inv;
  m.mu = (uint32_t)((((uint64_t)1) << 32) / p);
  m.r1 = (uint32_t)((((uint64_t)1) << 32) % p);
  m.r2 = (uint32_t)(((unsigned __int128)1 << 64) % p);
  m.r1s = shoup_companion(m.r1, p);
  m.m64 = (uint64_t)(((unsigned __int128)1 << 64) / p);
  return m;
}

// ---- 64-bit moduli (the wide path: 2^31 <= p < 2^62) ---------------------------
// Montgomery arithmetic with R = 2^64 in the subtractive form:
//   mont64(a, b) = a*b*2^-64 mod p,  canonical for a, b < p < 2^62
// (hi(a*b) < p/4, so hi + p - hi(q*p) < 1.25 p: one conditional subtraction).
struct Mod64 {
  uint64_t p;
  uint64_t qinv;   // p^-1 mod 2^64
  uint64_t r1;     // 2^64 mod p   (Montgomery one)
  uint64_t r2;     // 2^128 mod p  (to Montgomery form)
  uint64_t r96;    // 2^96 mod p   (Montgomery form of 2^32: limb Horner)
};

PDB_HD uint64_t mont64(uint64_t a, uint64_t b, const Mod64& m) {
  const uint64_t lo = a * b;
  const uint64_t hi = umulhi64(a, b);
  const uint64_t q = lo * m.qinv;
  const uint64_t v = hi + m.p - umulhi64(q, m.p);
  return v >= m.p ? v - m.p : v;
}

PDB_HD uint64_t add_mod64(uint64_t a, uint64_t b, uint64_t p) {
  const uint64_t s = a + b;
  return s >= p ? s - p : s;
}

PDB_HD uint64_t sub_mod64(uint64_t a, uint64_t b, uint64_t p) { return a >= b ? a - b : a + p - b; }

PDB_HD uint64_t to_mont64(uint64_t x, const Mod64& m) { return mont64(x, m.r2, m); }
PDB_HD uint64_t from_mont64(uint64_t x, const Mod64& m) { return mont64(x, 1, m); }

// Montgomery power: aR -> a^e R
PDB_HD uint64_t mont_pow64(uint64_t aR, uint64_t e, const Mod64& m) {
  uint64_t r = m.r1, b = aR;
  while (e) {
    if (e & 1) r = mont64(r, b, m);
    b = mont64(b, b, m);
    e >>= 1;
  }
  return r;
}

inline Mod64 make_mod64(uint64_t p) {
  Mod64 m;
  m.p = p;
  uint64_t inv = 1;   // Newton iteration for p^-1 mod 2^64 (p odd)
  for (int i = 0; i < 6; ++i) inv *= 2u - p * inv;
  m.qinv = inv;
  m.r1 = (uint64_t)(((unsigned __int128)1 << 64) % p);
  m.r2 = (uint64_t)((unsigned __int128)m.r1 * m.r1 % p);
  m.r96 = (uint64_t)((unsigned __int128)m.r2 * ((uint64_t)1 << 32) % p);
  return m;
}
