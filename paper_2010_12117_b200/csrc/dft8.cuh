// Evaluation of a polynomial with E <= 8 coefficients at 8 nodes
// {zeta * w8^v : v < 8} (w8 a primitive 8th root of unity): twist the
// coefficients by zeta^l, then an 8-point radix-2 DIT transform whose first
// stage is trivial for the coefficient slots >= E.  Used by the det kernel's
// fused fill (det_gj.cuh) and by the sparse forward NTT (ntt.cu): both
// evaluate entries with few coefficients along an axis at 8 nodes at a time,
// ~(E - 1 + 5) / 8 mul-mods per node instead of E - 1 for Horner.
#pragma once
#include "pdb_internal.cuh"

namespace pdb {

// Radix-2 butterfly (x, y) -> (x + y, x - y); ZERO: y is known to be 0.
template <bool ZERO>
__device__ __forceinline__ void gj_bf(uint32_t& x, uint32_t& y, uint32_t p) {
  if constexpr (ZERO) {
    y = x;
  } else {
    const uint32_t t = y;
    y = sub_mod(x, t, p);
    x = add_mod(x, t, p);
  }
}

// X[v] = sum_{l<E} c_l w^(u l) w8^(l v), v < 8: twist, then an 8-point DIT
// transform whose first stage is trivial for the coefficient slots >= E.
template <int E>
__device__ __forceinline__ void gj_dft8(const uint32_t (&c)[E], const uint32_t* tw, const uint32_t* tws,
                                        const uint32_t (&w)[4], const uint32_t (&ws)[4], uint32_t p,
                                        uint32_t (&x)[8]) {
  uint32_t q[8];
  q[0] = c[0];
#pragma unroll
  for (int l = 1; l < 8; ++l) q[l] = l < E ? shoup_mul(c[l < E ? l : 0], tw[l], tws[l], p) : 0u;
  // bit-reversed order
  x[0] = q[0]; x[1] = q[4]; x[2] = q[2]; x[3] = q[6]; x[4] = q[1]; x[5] = q[5]; x[6] = q[3]; x[7] = q[7];
  gj_bf<(4 >= E)>(x[0], x[1], p);
  gj_bf<(6 >= E)>(x[2], x[3], p);
  gj_bf<(5 >= E)>(x[4], x[5], p);
  gj_bf<(7 >= E)>(x[6], x[7], p);
  uint32_t t;
  gj_bf<false>(x[0], x[2], p);
  t = shoup_mul(x[3], w[2], ws[2], p); x[3] = t; gj_bf<false>(x[1], x[3], p);
  gj_bf<false>(x[4], x[6], p);
  t = shoup_mul(x[7], w[2], ws[2], p); x[7] = t; gj_bf<false>(x[5], x[7], p);
  gj_bf<false>(x[0], x[4], p);
  t = shoup_mul(x[5], w[1], ws[1], p); x[5] = t; gj_bf<false>(x[1], x[5], p);
  t = shoup_mul(x[6], w[2], ws[2], p); x[6] = t; gj_bf<false>(x[2], x[6], p);
  t = shoup_mul(x[7], w[3], ws[3], p); x[7] = t; gj_bf<false>(x[3], x[7], p);
}

}  // namespace pdb
