// det_gj: blocked Schur-complement elimination, one lane group per matrix.
//
// The value of det(M) mod p is algorithm independent (reference
// determinant.py:1-8), so this kernel chooses the schedule that suits the
// integer pipes of sm_100a (profiles/README_r01.md):
//
//   for every block of 8 pivots K..K+7 (the order r is padded to RP = 8*ceil(r/8)
//   with an identity block, which leaves the determinant unchanged):
//     P  X = c A11^-1: in the compile-time-order kernels by 4x4 blocks and
//        adjugates (gj_pinv44 / gj_pdet44 below: c = det(A) det(S)); otherwise
//        division-free Gauss-Jordan on the 8x8 pivot block A11, in registers
//        (LPM/8 lanes per row, pivot rows exchanged by shuffles):
//        X * A11 = c * I  with  c = prod z_s: the pivot row of step s is scaled by
//        lambda_s = z_0..z_{s-1} (the others by z_s), so every row ends up scaled
//        by c and the in-place inverse part E is X itself;
//        det(A11) = prod_s z_s^(s+1) / prod_s z_s^7
//     M  one delayed pass  negM = -X * A12           (8 MACs, one REDC per element)
//     T  trailing update   A22 <- c*A22 + A21*negM   (9 MACs, one REDC per element)
//        = c * (A22 - A21 A11^-1 A12),  so  det A = det A11 * det A22' / c^m.
//   Over all blocks: det = prod_b z_{b,7} / (prod_{b,k=1..6} lambda_{b,k} * C^8),
//   lambda_k = z_0..z_{k-1}, C = prod_{b<last} Q_b, Q_b = c_0 ... c_b.
//
// Arithmetic is Montgomery (R = 2^32) throughout: the stored entries are read
// as Montgomery forms of A' = A R^-1, so no conversion is needed anywhere and
// det(A) = det(A') R^r is applied once per node by det_gj_finalize, which also
// does the single modular inversion per node (batched by 32 per warp).
// Accumulators hold <= 9 products of canonical residues: 9 p^2 < 2^63.2 for
// p < 2^30 (Mod32::fast), inside REDC's bound; REDC output < 3.25 p is made
// canonical with two conditional subtractions (ALU pipe, no IMAD.HI).  For
// 2^30 <= p < 2^31 (template P31) the M and T passes reduce every two
// products and add the partial results mod p.
//
// A zero pivot (prob. ~r/p per node) diverts the node to det_robust, which
// applies the reference's first-nonzero pivoting (determinant.py:136-169).
//
// Shape choices measured on B200 (profiles/README_r01.md): 16 lanes per matrix
// (two matrices per warp), 8 warps per CTA, 2 CTAs per SM (shared memory holds
// 32 matrices of 40x40); 2x4 register tiles in the M and T passes (2x8, 4x4
// measured slower); matrix stride 16 (mod 32) words and swizzled 8-word tiles
// against bank conflicts.  Padded orders 40 and 16 are also built with the
// order as a template constant (RPC): the block loop unrolls and every
// shared-memory address becomes an immediate offset (+10 %).  The kernel is
// bound by the issue of IMAD.WIDE / IMAD.HI (~4 cycles per warp instruction
// each on B200); see DESIGN.md section 4 for the per-phase cost model.
#pragma once
#include <type_traits>

#include "pdb_internal.cuh"
#include "dft8.cuh"

namespace pdb {

constexpr int GJ_B = 8;
// negX rows: row j at word gj_nx_row(j); rows 0-3 and 4-7 are offset by 4 words so that
// the two row groups of the M pass fall in different shared-memory bank groups
__host__ __device__ constexpr int gj_nx_row(int j) { return j * GJ_B + (j / 4) * 4; }
constexpr int GJ_NX_WORDS = 8 * GJ_B + 4;

// matrix stride (words) for padded order RP: RP rows + negX, padded to 16 mod 32
// (the two matrices of a warp, and the U matrices a fill group writes, start in
// opposite bank halves)
__host__ __device__ constexpr int gj_matrix_stride(int RP, int S) {
  return RP * S + GJ_NX_WORDS + ((16 - (RP * S + GJ_NX_WORDS) % 32) + 32) % 32;
}

#define PDB_PRAGMA_(x) _Pragma(#x)
#define PDB_UNROLL_(n) PDB_PRAGMA_(unroll n)
#define PDB_UNROLL(n) PDB_UNROLL_(n)
#ifndef PDB_GJ_TUNROLL
#define PDB_GJ_TUNROLL 4   // unroll factor of the trailing-update tile loop (round 2 end: 4 +0.6 % over 2, 8 -0.4 %;
                           // before the 4x4-block pivot inverses shrank the kernel, 3/4/8 fell off an i-cache cliff)
#endif
#ifndef PDB_GJ_MUNROLL
#define PDB_GJ_MUNROLL 2   // unroll factor of the M-pass item loop (with TUNROLL 4: +0.3 %)
#endif

#ifndef PDB_GJ_MINB
#define PDB_GJ_MINB 2   // resident 256-thread CTAs per SM the register budget is sized for
#endif

struct GjGeom {
  int r;    // matrix order
  int RP;   // padded order, multiple of 8
  int S;    // row stride (words): RP + PDB_GJ_ROWPAD, a multiple of 4
  int MS;   // matrix stride (words): RP*S + negX, padded to 16 mod 32
  int M;    // matrices per CTA iteration
  int U;    // fused DFT-8 fill: distinct u per iteration (M = 8U); 0 = off
};

#ifndef PDB_GJ_ROWPAD
#define PDB_GJ_ROWPAD 0   // extra words per matrix row (0: densest packing, most resident matrices)
#endif

__host__ __device__ constexpr int gj_row_stride(int RP) { return RP + PDB_GJ_ROWPAD; }

#ifndef PDB_REDC_ADD
#define PDB_REDC_ADD 0   // 1: additive REDC form (ptxas still emits IMAD.HI; measured 1.8 % slower)
#endif
__device__ __forceinline__ uint32_t gj_redc(uint64_t acc, const Mod32& m) {
  return PDB_REDC_ADD ? redc_add(acc, m) : redc(acc, m);
}

// REDC of a <= 9-product accumulator, canonical: two conditional subtractions.
__device__ __forceinline__ uint32_t gj_red(uint64_t acc, const Mod32& m) {
  const uint32_t v = gj_redc(acc, m);
  return csub(csub(v, 2u * m.p), m.p);
}

// REDC of <= 2 products of canonical residues: output < 1.5 p, one subtraction.
__device__ __forceinline__ uint32_t gj_red2(uint64_t acc, const Mod32& m) { return csub(gj_redc(acc, m), m.p); }

// Montgomery product of canonical a, b (Montgomery forms stay Montgomery forms).
__device__ __forceinline__ uint32_t gj_mont(uint32_t a, uint32_t b, const Mod32& m) {
  return gj_red2(mad_wide(a, b, 0ull), m);
}

__device__ __forceinline__ void gj_cp_async4(uint32_t* dst, const uint32_t* src) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void gj_cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// (i, j) walk over a square of side n without per-step division.
struct GjPos {
  int i, j, di, dj, n;
  __device__ __forceinline__ GjPos(int first, int step, int n_) : n(n_) {
    i = first / n_; j = first - i * n_; di = step / n_; dj = step - di * n_;
  }
  __device__ __forceinline__ void next() {
    i += di; j += dj;
    if (j >= n) { j -= n; ++i; }
  }
};

__device__ __forceinline__ int64_t gj_node_linear(int64_t it, int slot, const GjGeom& g, int64_t nodes) {
  const int64_t n = it * g.M + slot;
  return n < nodes ? n : -1;
}

// DFT-8 fill geometry.  The launch covers whole compact last-axis rows of
// 8 * ulast nodes (k = v * ulast + u, node u + (NL/8) v of the full axis; ulast
// = NL/8 without pruning).  Iteration `it` takes the U consecutive u-slots
// q = it * U + uu of the flattened (row, u) index, so a pair may straddle two
// rows and ulast needs no rounding to a multiple of U; a slot past the last
// row (odd rows * ulast) is a dummy: clamped reads, no output.
struct GjD8 {
  int64_t o;   // full outer index of this thread's fill slot
  int u;       // its u
};
// (row, u) of u-slot it * U + uu: one 32-bit divmod of it * U (iterations per
// launch < 2^32 / U), then at most U row wraps
__device__ __forceinline__ void gj_slot(const FusedSrc& src, int U, int64_t it, int uu, uint32_t& orel, uint32_t& u) {
  const uint32_t q0 = (uint32_t)it * (uint32_t)U, ul = (uint32_t)src.ulast;
  orel = q0 / ul;
  u = q0 - orel * ul + (uint32_t)uu;
  if (u >= ul) {   // past the row's end: one wrap unless uu >= ulast (tiny rows)
    u -= ul;
    ++orel;
    if (u >= ul) {
      orel += u / ul;
      u %= ul;
    }
  }
}
__device__ __forceinline__ GjD8 gj_d8(const FusedSrc& src, int U, int64_t it, int uu, int64_t rows) {
  uint32_t orel, u;
  gj_slot(src, U, it, uu, orel, u);
  GjD8 d;
  d.u = (int)u;
  const int64_t row = (int64_t)orel < rows ? (int64_t)orel : rows - 1;
  // full outer index of the row: a table the launcher builds for pruned maps
  d.o = src.orow_full ? __ldg(src.orow_full + row) : src.orow0 + row;
  return d;
}

// compact index (relative to the launch) of matrix slot v * U + uu of iteration it; -1 for a dummy slot
__device__ __forceinline__ int64_t gj_node_dft8(const FusedSrc& src, int64_t it, int slot, int U, int64_t rows) {
  const int v = slot / U, uu = slot - v * U;
  uint32_t orel, u;
  gj_slot(src, U, it, uu, orel, u);
  if ((int64_t)orel >= rows) return -1;
  return (int64_t)orel * 8 * src.ulast + (int64_t)v * src.ulast + u;
}

__device__ __forceinline__ int src_ulast(const FusedSrc& src) { return src.ulast; }
__device__ __forceinline__ int src_ulast(const StagedSrc&) { return 0; }

// ---- fills: the RP x RP matrices of one iteration (padding = Montgomery identity) ----
__device__ __forceinline__ void gj_fill(const StagedSrc& src, uint32_t* mats, const GjGeom& g, const int32_t* ids,
                                        int64_t it, int64_t node_lo, int64_t nodes, uint32_t one, bool dense) {
  const int r = g.r, RP = g.RP, S = g.S, M = g.M;
  const int slot = threadIdx.x % M;
  const int64_t n = gj_node_linear(it, slot, g, nodes);
  if (n >= 0) {
    const uint32_t* col = src.grids + src.node(node_lo + n);
    uint32_t* dst = mats + (size_t)slot * g.MS;
    const int first = threadIdx.x / M, step = blockDim.x / M;
    if (dense) {
      // entry_ids[p] == p, no padding: position p is grid p and smem word p
      const int64_t jump = (int64_t)step * src.stride;
      const uint32_t* s0 = col + (int64_t)first * src.stride;
      for (int q = first; q < r * r; q += step, s0 += jump) gj_cp_async4(dst + q, s0);
    } else {
      GjPos pi(first, step, RP);
      for (; pi.i < RP; pi.next()) {
        if (pi.i < r && pi.j < r) gj_cp_async4(dst + pi.i * S + pi.j, col + (int64_t)__ldg(ids + pi.i * r + pi.j) * src.stride);
        else dst[pi.i * S + pi.j] = pi.i == pi.j ? one : 0u;
      }
    }
  }
  gj_cp_async_wait_all();
}

__device__ __forceinline__ void gj_fill(const FusedSrc& src, uint32_t* mats, const GjGeom& g, const int32_t* ids,
                                        int64_t it, int64_t node_lo, int64_t nodes, uint32_t one, bool) {
  const int r = g.r, RP = g.RP, S = g.S, M = g.M;
  const int slot = threadIdx.x % M;
  const int64_t n = gj_node_linear(it, slot, g, nodes);
  if (n < 0) return;
  uint32_t* dst = mats + (size_t)slot * g.MS;
  const int64_t at = src.node(node_lo + n);
  GjPos pi(threadIdx.x / M, blockDim.x / M, RP);
  for (; pi.i < RP; pi.next())
    dst[pi.i * S + pi.j] = (pi.i < r && pi.j < r) ? src.at(__ldg(ids + pi.i * r + pi.j), at)
                                                  : (pi.i == pi.j ? one : 0u);
}

// 8 nodes per thread: f(o*NL + u + (NL/8) v) = sum_l (T_l w^(u l)) w8^(l v) for
// the slot v*U + uu.  The coefficients of one outer index o are the slab
// part[o][l][e] (entries innermost): consecutive threads read consecutive
// entries; two positions are kept in flight per thread.
template <int E>
__device__ __forceinline__ void gj_fill_dft8_e(const FusedSrc& src, uint32_t* mats, const GjGeom& g,
                                               const int32_t* ids, const GjD8& d8, uint32_t one) {
  const int r = g.r, RP = g.RP, S = g.S, U = g.U, NL = src.NL, k = src.k;
  const uint32_t p = src.p;
  const int64_t o = d8.o;
  const int step8 = NL / 8;
  uint32_t w[4], ws[4];
#pragma unroll
  for (int v = 1; v < 4; ++v) { w[v] = __ldg(src.xs + v * step8); ws[v] = __ldg(src.xss + v * step8); }
  w[0] = ws[0] = 0;
  const int uu = threadIdx.x % U;
  uint32_t tw[8], tws[8];
  {
    const int u = d8.u;
    int kk = 0;
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      if (l < E) { tw[l] = __ldg(src.xs + kk); tws[l] = __ldg(src.xss + kk); }
      else { tw[l] = tws[l] = 0; }
      kk += u;
      if (kk >= NL) kk -= NL;
    }
  }
  const size_t ms = (size_t)U * g.MS;   // slot v*U + uu
  uint32_t* base = mats + (size_t)uu * g.MS;
  const uint32_t* slab = src.part + o * (int64_t)E * k;
  GjPos pi(threadIdx.x / U, blockDim.x / U, RP);
  while (pi.i < RP) {
    const int ia = pi.i, ja = pi.j;
    pi.next();
    const int ib = pi.i, jb = pi.j;
    const bool hb = ib < RP;
    if (hb) pi.next();
    const bool ra = ia < r && ja < r, rb = hb && ib < r && jb < r;
    const uint32_t* pa = slab + (ra ? __ldg(ids + ia * r + ja) : 0);
    const uint32_t* pb = slab + (rb ? __ldg(ids + ib * r + jb) : 0);
    uint32_t ca[E], cb[E];
#pragma unroll
    for (int l = 0; l < E; ++l) { ca[l] = __ldg(pa + (int64_t)l * k); cb[l] = __ldg(pb + (int64_t)l * k); }
    uint32_t x[8];
    uint32_t* d = base + ia * S + ja;
    if (ra) {
      gj_dft8<E>(ca, tw, tws, w, ws, p, x);
#pragma unroll
      for (int v = 0; v < 8; ++v) d[v * ms] = x[v];
    } else {
      const uint32_t c = ia == ja ? one : 0u;
#pragma unroll
      for (int v = 0; v < 8; ++v) d[v * ms] = c;
    }
    if (hb) {
      d = base + ib * S + jb;
      if (rb) {
        gj_dft8<E>(cb, tw, tws, w, ws, p, x);
#pragma unroll
        for (int v = 0; v < 8; ++v) d[v * ms] = x[v];
      } else {
        const uint32_t c = ib == jb ? one : 0u;
#pragma unroll
        for (int v = 0; v < 8; ++v) d[v * ms] = c;
      }
    }
  }
}

// Dense case (entry_ids[p] == p, no padding: the C3/C5 shape): position p is
// entry p and smem word p of its matrix, so addressing is affine and four
// positions (4E coalesced loads) are kept in flight per thread.
// UC, MSC, NC > 0: compile-time U, matrix stride and r^2 (256-thread CTAs), so
// the shared-memory stores and the coefficient loads use immediate offsets.
template <int E, int UC = 0, int MSC = 0, int NC = 0>
__device__ __forceinline__ void gj_fill_dft8_dense(const FusedSrc& src, uint32_t* mats, const GjGeom& g,
                                                   const GjD8& d8) {
  const int U = UC ? UC : g.U, NL = src.NL, k = src.k, n = NC ? NC : g.r * g.r;
  const int MS = MSC ? MSC : g.MS;
  const uint32_t p = src.p;
  const int64_t o = d8.o;
  const int step8 = NL / 8;
  uint32_t w[4], ws[4];
#pragma unroll
  for (int v = 1; v < 4; ++v) { w[v] = __ldg(src.xs + v * step8); ws[v] = __ldg(src.xss + v * step8); }
  w[0] = ws[0] = 0;
  const int uu = threadIdx.x % U;
  uint32_t tw[8], tws[8];
  {
    const int u = d8.u;
    int kk = 0;
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      if (l < E) { tw[l] = __ldg(src.xs + kk); tws[l] = __ldg(src.xss + kk); }
      else { tw[l] = tws[l] = 0; }
      kk += u;
      if (kk >= NL) kk -= NL;
    }
  }
  const int ms = U * MS;
  uint32_t* base = mats + uu * MS;
  const uint32_t* slab = src.part + o * (int64_t)E * k;
  const int step = UC ? 256 / UC : blockDim.x / U;
#ifndef PDB_GJ_FILLF
#define PDB_GJ_FILLF 6   // measured at the end of round 2: 6 +0.9 % over 4; 2, 3, 8 slower
#endif
  constexpr int F = PDB_GJ_FILLF;   // positions in flight
  int p0 = threadIdx.x / U;
  // one pointer per coefficient row, advanced by a constant: F*E loads per
  // round from E registers with immediate offsets when the geometry is static
  const uint32_t* sp[E];
#pragma unroll
  for (int l = 0; l < E; ++l) sp[l] = slab + (int64_t)l * k + p0;
  for (; p0 + (F - 1) * step < n; p0 += F * step) {
    uint32_t c[F][E];
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
      for (int l = 0; l < E; ++l) c[f][l] = __ldg(sp[l] + f * step);
#pragma unroll
    for (int l = 0; l < E; ++l) sp[l] += F * step;
#pragma unroll
    for (int f = 0; f < F; ++f) {
      uint32_t x[8];
      gj_dft8<E>(c[f], tw, tws, w, ws, p, x);
      uint32_t* d = base + p0 + f * step;
#pragma unroll
      for (int v = 0; v < 8; ++v) d[v * ms] = x[v];
    }
  }
  for (; p0 < n; p0 += step) {   // tail: single positions
    uint32_t c[E];
#pragma unroll
    for (int l = 0; l < E; ++l) { c[l] = __ldg(sp[l]); sp[l] += step; }
    uint32_t x[8];
    gj_dft8<E>(c, tw, tws, w, ws, p, x);
#pragma unroll
    for (int v = 0; v < 8; ++v) base[v * ms + p0] = x[v];
  }
}

// UC/MSC/NC: compile-time dense-fill geometry (0 = from g), see gj_fill_dft8_dense
template <int UC = 0, int MSC = 0, int NC = 0>
__device__ __forceinline__ void gj_fill_dft8(const FusedSrc& src, uint32_t* mats, const GjGeom& g, const int32_t* ids,
                                             const GjD8& d8, uint32_t one, bool dense) {
  if (dense) {
    switch (src.E) {
      case 1: gj_fill_dft8_dense<1, UC, MSC, NC>(src, mats, g, d8); return;
      case 2: gj_fill_dft8_dense<2, UC, MSC, NC>(src, mats, g, d8); return;
      case 3: gj_fill_dft8_dense<3, UC, MSC, NC>(src, mats, g, d8); return;
      case 4: gj_fill_dft8_dense<4, UC, MSC, NC>(src, mats, g, d8); return;
      case 5: gj_fill_dft8_dense<5, UC, MSC, NC>(src, mats, g, d8); return;
      case 6: gj_fill_dft8_dense<6, UC, MSC, NC>(src, mats, g, d8); return;
      case 7: gj_fill_dft8_dense<7, UC, MSC, NC>(src, mats, g, d8); return;
      default: gj_fill_dft8_dense<8, UC, MSC, NC>(src, mats, g, d8); return;
    }
  }
  switch (src.E) {
    case 1: gj_fill_dft8_e<1>(src, mats, g, ids, d8, one); break;
    case 2: gj_fill_dft8_e<2>(src, mats, g, ids, d8, one); break;
    case 3: gj_fill_dft8_e<3>(src, mats, g, ids, d8, one); break;
    case 4: gj_fill_dft8_e<4>(src, mats, g, ids, d8, one); break;
    case 5: gj_fill_dft8_e<5>(src, mats, g, ids, d8, one); break;
    case 6: gj_fill_dft8_e<6>(src, mats, g, ids, d8, one); break;
    case 7: gj_fill_dft8_e<7>(src, mats, g, ids, d8, one); break;
    default: gj_fill_dft8_e<8>(src, mats, g, ids, d8, one); break;
  }
}

// ---- T pass: A22 <- c*A22 + A21*negM over TR x TC tiles ------------------------------
template <int TC>
__device__ __forceinline__ void gj_ld(const uint32_t* a, uint32_t (&v)[TC]) {
  if constexpr (TC % 4 == 0) {
#pragma unroll
    for (int b = 0; b < TC; b += 4) {
      const uint4 x = *reinterpret_cast<const uint4*>(a + b);
      v[b] = x.x; v[b + 1] = x.y; v[b + 2] = x.z; v[b + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int b = 0; b < TC; b += 2) {
      const uint2 x = *reinterpret_cast<const uint2*>(a + b);
      v[b] = x.x; v[b + 1] = x.y;
    }
  }
}

template <int TC>
__device__ __forceinline__ void gj_st(uint32_t* a, const uint32_t (&v)[TC]) {
  if constexpr (TC % 4 == 0) {
#pragma unroll
    for (int b = 0; b < TC; b += 4) *reinterpret_cast<uint4*>(a + b) = make_uint4(v[b], v[b + 1], v[b + 2], v[b + 3]);
  } else {
#pragma unroll
    for (int b = 0; b < TC; b += 2) *reinterpret_cast<uint2*>(a + b) = make_uint2(v[b], v[b + 1]);
  }
}

// TC-word row segment with its two 16-byte halves rotated by sw (0 or 4 words, TC == 8 only)
template <int TC>
__device__ __forceinline__ void gj_ld_sw(const uint32_t* a, int sw, uint32_t (&v)[TC]) {
  if constexpr (TC == 8) {
    const uint4 x = *reinterpret_cast<const uint4*>(a + sw);
    const uint4 y = *reinterpret_cast<const uint4*>(a + (4 - sw));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
  } else {
    gj_ld<TC>(a, v);
  }
}

template <int TC>
__device__ __forceinline__ void gj_st_sw(uint32_t* a, int sw, const uint32_t (&v)[TC]) {
  if constexpr (TC == 8) {
    *reinterpret_cast<uint4*>(a + sw) = make_uint4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<uint4*>(a + (4 - sw)) = make_uint4(v[4], v[5], v[6], v[7]);
  } else {
    gj_st<TC>(a, v);
  }
}

// REDC of a <= 17-product accumulator (paired pivot blocks), canonical.  Valid
// for p < PDB_PAIR_PMAX (gj_pair_ok): 17 (p-1)^2 < 2^64, and subtracting 2p from
// hi(acc) (acc - 2p 2^32 == acc mod p) brings hi below 2^32 - p as REDC needs.
__device__ __forceinline__ uint32_t gj_red17(uint64_t acc, const Mod32& m) {
  const uint32_t lo = (uint32_t)acc;
  const uint32_t hi = csub((uint32_t)(acc >> 32), 2u * m.p);
  const uint32_t v = hi + m.p - umulhi32(lo * m.qinv, m.p);
  return csub(csub(v, 2u * m.p), m.p);
}

// One TR x TC tile of the trailing update A[i0.., cc..] <- c*A + A[i0.., K..K+B-1] * negM[K..K+B-1][cc..].
// P31: 2^30 <= p < 2^31 -- at most two products per reduction (2 p^2 < 2^63 keeps
// hi(acc) + p < 2^32); the partial results are summed mod p.  W17: B = 16 products
// (two pivot blocks) + the scale in one accumulator, reduced by gj_red17.
template <int TR, int TC, bool P31, int B, bool W17 = false>
__device__ __forceinline__ void gj_ttile(uint32_t* A, int S, int K, int i0, int cc, int sw, uint32_t cR,
                                         const Mod32& m) {
  const uint32_t* npr = A + K * S;    // negM rows K..K+B-1
  uint32_t a21[TR][B];
  uint64_t acc[TR][TC];
#pragma unroll
  for (int a = 0; a < TR; ++a) {
    const uint32_t* row = A + (i0 + a) * S;
    gj_ld<B>(row + K, a21[a]);
    uint32_t v[TC];
    gj_ld_sw<TC>(row + cc, sw, v);
#pragma unroll
    for (int b = 0; b < TC; ++b) acc[a][b] = mad_wide(v[b], cR, 0ull);
  }
  uint32_t sum[TR][TC];
#pragma unroll
  for (int q = 0; q < B; ++q) {
    uint32_t nm[TC];
    gj_ld_sw<TC>(npr + q * S + cc, sw, nm);
#pragma unroll
    for (int a = 0; a < TR; ++a)
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        const bool fresh = P31 && (q & 1);                   // q = 1, 3, 5, 7 open a new pair
        acc[a][b] = mad_wide(a21[a][q], nm[b], fresh ? 0ull : acc[a][b]);
        if (P31 && (q % 2 == 0 || q == B - 1)) {         // fold after q = 0, 2, 4, ..., B-1
          const uint32_t v = gj_red2(acc[a][b], m);
          sum[a][b] = q == 0 ? v : add_mod(sum[a][b], v, m.p);
        }
      }
  }
#pragma unroll
  for (int a = 0; a < TR; ++a) {
    uint32_t v[TC];
#pragma unroll
    for (int b = 0; b < TC; ++b) v[b] = P31 ? sum[a][b] : (W17 ? gj_red17(acc[a][b], m) : gj_red(acc[a][b], m));
    gj_st_sw<TC>(A + (i0 + a) * S + cc, sw, v);
  }
}

template <int TR, int TC, int LPM, bool P31, int B = GJ_B, bool W17 = false>
__device__ __forceinline__ void gj_tpass(uint32_t* A, int S, int K, int mrem, uint32_t cR, int l, const Mod32& m) {
  const int c0 = K + B;
  const int ntc = mrem / TC;
  const int tiles = (mrem / TR) * ntc;
  int ti = l / ntc, tc = l - (l / ntc) * ntc;
  const int dti = LPM / ntc, dtc = LPM - (LPM / ntc) * ntc;
  PDB_UNROLL(PDB_GJ_TUNROLL)
  for (int w = l; w < tiles; w += LPM) {
    // 8-wide tiles: odd tile rows visit their two 16-byte chunks in swapped order,
    // so the 8 lanes of a quarter-warp (two tile rows x four column tiles) hit 8
    // distinct bank groups; column v of this lane's tile is physical column
    // cc + ((v + sw) mod 8).
    const int sw = (TC == 8 && (ti & 1)) ? 4 : 0;
    gj_ttile<TR, TC, P31, B, W17>(A, S, K, c0 + TR * ti, c0 + TC * tc, sw, cR, m);
    ti += dti; tc += dtc;
    if (tc >= ntc) { tc -= ntc; ++ti; }
  }
}

// Trailing update of a 24 x 24 region at (c0, c0) with 16 lanes and no idle
// lane: 64 2x4 tiles (4 passes: rows c0..c0+23 x columns c0..c0+19, and rows
// c0+16..c0+23 x columns c0+20..c0+23) and 16 1x4 tiles (one pass: rows
// c0..c0+15 x columns c0+20..c0+23), instead of 72 2x4 tiles in 4.5 passes.
template <bool P31, int B, bool W17 = false>
__device__ __forceinline__ void gj_tpass24(uint32_t* A, int S, int K, int c0, uint32_t cR, int l, const Mod32& m) {
  PDB_UNROLL(PDB_GJ_TUNROLL)
  for (int w = l; w < 64; w += 16) {
    const bool main = w < 60;
    const int i0 = c0 + (main ? 2 * (w / 5) : 16 + 2 * (w - 60));
    const int cc = c0 + (main ? 4 * (w % 5) : 20);
    gj_ttile<2, 4, P31, B, W17>(A, S, K, i0, cc, 0, cR, m);
  }
  gj_ttile<1, 4, P31, B, W17>(A, S, K, c0 + l, c0 + 20, 0, cR, m);
}

// First block of a pivot pair: the trailing update of block K restricted to the
// panel the next block reads -- its pivot rows K+8..K+15 (all trailing columns)
// and the column strip K+8..K+15 of the rows below.  The rest of the trailing
// matrix is updated once for both blocks (gj_tpass<..., 16, true>).
// Panel of block K with 32 trailing columns and 16 lanes, no idle lane: 48 2x4
// tiles (rows c0..c0+7 x 32 columns, rows c0+8..c0+23 x columns c0..c0+7) in 3
// passes and 16 1x4 tiles (rows c0+24..c0+31 x columns c0..c0+7) in one.
__device__ __forceinline__ void gj_tpass_panel32(uint32_t* A, int S, int K, uint32_t cR, int l, const Mod32& m) {
  const int c0 = K + GJ_B;
#pragma unroll
  for (int w = l; w < 48; w += 16) {
    const bool top = w < 32;
    const int i0 = c0 + (top ? 2 * (w >> 3) : GJ_B + 2 * ((w - 32) >> 1));
    const int cc = c0 + (top ? 4 * (w & 7) : 4 * (w & 1));
    gj_ttile<2, 4, false, GJ_B>(A, S, K, i0, cc, 0, cR, m);
  }
  gj_ttile<1, 4, false, GJ_B>(A, S, K, c0 + 24 + (l >> 1), c0 + 4 * (l & 1), 0, cR, m);
}

template <int TR, int TC, int LPM>
__device__ __forceinline__ void gj_tpass_panel(uint32_t* A, int S, int K, int mrem, uint32_t cR, int l,
                                               const Mod32& m) {
  const int c0 = K + GJ_B;
  const int n1c = mrem / TC;
  const int t1 = (GJ_B / TR) * n1c;                          // rows c0..c0+7, every trailing column
  constexpr int n2c = GJ_B / TC;
  const int t2 = ((mrem - GJ_B) / TR) * n2c;                 // rows c0+8.., columns c0..c0+7
  for (int w = l; w < t1 + t2; w += LPM) {
    int i0, cc;
    if (w < t1) {
      i0 = c0 + TR * (w / n1c);
      cc = c0 + TC * (w % n1c);
    } else {
      const int w2 = w - t1;
      i0 = c0 + GJ_B + TR * (w2 / n2c);
      cc = c0 + TC * (w2 % n2c);
    }
    gj_ttile<TR, TC, false, GJ_B>(A, S, K, i0, cc, 0, cR, m);
  }
}

// negM rows K..K+7, columns c0.. (RP - c0 words each, a multiple of 4) scaled by cR (Montgomery form)
template <int LPM>
__device__ __forceinline__ void gj_scale_rows(uint32_t* A, int S, int K, int c0, int ncols, uint32_t cR, int l,
                                              const Mod32& m) {
  const int per_row = ncols / 4;
#pragma unroll
  for (int w = l; w < GJ_B * per_row; w += LPM) {
    uint32_t* a = A + (K + w / per_row) * S + c0 + 4 * (w % per_row);
    uint32_t v[4];
    gj_ld<4>(a, v);
#pragma unroll
    for (int b = 0; b < 4; ++b) v[b] = gj_mont(v[b], cR, m);
    gj_st<4>(a, v);
  }
}

template <int LPM, bool P31, int B = GJ_B>
__device__ __forceinline__ void gj_tpass_any(uint32_t* A, int S, int K, int mrem, uint32_t cR, int l, const Mod32& m) {
  // largest tile that keeps >= ~70 % of the lanes busy
  // fraction of lane slots busy >= pct/100, in integers
  auto util = [&](int tr, int tc, int pct) {
    const int t = (mrem / tr) * (mrem / tc);
    const int passes = (t + LPM - 1) / LPM;
    return 100 * t >= pct * passes * LPM;
  };
  // 2x8 tiles need ~70 registers: only when fewer than 4 CTAs share an SM
  constexpr int minb = PDB_GJ_MINB;
#ifndef PDB_GJ_T28
#define PDB_GJ_T28 0   // 2x8 trailing tiles: more reuse but spills at 128 registers (measured slower)
#endif
#ifndef PDB_GJ_T44
#define PDB_GJ_T44 0   // 4x4 trailing tiles (experiment)
#endif
  if (PDB_GJ_T28 && minb < 4 && util(2, 8, 70)) gj_tpass<2, 8, LPM, P31, B>(A, S, K, mrem, cR, l, m);
  else if (PDB_GJ_T44 && util(4, 4, 70)) gj_tpass<4, 4, LPM, P31, B>(A, S, K, mrem, cR, l, m);
  else if (util(2, 4, 70)) gj_tpass<2, 4, LPM, P31, B>(A, S, K, mrem, cR, l, m);
  else if (util(1, 4, 70)) gj_tpass<1, 4, LPM, P31, B>(A, S, K, mrem, cR, l, m);
  else gj_tpass<1, 2, LPM, P31, B>(A, S, K, mrem, cR, l, m);
}

// ---- M pass: negM[j][c] = sum_q negX[j][q] A12[q][c], in place in pivot rows K..K+7 ----
// Register tiles of RPI rows x TC columns per lane: one item reads the 8 x TC
// block of A12 and RPI rows of negX (16 B loads) for RPI*TC*8 MACs.  Items are
// numbered column-group major, so the lanes sharing a column group work in the
// same pass; they read it completely before any of them overwrites it.
// ---- P: division-free Gauss-Jordan on a B x B pivot block ----------------------------
// Lane l holds EPL = B / (LPM / B) entries of row pj, columns pc..pc+EPL-1.  On
// return v holds X with X * A11 = lam * I (lam = prod of the pivots z_s); zl is
// lambda_pj (the pivot prefix product when row pj was the pivot row) and zlast
// the last pivot, so det(A11) = zlast / (lambda_1 ... lambda_{B-2}).  lam == 0
// iff a pivot vanished.  GE: only the pivots are needed (last block): dead
// columns are skipped.
struct GjPiv {
  uint32_t lam, zl, zlast;
};
template <int B, int LPM, bool LAZY, int EPL>
__device__ __forceinline__ GjPiv gj_gauss_jordan(uint32_t (&v)[EPL], int pj, int pc, int l, unsigned omask, bool ge,
                                                 const Mod32& m) {
  constexpr int LPR = LPM / B;
  static_assert(EPL == B / LPR, "entries per lane");
  const uint32_t p = m.p, one = m.r1;
  auto lazy_canon = [&](uint32_t x) { return LAZY ? csub(x, p) : x; };
  uint32_t lam = one, zl = one, zlast = one;
#pragma unroll
  for (int s = 0; s < B; ++s) {
    // LAZY: pivot-block entries stay in [0, 2p) between steps (only the shuffled
    // pivot z and multiplier t are made canonical): with zz, nn <= p and a, b < 2p
    // the two products sum below 4 p^2, so REDC returns < hi + p < 2p (p < 2^30)
    const uint32_t z = lazy_canon(__shfl_sync(omask, v[s % EPL], s * LPR + s / EPL, LPM));
    const uint32_t t = lazy_canon(__shfl_sync(omask, v[s % EPL], pj * LPR + s / EPL, LPM));
    // last block (no trailing rows): only det(A11) is needed, i.e. the pivots --
    // Gaussian elimination suffices, and column slots k whose column is <= s in
    // every lane of the group (B - EPL + k <= s) are dead from step s on
    auto live = [&](int k) { return !ge || B - EPL + k > s; };
    uint32_t prow[EPL];
#pragma unroll
    for (int k = 0; k < EPL; ++k)
      if (live(k)) prow[k] = __shfl_sync(omask, v[k], s * LPR + l % LPR, LPM);
    // Other rows: z v - t prow, with -t lam at column s (the identity column of
    // row s is lam there).  Row s is scaled by lam = prod_{t<s} z_t instead
    // (lam * v; lam^2 at column s): then every row ends up scaled by c =
    // prod z overall, so the in-place inverse part is X = c A11^-1 itself.
    const bool piv = pj == s;
    zl = piv ? lam : zl;
    const uint32_t zz = piv ? lam : z;
    const uint32_t nn = piv ? 0u : p - t;   // p - t in (0, p]: a valid 2-product multiplier
#pragma unroll
    for (int k = 0; k < EPL; ++k) {
      if (!live(k)) continue;
      uint32_t a = v[k], b = prow[k];
      if (k == s % EPL) {   // the only element of this lane that can sit in column s
        const bool diag = pc == s - s % EPL;
        a = diag ? (piv ? lam : 0u) : a;
        b = diag ? lam : b;
      }
      const uint64_t acc = mad_wide(zz, a, mad_wide(nn, b, 0ull));
      v[k] = LAZY ? gj_redc(acc, m) : gj_red2(acc, m);
    }
    if (s == B - 1) zlast = z;
    lam = gj_mont(lam, z, m);
  }
  return {lam, zl, zlast};
}

// ---- 4x4 adjugate, one entry per lane of a 16-lane group ------------------------------
// M: 4x4 in shared memory (row stride S).  Lanes 0..11 form the 2x2 minors of
// rows (0, 1) (index q) and rows (2, 3) (6 + q) for the column pairs q = (0,1),
// (0,2), (0,3), (1,2), (1,3), (2,3); lane (i, j) then expands the cofactor of
// entry (j, i) along the partner row j^1:
//   adj_ij = sum_{t<3} (-1)^(i+j+t) M[j^1][k_t] * minor(other row pair, columns {0..3} \ {i, k_t}),
// k_t the t-th column other than i (table checked against the adjugate identity
// adj M = det(M) I on random matrices).  det(M) = sum_t M[0][t] adj[t][0].
// Returns adj_ij (canonical); det in every lane.  mins: 12 words of scratch.
__device__ __forceinline__ uint32_t gj_adj4(const uint32_t* M, int S, uint32_t* mins, int l, unsigned omask,
                                           const Mod32& m, uint32_t& det) {
  const uint32_t p = m.p;
  const int i = l >> 2, j = l & 3;
  if (l < 12) {
    const int q = l < 6 ? l : l - 6;
    const int ca = q < 3 ? 0 : (q < 5 ? 1 : 2), cb = q < 3 ? q + 1 : (q < 5 ? q - 1 : 3);
    const uint32_t* R0 = M + (l < 6 ? 0 : 2) * S;
    const uint32_t* R1 = R0 + S;
    mins[l] = gj_red2(mad_wide(R0[ca], R1[cb], mad_wide(p - R1[ca], R0[cb], 0ull)), m);
  }
  __syncwarp(omask);
  const uint32_t* R = M + (j ^ 1) * S;
  const int off = j < 2 ? 6 : 0;
  uint64_t acc = 0;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const int k = t + (t >= i);
    const int a = i < k ? i : k, b = i < k ? k : i;
    const int mu = off + 5 - (a + b - 1 + (a > 0));   // complement of the column pair {a, b}
    const uint32_t e = R[k];
    acc = mad_wide(((i + j + t) & 1) ? p - e : e, mins[mu], acc);   // p - e <= p: a valid multiplier
  }
  const uint32_t adj = gj_red2(acc, m);
  uint32_t row0[4];
  gj_ld<4>(M, row0);
  uint64_t d = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) d = mad_wide(row0[t], __shfl_sync(omask, adj, 4 * t, 16), d);
  det = gj_red(d, m);
  return adj;
}

// det(M) of a 4x4 in shared memory from its 2x2 minors (Laplace expansion by
// rows (0, 1) and (2, 3)): s0 c5 - s1 c4 + s2 c3 + s3 c2 - s4 c1 + s5 c0.  Every lane gets it.
__device__ __forceinline__ uint32_t gj_det4(const uint32_t* M, int S, uint32_t* mins, int l, unsigned omask,
                                           const Mod32& m) {
  const uint32_t p = m.p;
  if (l < 12) {
    const int q = l < 6 ? l : l - 6;
    const int ca = q < 3 ? 0 : (q < 5 ? 1 : 2), cb = q < 3 ? q + 1 : (q < 5 ? q - 1 : 3);
    const uint32_t* R0 = M + (l < 6 ? 0 : 2) * S;
    const uint32_t* R1 = R0 + S;
    mins[l] = gj_red2(mad_wide(R0[ca], R1[cb], mad_wide(p - R1[ca], R0[cb], 0ull)), m);
  }
  __syncwarp(omask);
  uint32_t v[12];
  gj_ld<4>(mins, *reinterpret_cast<uint32_t(*)[4]>(v));
  gj_ld<4>(mins + 4, *reinterpret_cast<uint32_t(*)[4]>(v + 4));
  gj_ld<4>(mins + 8, *reinterpret_cast<uint32_t(*)[4]>(v + 8));
  uint64_t acc = mad_wide(v[0], v[11], 0ull);
  acc = mad_wide(p - v[1], v[10], acc);
  acc = mad_wide(v[2], v[9], acc);
  acc = mad_wide(v[3], v[8], acc);
  acc = mad_wide(p - v[4], v[7], acc);
  acc = mad_wide(v[5], v[6], acc);
  return gj_red(acc, m);
}

// ---- P by 4x4 blocks (8x8 pivot block, 16 lanes: one 4x4 entry per lane) --------------
// A11 = [[A, B], [C, D]].  X_A = adj(A) (= a A^-1, a = det A), N = -X_A B,
// S = a D + C N = a Sigma (Sigma = D - C A^-1 B), X_S = adj(S) (= s S^-1,
// s = det S), then X = c A11^-1 with c = a s from the block inverse:
//   Y = a X_S = s Sigma^-1,  X22 = a Y,  X12 = N Y,  Z = X_S (C X_A),
//   X21 = -a Z,  X11 = s X_A - N Z.
// Two adjugates (gj_adj4: 2 + 3 + 4 products per lane, no elimination chain)
// plus six 4x4 products with one reduction per 4-5 products, against 8
// elimination steps of 2 products and a reduction per entry.
// det(A11) = det(A) det(Sigma) = a s / a^4: num *= s, and the a's are
// collected in aprod (den *= aprod^3 once per node).  Scratch: X_A and N in
// negX rows 0-3, the minors in negX row 4, then the dead pivot block itself.
// Returns false if A or Sigma is singular (the node goes to det_robust).
__device__ __forceinline__ bool gj_pinv44(uint32_t* A, uint32_t* NX, int S, int K, int l, unsigned omask,
                                          const Mod32& m, uint32_t& num, uint32_t& aprod, uint32_t& cR) {
  const uint32_t p = m.p;
  const int i = l >> 2, j = l & 3;
  uint32_t* P0 = A + K * S + K;   // the pivot block, row stride S
  auto neg = [&](uint32_t x) { return x ? p - x : 0u; };
  // X_A = adj(A), a = det(A)
  uint32_t aR;
  const uint32_t xa = gj_adj4(P0, S, NX + gj_nx_row(4), l, omask, m, aR);
  if (aR == 0) return false;
  uint32_t crow[4];
  gj_ld<4>(P0 + (4 + i) * S, crow);
  const uint32_t dv = P0[(4 + i) * S + 4 + j];
  NX[i * GJ_B + j] = xa;
  __syncwarp(omask);
  // N = -X_A B (negX rows 0-3, columns 4-7) and P1 = C X_A (the C position: C is in registers)
  {
    uint32_t xr[4];
    gj_ld<4>(NX + i * GJ_B, xr);
    uint64_t an = 0, ap = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      an = mad_wide(xr[q], P0[q * S + 4 + j], an);
      ap = mad_wide(crow[q], NX[q * GJ_B + j], ap);
    }
    NX[i * GJ_B + 4 + j] = neg(gj_red(an, m));
    P0[(4 + i) * S + j] = gj_red(ap, m);   // every C row was read before the last __syncwarp
  }
  __syncwarp(omask);
  // S = a D + C N at the A position
  {
    uint64_t acc = mad_wide(dv, aR, 0ull);
#pragma unroll
    for (int q = 0; q < 4; ++q) acc = mad_wide(crow[q], NX[q * GJ_B + 4 + j], acc);
    P0[i * S + j] = gj_red(acc, m);
  }
  __syncwarp(omask);
  // X_S = adj(S), s = det(S); X_S at the D position, Y = a X_S at the B position (both dead)
  uint32_t sR;
  const uint32_t xs = gj_adj4(P0, S, NX + gj_nx_row(4), l, omask, m, sR);
  if (sR == 0) return false;
  const uint32_t y = gj_mont(xs, aR, m);
  P0[(4 + i) * S + 4 + j] = xs;
  P0[i * S + 4 + j] = y;
  __syncwarp(omask);
  uint32_t zp;
  {
    uint32_t xr[4];                        // Z = X_S P1, -Z at the A position (S is dead)
    gj_ld<4>(P0 + (4 + i) * S + 4, xr);
    uint64_t acc = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) acc = mad_wide(xr[q], P0[(4 + q) * S + j], acc);
    zp = gj_red(acc, m);
  }
  P0[i * S + j] = neg(zp);
  __syncwarp(omask);
  uint32_t x11, x12;
  {
    uint32_t nr[4];                        // X12 = N Y, X11 = s X_A + N (-Z)
    gj_ld<4>(NX + i * GJ_B + 4, nr);
    uint64_t a12 = 0, a11 = mad_wide(xa, sR, 0ull);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a12 = mad_wide(nr[q], P0[q * S + 4 + j], a12);
      a11 = mad_wide(nr[q], P0[q * S + j], a11);
    }
    x12 = gj_red(a12, m);
    x11 = gj_red(a11, m);
  }
  __syncwarp(omask);
  NX[gj_nx_row(i) + j] = neg(x11);
  NX[gj_nx_row(i) + 4 + j] = neg(x12);
  NX[gj_nx_row(4 + i) + j] = gj_mont(zp, aR, m);            // -X21 = a Z
  NX[gj_nx_row(4 + i) + 4 + j] = gj_mont(y, neg(aR), m);    // -X22 = -a Y
  // det(A11) = det(A) det(Sigma) = a s / a^4
  num = gj_mont(num, sR, m);
  aprod = gj_mont(aprod, aR, m);
  cR = gj_mont(aR, sR, m);
  return true;
}

// Last pivot block (no trailing rows): det(A11) only, = det(A) det(S) / a^4 with
// S = a D - C adj(A) B as in gj_pinv44 (num *= det S, aprod *= a), instead of
// eight elimination steps.  false: A or Sigma singular (det_robust decides).
__device__ __forceinline__ bool gj_pdet44(uint32_t* A, uint32_t* NX, int S, int K, int l, unsigned omask,
                                          const Mod32& m, uint32_t& num, uint32_t& aprod) {
  const uint32_t p = m.p;
  const int i = l >> 2, j = l & 3;
  uint32_t* P0 = A + K * S + K;
  uint32_t aR;
  const uint32_t xa = gj_adj4(P0, S, NX + gj_nx_row(4), l, omask, m, aR);
  if (aR == 0) return false;
  uint32_t crow[4];
  gj_ld<4>(P0 + (4 + i) * S, crow);
  const uint32_t dv = P0[(4 + i) * S + 4 + j];
  NX[i * GJ_B + j] = xa;
  __syncwarp(omask);
  {
    uint32_t xr[4];                        // N = -X_A B
    gj_ld<4>(NX + i * GJ_B, xr);
    uint64_t acc = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) acc = mad_wide(xr[q], P0[q * S + 4 + j], acc);
    const uint32_t x = gj_red(acc, m);
    NX[i * GJ_B + 4 + j] = x ? p - x : 0u;
  }
  __syncwarp(omask);
  {
    uint64_t acc = mad_wide(dv, aR, 0ull); // S = a D + C N at the A position
#pragma unroll
    for (int q = 0; q < 4; ++q) acc = mad_wide(crow[q], NX[q * GJ_B + 4 + j], acc);
    P0[i * S + j] = gj_red(acc, m);
  }
  __syncwarp(omask);
  const uint32_t sR = gj_det4(P0, S, NX + gj_nx_row(4), l, omask, m);
  if (sR == 0) return false;
  num = gj_mont(num, sR, m);
  aprod = gj_mont(aprod, aR, m);
  return true;
}

// One M-pass item: rows rg*RPI.. of negM, columns c..c+TC-1 (reads negX and the
// 8 x TC block of A12 at column c; the caller stores after a __syncwarp).
template <int RPI, int TC, bool P31, int B>
__device__ __forceinline__ void gj_mitem(const uint32_t* A, const uint32_t* NX, int S, int K, int c, int rg,
                                         uint32_t (&res)[RPI][TC], const Mod32& m) {
  uint32_t x[RPI][B];   // this item's negX rows, 16 B loads
#pragma unroll
  for (int t = 0; t < RPI; ++t) gj_ld<B>(NX + gj_nx_row(rg * RPI + t), x[t]);
  uint64_t acc[RPI][TC];
#pragma unroll
  for (int q = 0; q < B; ++q) {
    uint32_t a[TC];
    gj_ld<TC>(A + (K + q) * S + c, a);
#pragma unroll
    for (int t = 0; t < RPI; ++t)
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        const bool fresh = q == 0 || (P31 && q % 2 == 0);
        acc[t][b] = mad_wide(x[t][q], a[b], fresh ? 0ull : acc[t][b]);
        if (P31 && (q & 1)) {                              // fold pairs (0,1), (2,3), ...
          const uint32_t v = gj_red2(acc[t][b], m);
          res[t][b] = q == 1 ? v : add_mod(res[t][b], v, m.p);
        }
      }
  }
  if (!P31) {
#pragma unroll
    for (int t = 0; t < RPI; ++t)
#pragma unroll
      for (int b = 0; b < TC; ++b) res[t][b] = gj_red(acc[t][b], m);
  }
}

template <int RPI, int TC, int LPM, bool P31, int B = GJ_B>
__device__ __forceinline__ void gj_mpass(uint32_t* A, const uint32_t* NX, int S, int K, int mrem, int l,
                                         unsigned omask, const Mod32& m) {
  constexpr int NRG = B / RPI;
  const int items = (mrem / TC) * NRG;
  PDB_UNROLL(PDB_GJ_MUNROLL)
  for (int w0 = 0; w0 < items; w0 += LPM) {
    const int w = w0 + l;
    const bool act = w < items;
    const int cg = w / NRG, rg = w - (w / NRG) * NRG;
    const int c = K + B + TC * cg;
    uint32_t res[RPI][TC];
    if (act) gj_mitem<RPI, TC, P31, B>(A, NX, S, K, c, rg, res, m);
    if (NRG > 1) __syncwarp(omask);
    if (act) {
#pragma unroll
      for (int t = 0; t < RPI; ++t) gj_st<TC>(A + (K + rg * RPI + t) * S + c, res[t]);
    }
  }
}

// M pass over 24 trailing columns with 16 lanes and no idle lane: one pass of
// 2x4 items over columns 0..15, one of 1x4 items over columns 16..23 (2x4 items
// alone need 1.5 passes, and a pass costs its full issue whatever the lanes do).
template <bool P31, int B = GJ_B>
__device__ __forceinline__ void gj_mpass24(uint32_t* A, const uint32_t* NX, int S, int K, int l, unsigned omask,
                                           const Mod32& m) {
  {
    const int rg = l & 3, c = K + B + 4 * (l >> 2);
    uint32_t res[2][4];
    gj_mitem<2, 4, P31, B>(A, NX, S, K, c, rg, res, m);
    __syncwarp(omask);
    gj_st<4>(A + (K + 2 * rg) * S + c, res[0]);
    gj_st<4>(A + (K + 2 * rg + 1) * S + c, res[1]);
  }
  {
    const int rg = l & 7, c = K + B + 16 + 4 * (l >> 3);
    uint32_t res[1][4];
    gj_mitem<1, 4, P31, B>(A, NX, S, K, c, rg, res, m);
    __syncwarp(omask);
    gj_st<4>(A + (K + rg) * S + c, res[0]);
  }
}

template <int LPM, bool P31, int B = GJ_B>
__device__ __forceinline__ void gj_mpass_any(uint32_t* A, const uint32_t* NX, int S, int K, int mrem, int l,
                                             unsigned omask, const Mod32& m) {
  auto util = [&](int rpi, int tc, int pct) {
    const int t = (mrem / tc) * (B / rpi);
    return 100 * t >= pct * ((t + LPM - 1) / LPM) * LPM;
  };
#ifndef PDB_GJ_M44
#define PDB_GJ_M44 0   // 4x4 M-pass tiles (measured slower than 2x4 at 128 registers)
#endif
  if (PDB_GJ_M44 && util(4, 4, 74)) gj_mpass<4, 4, LPM, P31, B>(A, NX, S, K, mrem, l, omask, m);
  else if (util(2, 4, 74)) gj_mpass<2, 4, LPM, P31, B>(A, NX, S, K, mrem, l, omask, m);
  else if (util(4, 2, 74)) gj_mpass<4, 2, LPM, P31, B>(A, NX, S, K, mrem, l, omask, m);
  else if (util(1, 4, 74)) gj_mpass<1, 4, LPM, P31, B>(A, NX, S, K, mrem, l, omask, m);
  else if (util(2, 2, 74)) gj_mpass<2, 2, LPM, P31, B>(A, NX, S, K, mrem, l, omask, m);
  else gj_mpass<1, 2, LPM, P31, B>(A, NX, S, K, mrem, l, omask, m);
}

// f(integral_constant<int, K>) for K = FIRST, FIRST + STEP, ... < END: a loop whose
// unrolling does not depend on the compiler's heuristics (the block loop of the
// compile-time-order kernels must unroll so every shared-memory offset is an immediate)
template <int K, int END, int STEP, class F>
__device__ __forceinline__ void gj_unrolled(F&& f) {
  if constexpr (K < END) {
    f(std::integral_constant<int, K>{});
    gj_unrolled<K + STEP, END, STEP>(f);
  }
}

// ---- the kernel ------------------------------------------------------------------------------
#ifndef PDB_GJ_P44
#define PDB_GJ_P44 1   // 8x8 pivot blocks with trailing rows inverted by 4x4 blocks (gj_pinv44)
#endif
#ifndef PDB_GJ_LAZYP
#define PDB_GJ_LAZYP 1   // pivot-block entries in [0, 2p) between Gauss-Jordan steps (p < 2^30)
#endif
#ifndef PDB_GJ_GELAST
#define PDB_GJ_GELAST 1   // last pivot block: elimination without the Gauss-Jordan back part
#endif
#ifndef PDB_GJ_ABL
#define PDB_GJ_ABL 0   // profiling ablation only (1: no M pass, 2: no T pass, 3: one fill per CTA); results are wrong
#endif
// RPC > 0: the padded order is the compile-time constant RPC (row stride
// gj_row_stride(RPC)); the block loop unrolls, every pass sees a constant
// trailing size, and all shared-memory addressing folds into immediates.
// PAIR: the first two pivot blocks share one trailing update (17 products per
// reduction, p < PDB_PAIR_PMAX; compile-time orders RPC >= 32 only).
// Order-16 kernels are latency-bound at 2 CTAs/SM (shared memory allows 4):
// staged ones run 4 (64 registers, +9 % at r = 16, +11 % at r = 10), fused ones
// 3 (80 registers; at 64 the DFT-8 fill spills)
#ifndef PDB_GJ_MINB16
#define PDB_GJ_MINB16 4
#endif
#ifndef PDB_GJ_MINB16F
#define PDB_GJ_MINB16F 3
#endif
template <class Src, bool DFT8, int LPM, bool P31, int RPC, bool PAIR = false>
__global__ void __launch_bounds__(256, RPC == 16 ? (DFT8 ? PDB_GJ_MINB16F : PDB_GJ_MINB16) : PDB_GJ_MINB)
det_gj_kernel(Src src, const int32_t* __restrict__ ids_g, int64_t node_lo, int64_t nodes,
              uint32_t* __restrict__ num_out, uint32_t* __restrict__ den_out,
              unsigned long long* __restrict__ flag_count, int64_t* __restrict__ flag_nodes, GjGeom g, Mod32 m) {
  static_assert(LPM == 8 || LPM == 16 || LPM == 32, "8, 16 or 32 lanes per matrix");
  static_assert(RPC % GJ_B == 0, "compile-time order must be padded to the block size");
  static_assert(!PAIR || (RPC >= 32 && !P31), "paired blocks: compile-time order >= 32, p < 2^30");
  // Pivot-block schedule: blocks of 8, except that the staged compile-time
  // kernels (orders 40 and 16, p < 2^30, 16 lanes) eliminate their last 8
  // columns as two blocks of 4 (a 4x4 Gauss-Jordan costs a third of an 8x8 one
  // per column; the last block has no trailing update to pay for it).
  // Measured (profiles/README_r01.md): staged r = 40 +2 %, r = 16 +3.5 %; the
  // fused kernel is fastest with blocks of 8 throughout, so it keeps them.
#ifndef PDB_GJ_TAIL4
#define PDB_GJ_TAIL4 8
#endif
#ifndef PDB_GJ_TAIL4_16
#define PDB_GJ_TAIL4_16 8
#endif
  constexpr int TAIL4 = (!P31 && LPM == 16 && !DFT8) ? (RPC == 40 ? PDB_GJ_TAIL4 : (RPC == 16 ? PDB_GJ_TAIL4_16 : 0)) : 0;
  extern __shared__ __align__(16) uint32_t smem[];
  const int r = g.r;
  const int RP = RPC ? RPC : g.RP;
  const int S = RPC ? gj_row_stride(RPC) : g.S;
  const int32_t* ids = ids_g;     // read through L1 by the fills
  uint32_t* mats = smem;
  const int MS = RPC ? gj_matrix_stride(RPC, gj_row_stride(RPC)) : g.MS;
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPM, l = lane % LPM;
  const unsigned omask = (LPM == 32 ? 0xffffffffu : ((1u << LPM) - 1u)) << (grp * LPM);
  const int slot = (threadIdx.x >> 5) * (32 / LPM) + grp;
  uint32_t* A = mats + (size_t)slot * MS;
  uint32_t* NX = A + RP * S;          // negX [8][8]
  const uint32_t p = m.p, one = m.r1;

  const int64_t rows8 = DFT8 && src_ulast(src) > 0 ? nodes / (8 * (int64_t)src_ulast(src)) : 0;   // compact rows
  const int64_t iters = DFT8 ? (nodes / 8 + g.U - 1) / g.U : (nodes + g.M - 1) / g.M;
  bool dense;   // identity entry ids and no padding: affine fills
  {
    bool id = g.RP == r && g.S == r;
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) id = id && __ldg(ids + e) == e;
    dense = __syncthreads_and(id) != 0;
  }

  for (int64_t it = blockIdx.x; it < iters; it += gridDim.x) {
    __syncthreads();
    GjD8 d8{};
    if constexpr (DFT8) {
      d8 = gj_d8(src, g.U, it, threadIdx.x % g.U, rows8);
      if (PDB_GJ_ABL != 3 || it == blockIdx.x) {
        if constexpr (RPC > 0)   // launched with 256 threads, M = 256 / LPM matrices, RP = RPC
          gj_fill_dft8<256 / LPM / 8, gj_matrix_stride(RPC, gj_row_stride(RPC)), RPC * RPC>(src, mats, g, ids, d8,
                                                                                           one, dense);
        else
          gj_fill_dft8(src, mats, g, ids, d8, one, dense);
      }
    }
    else gj_fill(src, mats, g, ids, it, node_lo, nodes, one, dense);
    __syncthreads();
    int64_t node;
    if constexpr (DFT8) node = gj_node_dft8(src, it, slot, g.U, rows8);
    else node = gj_node_linear(it, slot, g, nodes);
    if (node < 0) continue;

    // C8 / C4: products of the running c-prefix Q taken before each block of 8 / 4
    // (det A picks up Q^B per block: den *= C8^8 C4^4 at the end)
    uint32_t num = one, den = one, Q = one, C8 = one, C4 = one;
    uint32_t cPrev = one;   // c of the first block of a pair
    uint32_t aprod = one;   // 4x4-block pivot blocks: product of the a = det(A)'s (den *= aprod^3)

    // One block of B pivots at column K; false if a pivot vanished.
    auto block = [&](auto Bc, int K) -> bool {
      constexpr int B = decltype(Bc)::value;
      constexpr int LPR = LPM / B;   // lanes per pivot-block row
      constexpr int EPL = B / LPR;   // pivot-block elements per lane
      static_assert(EPL >= 1, "block narrower than the lane group");
      const int pj = l / LPR, pc = EPL * (l % LPR);   // my pivot-block row / first column
      const int mrem = RP - K - B;
      // compile-time orders with 16 lanes: the idle-lane-free variants where mrem = 24
      constexpr bool FIT = RPC > 0 && LPM == 16 && B == GJ_B;
      // ---------------- P: the pivot block -> X = c A11^-1 (negated into NX), c ----------------
      // 4x4 blocks + adjugates where the order is a compile-time constant (the last
      // block only needs det(A11)); 8-step division-free Gauss-Jordan otherwise
      uint32_t cR;
      if (PDB_GJ_P44 && FIT && !P31 && mrem > 0) {
        if (!gj_pinv44(A, NX, S, K, l, omask, m, num, aprod, cR)) return false;
      } else if (PDB_GJ_P44 && FIT && !P31) {
        return gj_pdet44(A, NX, S, K, l, omask, m, num, aprod);
      } else {
        uint32_t v[EPL];
        {
          const uint32_t* src_row = A + (K + pj) * S + K + pc;
#pragma unroll
          for (int k = 0; k < EPL; ++k) v[k] = src_row[k];
        }
        constexpr bool LAZY = PDB_GJ_LAZYP && !P31 && EPL >= 4;
        const GjPiv gp = gj_gauss_jordan<B, LPM, LAZY>(v, pj, pc, l, omask, PDB_GJ_GELAST && mrem == 0, m);
        if (gp.lam == 0) return false;   // lam = prod z_s: zero iff a pivot vanished
        // det(A11) = z_{B-1} / (lambda_1 ... lambda_{B-2}): row pj holds lambda_pj = zl;
        // each row's first lane keeps its factors, the group multiplies them once per node
        den = gj_mont(den, (pj >= 1 && pj <= B - 2 && l % LPR == 0) ? gp.zl : one, m);
        num = gj_mont(num, gp.zlast, m);
        if (mrem == 0) return true;
        cR = gp.lam;   // c = prod z_s
        // negX = -X  ->  NX[pj][pc + k]
#pragma unroll
        for (int k = 0; k < EPL; ++k) {
          const uint32_t x = LAZY ? csub(v[k], p) : v[k];
          NX[gj_nx_row(pj) + pc + k] = x ? p - x : 0u;
        }
      }
      Q = gj_mont(Q, cR, m);
      if (K + B < RP - TAIL4) C8 = gj_mont(C8, Q, m);   // the next block has 8 pivots
      else C4 = gj_mont(C4, Q, m);
      __syncwarp(omask);
      // ---------------- M: negM = negX * A12, in place in the pivot rows ----------------
      if (PDB_GJ_ABL != 1) {
        if (FIT && mrem == 24) gj_mpass24<P31, B>(A, NX, S, K, l, omask, m);
        else gj_mpass_any<LPM, P31, B>(A, NX, S, K, mrem, l, omask, m);
      }
      __syncwarp(omask);
      // ---------------- T: trailing rows ----------------
      if (PAIR && K == 0) {
        // first block of the pair: only the panel the second block reads
        cPrev = cR;
        if (FIT && mrem == 32) gj_tpass_panel32(A, S, K, cR, l, m);
        else gj_tpass_panel<2, 4, LPM>(A, S, K, mrem, cR, l, m);
      } else if (PAIR && K == GJ_B) {
        // second block: c1 * negM0 beside negM1, then one 16-deep update with scale c0 c1:
        // c1 (c0 A33 + A31 negM0) + A32' negM1 (A32' = the panel strip of block 0)
        gj_scale_rows<LPM>(A, S, 0, K + B, mrem, cR, l, m);
        __syncwarp(omask);
        if (FIT && mrem == 24) gj_tpass24<false, 2 * GJ_B, true>(A, S, 0, K + B, gj_mont(cPrev, cR, m), l, m);
        else gj_tpass<2, 4, LPM, false, 2 * GJ_B, true>(A, S, 0, mrem, gj_mont(cPrev, cR, m), l, m);
      } else if (PDB_GJ_ABL != 2) {
        if (FIT && mrem == 24) gj_tpass24<P31, B>(A, S, K, K + B, cR, l, m);
        else gj_tpass_any<LPM, P31, B>(A, S, K, mrem, cR, l, m);
      }
      __syncwarp(omask);
      return true;
    };

    bool ok = true;
    if constexpr (TAIL4 > 0) {
      // e.g. RPC = 40: 8 8 8 8 | 4 4 (TAIL4 = 8) -- every K and block size a constant
      constexpr int K8 = RPC - TAIL4;
      static_assert(K8 % GJ_B == 0 && TAIL4 % 4 == 0, "tail split");
      gj_unrolled<0, K8, 8>([&](auto Kc) { if (ok && !block(std::integral_constant<int, 8>{}, Kc())) ok = false; });
      gj_unrolled<K8, RPC, 4>([&](auto Kc) { if (ok && !block(std::integral_constant<int, 4>{}, Kc())) ok = false; });
    } else if constexpr (RPC > 0) {
      gj_unrolled<0, RPC, GJ_B>([&](auto Kc) { if (ok && !block(std::integral_constant<int, GJ_B>{}, Kc())) ok = false; });
    } else {
#pragma unroll
      for (int K = 0; K < RP; K += GJ_B)
        if (!block(std::integral_constant<int, GJ_B>{}, K)) { ok = false; break; }
    }
#pragma unroll
    // every block by 4x4 blocks (compile-time order, 8-pivot blocks only): den and C4
    // are never touched, det = num / (C8^8 aprod^3)
    constexpr bool ALL44 = PDB_GJ_P44 && RPC > 0 && LPM == 16 && !P31 && TAIL4 == 0;
    if constexpr (!ALL44) {
#pragma unroll
      for (int d = 1; d < LPM; d <<= 1) den = gj_mont(den, __shfl_xor_sync(omask, den, d, LPM), m);
    }
    if (l == 0) {
      if (ok) {
        uint32_t c = C8;   // C8^8 * C4^4
#pragma unroll
        for (int i = 0; i < 3; ++i) c = gj_mont(c, c, m);
        if constexpr (TAIL4 > 0) {
          uint32_t c4 = C4;
#pragma unroll
          for (int i = 0; i < 2; ++i) c4 = gj_mont(c4, c4, m);
          c = gj_mont(c, c4, m);
        }
        num_out[node] = num;
        if (PDB_GJ_P44) c = gj_mont(c, gj_mont(gj_mont(aprod, aprod, m), aprod, m), m);   // aprod^3
        den_out[node] = ALL44 ? c : gj_mont(den, c, m);
      } else {
        den_out[node] = 0u;
        unsigned long long k = atomicAdd(flag_count, 1ull);
        flag_nodes[k] = node_lo + node;
      }
    }
    __syncwarp(omask);
  }
}

// det = num / den * R^r per node (Montgomery forms).  Each lane owns D nodes
// (lane-strided, coalesced); prefix products in the lane, then across the warp
// by shuffles: one Fermat inversion per 32 D nodes (the exponentiation, not the
// 12 bytes of traffic per node, bounded the one-node-per-lane version).
constexpr int GJ_FIN_D = 8;
__global__ void __launch_bounds__(256)
det_gj_finalize(uint32_t* __restrict__ out, const uint32_t* __restrict__ den, int64_t nodes, uint32_t Rr, Mod32 m) {
  constexpr int D = GJ_FIN_D;
  const int lane = threadIdx.x & 31;
  const uint32_t one = m.r1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * D;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) * D; base < nodes; base += stride) {
    uint32_t dv[D], pre[D];
    uint32_t run = one;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t idx = base + d * 32 + lane;
      dv[d] = idx < nodes ? den[idx] : 0u;
      run = gj_mont(run, dv[d] ? dv[d] : one, m);   // flagged (0) and tail nodes count as 1
      pre[d] = run;                                  // product of this lane's dens up to d
    }
    uint32_t pre_x = run, suf_x = run;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const uint32_t up = __shfl_up_sync(0xffffffffu, pre_x, k);
      const uint32_t dn = __shfl_down_sync(0xffffffffu, suf_x, k);
      if (lane >= k) pre_x = gj_mont(pre_x, up, m);
      if (lane + k < 32) suf_x = gj_mont(suf_x, dn, m);
    }
    const uint32_t total = __shfl_sync(0xffffffffu, pre_x, 31);
    const uint32_t inv_total = mont_pow(total, (uint64_t)m.p - 2, m);
    uint32_t left = __shfl_up_sync(0xffffffffu, pre_x, 1);
    uint32_t right = __shfl_down_sync(0xffffffffu, suf_x, 1);
    if (lane == 0) left = one;
    if (lane == 31) right = one;
    uint32_t inv = gj_mont(gj_mont(left, right, m), inv_total, m);   // 1 / (this lane's product)
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      const int64_t idx = base + d * 32 + lane;
      const uint32_t inv_d = d ? gj_mont(inv, pre[d - 1], m) : inv;   // 1 / dv[d]
      inv = gj_mont(inv, dv[d] ? dv[d] : one, m);
      if (idx < nodes && dv[d]) out[idx] = gj_mont(gj_mont(out[idx], inv_d, m), Rr, m);
    }
  }
}

inline GjGeom gj_geom(int r, int warps, int lpm, bool dft8) {
  GjGeom g;
  g.r = r;
  g.RP = (r + 7) & ~7;
  g.S = gj_row_stride(g.RP);
  // matrix stride = 16 (mod 32) words: the two matrices of a warp (and the U
  // matrices a fill thread group writes) start in opposite bank halves
  g.MS = gj_matrix_stride(g.RP, g.S);
  g.M = warps * (32 / lpm);
  g.U = dft8 ? g.M / 8 : 0;
  return g;
}

inline size_t gj_smem(const GjGeom& g) {
  return sizeof(uint32_t) * (size_t)g.M * g.MS;
}

// warps per CTA: DFT-8 needs M % 8 == 0; otherwise as many resident matrices as fit
inline GjGeom gj_pick(int r, int lpm, bool dft8) {
  const size_t budget = 227 * 1024;
  GjGeom best = gj_geom(r, 8, lpm, dft8);
  double best_score = -1;
  static const char* wenv = getenv("PDB_GJ_WARPS");   // experiments: force warps per CTA
  const int wforce = wenv && *wenv ? atoi(wenv) : 0;
  for (int warps = 1; warps <= 8; ++warps) {
    if (wforce && warps != wforce) continue;
    GjGeom g = gj_geom(r, warps, lpm, dft8);
    if (dft8 && (g.M % 8)) continue;
    const size_t sm = gj_smem(g) + 1024;
    int ctas = (int)(budget / sm);
    if (ctas > 32) ctas = 32;
    if (ctas < 1) continue;
    const int resident = ctas * warps > 64 ? 64 : ctas * warps;
    const double score = resident * (32 / lpm) + 0.01 * warps;   // resident matrices, then bigger CTAs
    if (score > best_score) { best_score = score; best = g; }
  }
  return best;
}

}  // namespace pdb
