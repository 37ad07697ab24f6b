// det_gj: blocked Schur-complement elimination, one lane group per matrix.
//
// The value of det(M) mod p is algorithm independent (reference
// determinant.py:1-8), so this kernel chooses the schedule that suits the
// integer pipes of sm_100a (profiles/README_r01.md):
//
//   for every block of 8 pivots K..K+7 (the order r is padded to RP = 8*ceil(r/8)
//   with an identity block, which leaves the determinant unchanged):
//     P  division-free Gauss-Jordan on the 8x8 pivot block A11, in registers
//        (LPM/8 lanes per row, pivot rows exchanged by shuffles):
//        X * A11 = c * I  with  X = diag(Z_{<j}) * E,  c = prod z_s,
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
// canonical with two conditional subtractions (ALU pipe, no IMAD.HI).
//
// A zero pivot (prob. ~r/p per node) diverts the node to det_robust, which
// applies the reference's first-nonzero pivoting (determinant.py:136-169).
#pragma once
#include "pdb_internal.cuh"

namespace pdb {

constexpr int GJ_B = 8;

#ifndef PDB_GJ_MINB
#define PDB_GJ_MINB 3   // resident CTAs per SM the register budget is sized for
#endif

struct GjGeom {
  int r;    // matrix order
  int RP;   // padded order, multiple of 8
  int S;    // row stride (words): multiple of 4 with S/4 odd, >= RP
  int MS;   // matrix stride (words): RP*S + negX (64)
  int M;    // matrices per CTA iteration
  int U;    // fused DFT-8 fill: distinct u per iteration (M = 8U); 0 = off
};

__host__ __device__ inline int gj_row_stride(int RP) {
  int S = RP + 4;
  while (((S >> 2) & 1) == 0) S += 4;
  return S;
}

// REDC of a <= 9-product accumulator, canonical: two conditional subtractions.
__device__ __forceinline__ uint32_t gj_red(uint64_t acc, const Mod32& m) {
  const uint32_t v = redc(acc, m);
  return csub(csub(v, 2u * m.p), m.p);
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

__device__ __forceinline__ int64_t gj_node_dft8(int64_t it, int slot, const GjGeom& g, int NL) {
  const int per_o = NL / (8 * g.U);
  const int64_t o = it / per_o;
  const int ublk = (int)(it - o * per_o);
  const int v = slot / g.U, uu = slot - v * g.U;
  return o * NL + ublk * g.U + uu + (int64_t)(NL / 8) * v;
}

// ---- fills: the RP x RP matrices of one iteration (padding = Montgomery identity) ----
__device__ __forceinline__ void gj_fill(const StagedSrc& src, uint32_t* mats, const GjGeom& g, const int32_t* ids,
                                        int64_t it, int64_t node_lo, int64_t nodes, uint32_t one) {
  const int r = g.r, RP = g.RP, S = g.S, M = g.M;
  const int slot = threadIdx.x % M;
  const int64_t n = gj_node_linear(it, slot, g, nodes);
  if (n >= 0) {
    const uint32_t* col = src.grids + node_lo + n;
    uint32_t* dst = mats + (size_t)slot * g.MS;
    GjPos pi(threadIdx.x / M, blockDim.x / M, RP);
    for (; pi.i < RP; pi.next()) {
      if (pi.i < r && pi.j < r) gj_cp_async4(dst + pi.i * S + pi.j, col + (int64_t)ids[pi.i * r + pi.j] * src.stride);
      else dst[pi.i * S + pi.j] = pi.i == pi.j ? one : 0u;
    }
  }
  gj_cp_async_wait_all();
}

__device__ __forceinline__ void gj_fill(const FusedSrc& src, uint32_t* mats, const GjGeom& g, const int32_t* ids,
                                        int64_t it, int64_t node_lo, int64_t nodes, uint32_t one) {
  const int r = g.r, RP = g.RP, S = g.S, M = g.M;
  const int slot = threadIdx.x % M;
  const int64_t n = gj_node_linear(it, slot, g, nodes);
  if (n < 0) return;
  uint32_t* dst = mats + (size_t)slot * g.MS;
  GjPos pi(threadIdx.x / M, blockDim.x / M, RP);
  for (; pi.i < RP; pi.next())
    dst[pi.i * S + pi.j] = (pi.i < r && pi.j < r) ? src.get(ids[pi.i * r + pi.j], node_lo + n)
                                                  : (pi.i == pi.j ? one : 0u);
}

// 8 nodes per thread: f(o*NL + u + (NL/8) v) = sum_l (T_l w^(u l)) w8^(l v), an
// 8-point DIT transform of the twisted coefficients (E <= 8).
__device__ __forceinline__ void gj_fill_dft8(const FusedSrc& src, uint32_t* mats, const GjGeom& g, const int32_t* ids,
                                             int64_t it, int64_t node_lo, uint32_t one) {
  const int r = g.r, RP = g.RP, S = g.S, U = g.U, NL = src.NL, E = src.E;
  const uint32_t p = src.p;
  const int per_o = NL / (8 * U);
  const int64_t o = (node_lo / NL) + it / per_o;
  const int ublk = (int)(it % per_o);
  const int step8 = NL / 8;
  const uint32_t w1 = __ldg(src.xs + step8), w1s = __ldg(src.xss + step8);
  const uint32_t w2 = __ldg(src.xs + 2 * step8), w2s = __ldg(src.xss + 2 * step8);
  const uint32_t w3 = __ldg(src.xs + 3 * step8), w3s = __ldg(src.xss + 3 * step8);
  const int uu = threadIdx.x % U;
  uint32_t tw[8], tws[8];
  {
    const int u = ublk * U + uu;
    int k = 0;
#pragma unroll
    for (int ll = 0; ll < 8; ++ll) {
      tw[ll] = __ldg(src.xs + k);
      tws[ll] = __ldg(src.xss + k);
      k += u;
      if (k >= NL) k -= NL;
    }
  }
  const size_t ms = (size_t)U * g.MS;   // slot v*U + uu
  uint32_t* base = mats + (size_t)uu * g.MS;
  GjPos pi(threadIdx.x / U, blockDim.x / U, RP);
  for (; pi.i < RP; pi.next()) {
    const int i = pi.i, j = pi.j;
    uint32_t* d = base + i * S + j;
    if (i >= r || j >= r) {
      const uint32_t c = i == j ? one : 0u;
#pragma unroll
      for (int v = 0; v < 8; ++v) d[v * ms] = c;
      continue;
    }
    const uint32_t* a = src.part + ((int64_t)ids[i * r + j] * src.outer + o) * E;
    uint32_t q[8];
    q[0] = __ldg(a);
#pragma unroll
    for (int ll = 1; ll < 8; ++ll) q[ll] = ll < E ? shoup_mul(__ldg(a + ll), tw[ll], tws[ll], p) : 0u;
    uint32_t x0 = q[0], x1 = q[4], x2 = q[2], x3 = q[6], x4 = q[1], x5 = q[5], x6 = q[3], x7 = q[7];
    uint32_t t;
    t = x1; x1 = sub_mod(x0, t, p); x0 = add_mod(x0, t, p);
    t = x3; x3 = sub_mod(x2, t, p); x2 = add_mod(x2, t, p);
    t = x5; x5 = sub_mod(x4, t, p); x4 = add_mod(x4, t, p);
    t = x7; x7 = sub_mod(x6, t, p); x6 = add_mod(x6, t, p);
    t = x2; x2 = sub_mod(x0, t, p); x0 = add_mod(x0, t, p);
    t = shoup_mul(x3, w2, w2s, p); x3 = sub_mod(x1, t, p); x1 = add_mod(x1, t, p);
    t = x6; x6 = sub_mod(x4, t, p); x4 = add_mod(x4, t, p);
    t = shoup_mul(x7, w2, w2s, p); x7 = sub_mod(x5, t, p); x5 = add_mod(x5, t, p);
    t = x4; x4 = sub_mod(x0, t, p); x0 = add_mod(x0, t, p);
    t = shoup_mul(x5, w1, w1s, p); x5 = sub_mod(x1, t, p); x1 = add_mod(x1, t, p);
    t = shoup_mul(x6, w2, w2s, p); x6 = sub_mod(x2, t, p); x2 = add_mod(x2, t, p);
    t = shoup_mul(x7, w3, w3s, p); x7 = sub_mod(x3, t, p); x3 = add_mod(x3, t, p);
    d[0] = x0; d[ms] = x1; d[2 * ms] = x2; d[3 * ms] = x3;
    d[4 * ms] = x4; d[5 * ms] = x5; d[6 * ms] = x6; d[7 * ms] = x7;
  }
}

// ---- T pass: A22 <- c*A22 + A21*negM over TR x TC tiles ------------------------------
template <int TR, int TC, int LPM>
__device__ __forceinline__ void gj_tpass(uint32_t* A, int S, int K, int mrem, uint32_t cR, int l, const Mod32& m) {
  const int c0 = K + GJ_B;
  const int ntc = mrem / TC;
  const int tiles = (mrem / TR) * ntc;
  const uint32_t* npr = A + K * S;    // negM rows K..K+7
  for (int w = l; w < tiles; w += LPM) {
    const int ti = w / ntc, tc = w - ti * ntc;
    const int i0 = c0 + TR * ti, cc = c0 + TC * tc;
    uint32_t a21[TR][GJ_B];
    uint64_t acc[TR][TC];
#pragma unroll
    for (int a = 0; a < TR; ++a) {
      const uint32_t* row = A + (i0 + a) * S;
      const uint4 x = *reinterpret_cast<const uint4*>(row + K);
      const uint4 y = *reinterpret_cast<const uint4*>(row + K + 4);
      a21[a][0] = x.x; a21[a][1] = x.y; a21[a][2] = x.z; a21[a][3] = x.w;
      a21[a][4] = y.x; a21[a][5] = y.y; a21[a][6] = y.z; a21[a][7] = y.w;
#pragma unroll
      for (int b = 0; b < TC; b += 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(row + cc + b);
        acc[a][b] = mad_wide(v.x, cR, 0ull);
        acc[a][b + 1] = mad_wide(v.y, cR, 0ull);
      }
    }
#pragma unroll
    for (int q = 0; q < GJ_B; ++q) {
      uint32_t nm[TC];
#pragma unroll
      for (int b = 0; b < TC; b += 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(npr + q * S + cc + b);
        nm[b] = v.x; nm[b + 1] = v.y;
      }
#pragma unroll
      for (int a = 0; a < TR; ++a)
#pragma unroll
        for (int b = 0; b < TC; ++b) acc[a][b] = mad_wide(a21[a][q], nm[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < TR; ++a) {
      uint32_t* row = A + (i0 + a) * S;
#pragma unroll
      for (int b = 0; b < TC; b += 2) {
        uint2 v;
        v.x = gj_red(acc[a][b], m);
        v.y = gj_red(acc[a][b + 1], m);
        *reinterpret_cast<uint2*>(row + cc + b) = v;
      }
    }
  }
}

template <int LPM>
__device__ __forceinline__ void gj_tpass_any(uint32_t* A, int S, int K, int mrem, uint32_t cR, int l, const Mod32& m) {
  // largest tile that keeps >= ~70 % of the lanes busy
  auto util = [&](int tr, int tc) {
    const int t = (mrem / tr) * (mrem / tc);
    const int passes = (t + LPM - 1) / LPM;
    return (float)t / (float)(passes * LPM);
  };
  if (util(2, 8) >= 0.7f) gj_tpass<2, 8, LPM>(A, S, K, mrem, cR, l, m);
  else if (util(2, 4) >= 0.7f) gj_tpass<2, 4, LPM>(A, S, K, mrem, cR, l, m);
  else if (util(1, 4) >= 0.7f) gj_tpass<1, 4, LPM>(A, S, K, mrem, cR, l, m);
  else gj_tpass<1, 2, LPM>(A, S, K, mrem, cR, l, m);
}

// ---- the kernel ------------------------------------------------------------------------------
template <class Src, bool DFT8, int LPM>
__global__ void __launch_bounds__(256, PDB_GJ_MINB)
det_gj_kernel(Src src, const int32_t* __restrict__ ids_g, int64_t node_lo, int64_t nodes,
              uint32_t* __restrict__ num_out, uint32_t* __restrict__ den_out,
              unsigned long long* __restrict__ flag_count, int64_t* __restrict__ flag_nodes, GjGeom g, Mod32 m) {
  static_assert(LPM == 8 || LPM == 16 || LPM == 32, "8, 16 or 32 lanes per matrix");
  constexpr int LPR = LPM / 8;   // lanes per pivot-block row
  constexpr int EPL = 8 / LPR;   // pivot-block elements per lane
  extern __shared__ __align__(16) uint32_t smem[];
  const int r = g.r, RP = g.RP, S = g.S;
  int32_t* ids = reinterpret_cast<int32_t*>(smem);
  uint32_t* mats = smem + ((r * r + 3) & ~3);
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPM, l = lane % LPM;
  const unsigned omask = (LPM == 32 ? 0xffffffffu : ((1u << LPM) - 1u)) << (grp * LPM);
  const int slot = (threadIdx.x >> 5) * (32 / LPM) + grp;
  uint32_t* A = mats + (size_t)slot * g.MS;
  uint32_t* NX = A + RP * S;          // negX [8][8]
  const uint32_t p = m.p, one = m.r1;
  const int pj = l / LPR, pc = EPL * (l % LPR);   // my pivot-block row / first column

  for (int e = threadIdx.x; e < r * r; e += blockDim.x) ids[e] = ids_g[e];
  const int64_t iters = DFT8 ? (nodes / g.M) : (nodes + g.M - 1) / g.M;

  for (int64_t it = blockIdx.x; it < iters; it += gridDim.x) {
    __syncthreads();
    if constexpr (DFT8) gj_fill_dft8(src, mats, g, ids, it, node_lo, one);
    else gj_fill(src, mats, g, ids, it, node_lo, nodes, one);
    __syncthreads();
    int64_t node;
    if constexpr (DFT8) node = gj_node_dft8(it, slot, g, src.NL);
    else node = gj_node_linear(it, slot, g, nodes);
    if (node < 0) continue;

    uint32_t num = one, den = one, Q = one, C = one;
    bool ok = true;
    for (int K = 0; K < RP; K += GJ_B) {
      const int mrem = RP - K - GJ_B;
      // ---------------- P: Gauss-Jordan on the pivot block ----------------
      uint32_t v[EPL];
      {
        const uint32_t* src_row = A + (K + pj) * S + K + pc;
#pragma unroll
        for (int k = 0; k < EPL; ++k) v[k] = src_row[k];
      }
      uint32_t lam = one, zl = one, z7 = one;
#pragma unroll
      for (int s = 0; s < GJ_B; ++s) {
        const uint32_t z = __shfl_sync(omask, v[s % EPL], s * LPR + s / EPL, LPM);
        const uint32_t t = __shfl_sync(omask, v[s % EPL], pj * LPR + s / EPL, LPM);
        uint32_t prow[EPL];
#pragma unroll
        for (int k = 0; k < EPL; ++k) prow[k] = __shfl_sync(omask, v[k], s * LPR + l % LPR, LPM);
        if (z == 0) { ok = false; break; }
        if (pj == s) zl = lam;
        const uint32_t nt = t ? p - t : 0u;
#pragma unroll
        for (int k = 0; k < EPL; ++k) {
          const int cc = pc + k;
          if (pj != s) {
            const uint32_t a = cc == s ? 0u : v[k];
            const uint32_t b = cc == s ? lam : prow[k];
            v[k] = gj_red(mad_wide(z, a, mad_wide(nt, b, 0ull)), m);
          } else if (cc == s) {
            v[k] = lam;
          }
        }
        if (s >= 1 && s <= 6) den = mont(den, lam, m);
        if (s == GJ_B - 1) z7 = z;
        lam = mont(lam, z, m);
      }
      if (!ok) break;
      num = mont(num, z7, m);
      if (mrem == 0) break;
      const uint32_t cR = lam;   // c = prod z_s
      Q = mont(Q, cR, m);
      C = mont(C, Q, m);
      // negX = -Z_{<j} E  ->  NX[pj][pc + k]
#pragma unroll
      for (int k = 0; k < EPL; ++k) {
        const uint32_t x = mont(v[k], zl, m);
        NX[pj * GJ_B + pc + k] = x ? p - x : 0u;
      }
      __syncwarp(omask);
      // ---------------- M: negM = negX * A12, in place in the pivot rows ----------------
      {
        int G = 1;
        while (G < GJ_B && mrem * G * 2 <= LPM) G *= 2;
        const int rpi = GJ_B / G;
        const int items = mrem * G;
        for (int w0 = 0; w0 < items; w0 += LPM) {
          const int w = w0 + l;
          uint32_t res[GJ_B];
          int c = 0, jg = 0;
          if (w < items) {
            jg = w / mrem;
            c = K + GJ_B + (w - jg * mrem);
            uint32_t a[GJ_B];
#pragma unroll
            for (int q = 0; q < GJ_B; ++q) a[q] = A[(K + q) * S + c];
#pragma unroll
            for (int t = 0; t < GJ_B; ++t) {
              if (t < rpi) {
                const uint32_t* xr = NX + (jg * rpi + t) * GJ_B;
                const uint4 x0 = *reinterpret_cast<const uint4*>(xr);
                const uint4 x1 = *reinterpret_cast<const uint4*>(xr + 4);
                uint64_t acc = mad_wide(x0.x, a[0], 0ull);
                acc = mad_wide(x0.y, a[1], acc);
                acc = mad_wide(x0.z, a[2], acc);
                acc = mad_wide(x0.w, a[3], acc);
                acc = mad_wide(x1.x, a[4], acc);
                acc = mad_wide(x1.y, a[5], acc);
                acc = mad_wide(x1.z, a[6], acc);
                acc = mad_wide(x1.w, a[7], acc);
                res[t] = gj_red(acc, m);
              }
            }
          }
          __syncwarp(omask);
          if (w < items) {
#pragma unroll
            for (int t = 0; t < GJ_B; ++t)
              if (t < rpi) A[(K + jg * rpi + t) * S + c] = res[t];
          }
        }
      }
      __syncwarp(omask);
      // ---------------- T: trailing rows ----------------
      gj_tpass_any<LPM>(A, S, K, mrem, cR, l, m);
      __syncwarp(omask);
    }
    if (l == 0) {
      if (ok) {
        // C^8
        C = mont(C, C, m);
        C = mont(C, C, m);
        C = mont(C, C, m);
        num_out[node] = num;
        den_out[node] = mont(den, C, m);
      } else {
        den_out[node] = 0u;
        unsigned long long k = atomicAdd(flag_count, 1ull);
        flag_nodes[k] = node_lo + node;
      }
    }
    __syncwarp(omask);
  }
}

// det = num / den * R^r per node (Montgomery forms), 32 inversions per Fermat.
__global__ void __launch_bounds__(256)
det_gj_finalize(uint32_t* __restrict__ out, const uint32_t* __restrict__ den, int64_t nodes, uint32_t Rr, Mod32 m) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < nodes; base += stride) {
    const int64_t idx = base + lane;
    const bool valid = idx < nodes;
    const uint32_t d = valid ? den[idx] : 0u;
    const bool use = d != 0u;
    const uint32_t x = use ? d : m.r1;
    uint32_t pre_x = x, suf_x = x;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const uint32_t up = __shfl_up_sync(0xffffffffu, pre_x, k);
      const uint32_t dn = __shfl_down_sync(0xffffffffu, suf_x, k);
      if (lane >= k) pre_x = mont(pre_x, up, m);
      if (lane + k < 32) suf_x = mont(suf_x, dn, m);
    }
    const uint32_t totalR = __shfl_sync(0xffffffffu, pre_x, 31);
    const uint32_t inv_totalR = mont_pow(totalR, (uint64_t)m.p - 2, m);
    uint32_t left = __shfl_up_sync(0xffffffffu, pre_x, 1);
    uint32_t right = __shfl_down_sync(0xffffffffu, suf_x, 1);
    if (lane == 0) left = m.r1;
    if (lane == 31) right = m.r1;
    const uint32_t invR = mont(mont(left, right, m), inv_totalR, m);
    if (use) out[idx] = mont(mont(out[idx], invR, m), Rr, m);
  }
}

inline GjGeom gj_geom(int r, int warps, int lpm, bool dft8) {
  GjGeom g;
  g.r = r;
  g.RP = (r + 7) & ~7;
  g.S = gj_row_stride(g.RP);
  g.MS = g.RP * g.S + GJ_B * GJ_B;
  g.M = warps * (32 / lpm);
  g.U = dft8 ? g.M / 8 : 0;
  return g;
}

inline size_t gj_smem(const GjGeom& g) {
  return sizeof(uint32_t) * ((size_t)((g.r * g.r + 3) & ~3) + (size_t)g.M * g.MS);
}

// lanes per matrix: a full warp once the trailing blocks are large enough
inline int gj_lpm(int r) {
  static const char* env = getenv("PDB_GJ_LPM");
  if (env) {
    const int v = atoi(env);
    return v == 8 || v == 16 ? v : 32;
  }
  return r > 24 ? 32 : (r > 16 ? 16 : 8);
}

// warps per CTA: DFT-8 needs M % 8 == 0; otherwise as many resident matrices as fit
inline GjGeom gj_pick(int r, int lpm, bool dft8) {
  const size_t budget = 227 * 1024;
  GjGeom best = gj_geom(r, 8, lpm, dft8);
  double best_score = -1;
  for (int warps = 1; warps <= 8; ++warps) {
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
