// det_octet: blocked division-free elimination, 8 lanes per matrix.
//
// Why this shape (measured in profiles/intpipe_r01.json):
//   * IMAD.WIDE (64-bit multiply-accumulate) issues at half rate like
//     IMAD.HI, so a Shoup mul-mod costs 4 fma-heavy slots while a delayed
//     64-bit MAC costs 2.  Accumulating the B+1 products of a rank-B block
//     update in 64 bits and reducing once (Montgomery REDC + Barrett) cuts the
//     slot count per elimination update to ~2.7.
//   * Normalised multipliers need one modular inverse per pivot; with only
//     ~24-32 resident 40x40 matrices per SM those per-step inverses would cost
//     as much as the updates.  The division-free (condensation) form of the
//     reference (determinant.py:136-169) needs one inverse per matrix; its
//     per-row scalings are folded into scalars (tau, ZP, V below).
//
// One block of pivots K..K+B-1 (z_s = pivot s, prow_s = pivot row s):
//   P phase (pivot rows, sequential in s): row K+s is final once pivots < s
//     have been applied; it is stored as NPR_s = -R*prow_s mod p (R = 2^32,
//     Montgomery form) and applied at once, division-free, to the pending
//     pivot rows: row_j <- z_s*row_j - row_j[K+s]*prow_s  == REDC(row_j*zR + t*NPR).
//   T phase (trailing rows, every lane its own rows, no synchronisation):
//     row_i after the block = ZP[B]*row_i - sum_s tau_s * prow_s with
//     ZP[S] = prod_{s<S} z_s, tau_s = t_s * prod_{s<s'<B} z_s', and the
//     multipliers t_s = (row_i after s pivots)[K+s] from the triangular
//     recurrence t_S = ZP[S]*row_i[K+S] + sum_{s<S} t_s*V[s][S],
//     V[s][S] = -prow_s[K+S]*prod_{s<s'<S} z_s'.  Each new element is
//     REDC(row*ZPR + sum tau*NPR): B+1 = 9 MACs, one reduction.
//   det = prod z_k / prod z_k^(r-1-k) (one inverse per matrix).
// A zero diagonal pivot aborts the matrix and appends its node to the
// robust kernel's list (first-nonzero pivoting, the reference's rule).
//
// Matrix loading (fill): staged grids are gathered with cp.async (no
// register round trip); fused sources evaluate the last variable in the
// kernel, 8 nodes at a time with an 8-point NTT when the CTA's matrices are
// the nodes {o*NL + u + (NL/8) v : v < 8} (fused_dft8), else by Horner.
#pragma once
#include <cstdlib>
#include "pdb_internal.cuh"

namespace pdb {

constexpr int OCT_B = 8;      // pivots per block
constexpr int OCT_LPM = 8;    // lanes per matrix

struct OctGeom {
  int r;       // matrix order
  int S;       // row stride (words), multiple of 4, >= ceil4(r)
  int MS;      // matrix stride (words) incl. scalar area
  int M;       // matrices per CTA iteration (= 4 * warps)
  int U;       // fused DFT-8 mode: distinct u per iteration (M = 8 U), 0 = off
};

__host__ __device__ inline int oct_row_stride(int r) {
  int S = (r + 3) & ~3;
  while (((S >> 2) & 1) == 0) S += 4;  // S/4 odd -> 8 rows hit 8 distinct 16B bank groups
  return S;
}

// scalar area per matrix: V (B*B), ZPR (B+1), ZETAR (B), ZR (B)
constexpr int PBW = 2 * OCT_B;   // P-panel row width
constexpr int OCT_SCALARS = OCT_B * PBW + OCT_B * OCT_B + (OCT_B + 1) + 2 * OCT_B + 3;

__device__ __forceinline__ uint32_t oct_reduce(uint64_t acc, const Mod32& m) {
  return canon32(redc(acc, m), m);
}

__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// ---- loaders ------------------------------------------------------------------
// node offset (relative to node_lo) of matrix slot m in iteration it, or -1
__device__ __forceinline__ int64_t oct_node_linear(int64_t it, int m, const OctGeom& g, int64_t nodes) {
  int64_t n = it * g.M + m;
  return n < nodes ? n : -1;
}

__device__ __forceinline__ int64_t oct_node_dft8(int64_t it, int m, const OctGeom& g, int NL) {
  const int per_o = NL / (8 * g.U);
  const int64_t o = it / per_o;
  const int ublk = (int)(it - o * per_o);
  const int v = m / g.U, uu = m - v * g.U;
  return o * NL + ublk * g.U + uu + (int64_t)(NL / 8) * v;
}

// Position iterator over the r*r real entries without per-element division:
// flat index pos = first + k*step, tracked as (i, j) with an incremental carry.
struct PosIter {
  int i, j, di, dj, r;
  __device__ __forceinline__ PosIter(int first, int step, int r_) : r(r_) {
    i = first / r_; j = first - i * r_; di = step / r_; dj = step - di * r_;
  }
  __device__ __forceinline__ void next() {
    i += di; j += dj;
    if (j >= r) { j -= r; ++i; }
  }
};

// Staged grids: thread -> (matrix slot m = t % M, positions t/M + k*(blockDim/M)),
// gathered with cp.async (consecutive threads read consecutive nodes).
__device__ __forceinline__ void oct_fill(const StagedSrc& src, uint32_t* mats, const OctGeom& g, const int32_t* ids,
                         int64_t it, int64_t node_lo, int64_t nodes) {
  const int r = g.r, S = g.S, M = g.M;
  const int m = threadIdx.x % M;
  const int64_t n = oct_node_linear(it, m, g, nodes);
  if (n >= 0) {
    const uint32_t* col = src.grids + node_lo + n;
    uint32_t* dst = mats + (size_t)m * g.MS;
    PosIter pi(threadIdx.x / M, blockDim.x / M, r);
    for (; pi.i < r; pi.next())
      cp_async4(dst + pi.i * S + pi.j, col + (int64_t)ids[pi.i * r + pi.j] * src.stride);
  }
  cp_async_wait_all();
}

// Horner evaluation, any geometry (matrix slot m <-> node it*M + m).
__device__ __forceinline__ void oct_fill(const FusedSrc& src, uint32_t* mats, const OctGeom& g, const int32_t* ids,
                         int64_t it, int64_t node_lo, int64_t nodes) {
  const int r = g.r, S = g.S, M = g.M;
  const int m = threadIdx.x % M;
  const int64_t n = oct_node_linear(it, m, g, nodes);
  if (n < 0) return;
  uint32_t* dst = mats + (size_t)m * g.MS;
  PosIter pi(threadIdx.x / M, blockDim.x / M, r);
  for (; pi.i < r; pi.next()) dst[pi.i * S + pi.j] = src.get(ids[pi.i * r + pi.j], node_lo + n);
}

// 8 nodes per thread: f(o*NL + u + (NL/8) v) = sum_l Q_l w8^(l v),  Q_l = sum_{l' = l mod 8} T_l' w^(u l').
__device__ __forceinline__ void oct_fill_dft8(const FusedSrc& src, uint32_t* mats, const OctGeom& g, const int32_t* ids,
                              int64_t it, int64_t node_lo) {
  const int r = g.r, S = g.S, U = g.U, NL = src.NL, E = src.E;
  const uint32_t p = src.p;
  const int per_o = NL / (8 * U);
  const int64_t o = (node_lo / NL) + it / per_o;
  const int ublk = (int)(it % per_o);
  const int step8 = NL / 8;
  const uint32_t w1 = __ldg(src.xs + step8), w1s = __ldg(src.xss + step8);
  const uint32_t w2 = __ldg(src.xs + 2 * step8), w2s = __ldg(src.xss + 2 * step8);
  const uint32_t w3 = __ldg(src.xs + 3 * step8), w3s = __ldg(src.xss + 3 * step8);
  const int uu = threadIdx.x % U;
  // twists w^(u l), l < 8, for this thread's u (indices stepped without any modulo)
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
  const size_t ms = (size_t)U * g.MS;
  uint32_t* slot = mats + (size_t)uu * g.MS;
  PosIter pi(threadIdx.x / U, blockDim.x / U, r);
  for (; pi.i < r; pi.next()) {
    const int i = pi.i, j = pi.j;
    uint32_t* d = slot + i * S + j;
    const uint32_t* a = src.part + ((int64_t)ids[i * r + j] * src.outer + o) * E;
    uint32_t q[8];
    q[0] = __ldg(a);
#pragma unroll
    for (int ll = 1; ll < 8; ++ll)   // E <= 8 on this path (checked at launch)
      q[ll] = ll < E ? shoup_mul(__ldg(a + ll), tw[ll], tws[ll], p) : 0u;
    // radix-2 DIT on bit-reversed input -> natural order X[v] = sum_l q_l w8^(l v)
    uint32_t x0 = q[0], x1 = q[4], x2 = q[2], x3 = q[6], x4 = q[1], x5 = q[5], x6 = q[3], x7 = q[7];
    uint32_t t;
    // stage 1 (span 1, twiddle 1)
    t = x1; x1 = sub_mod(x0, t, p); x0 = add_mod(x0, t, p);
    t = x3; x3 = sub_mod(x2, t, p); x2 = add_mod(x2, t, p);
    t = x5; x5 = sub_mod(x4, t, p); x4 = add_mod(x4, t, p);
    t = x7; x7 = sub_mod(x6, t, p); x6 = add_mod(x6, t, p);
    // stage 2 (span 2, twiddles 1, w8^2)
    t = x2; x2 = sub_mod(x0, t, p); x0 = add_mod(x0, t, p);
    t = shoup_mul(x3, w2, w2s, p); x3 = sub_mod(x1, t, p); x1 = add_mod(x1, t, p);
    t = x6; x6 = sub_mod(x4, t, p); x4 = add_mod(x4, t, p);
    t = shoup_mul(x7, w2, w2s, p); x7 = sub_mod(x5, t, p); x5 = add_mod(x5, t, p);
    // stage 3 (span 4, twiddles 1, w8, w8^2, w8^3)
    t = x4; x4 = sub_mod(x0, t, p); x0 = add_mod(x0, t, p);
    t = shoup_mul(x5, w1, w1s, p); x5 = sub_mod(x1, t, p); x1 = add_mod(x1, t, p);
    t = shoup_mul(x6, w2, w2s, p); x6 = sub_mod(x2, t, p); x2 = add_mod(x2, t, p);
    t = shoup_mul(x7, w3, w3s, p); x7 = sub_mod(x3, t, p); x3 = add_mod(x3, t, p);
    d[0] = x0; d[ms] = x1; d[2 * ms] = x2; d[3 * ms] = x3;
    d[4 * ms] = x4; d[5 * ms] = x5; d[6 * ms] = x6; d[7 * ms] = x7;
  }
}

// Multipliers of one trailing row w.r.t. the block's pivots:
// t_q = ZP[q]*pan[q] - sum_{s<q} t_s prow_s[K+q] prod_{s<s'<q} z_s'  (REDC of R-scaled
// constants), tau_q = t_q * prod_{q<s'<B} z_s'.
__device__ __forceinline__ void oct_chain(const uint32_t* pan_ptr, const uint32_t* zp, const uint32_t* vr,
                                          const uint32_t* ze, const Mod32& m, uint32_t* tau) {
  const uint4 pa = *reinterpret_cast<const uint4*>(pan_ptr);
  const uint4 pb = *reinterpret_cast<const uint4*>(pan_ptr + 4);
  const uint32_t pan[OCT_B] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
  uint32_t t[OCT_B];
#pragma unroll
  for (int q = 0; q < OCT_B; ++q) {
    uint64_t acc = mad_wide(pan[q], zp[q], 0ull);
#pragma unroll
    for (int s2 = 0; s2 < q; ++s2) acc = mad_wide(t[s2], vr[q * (q - 1) / 2 + s2], acc);
    t[q] = oct_reduce(acc, m);
    tau[q] = mont(t[q], ze[q], m);
  }
}

template <class Src, bool DFT8, int LPM>
__global__ void __launch_bounds__(256)
det_octet_kernel(Src src, const int32_t* __restrict__ ids_g, int64_t node_lo, int64_t nodes,
                 uint32_t* __restrict__ out, unsigned long long* __restrict__ flag_count,
                 int64_t* __restrict__ flag_nodes, OctGeom g, Mod32 m) {
  static_assert(LPM == 8 || LPM == 16, "8 or 16 lanes per matrix");
  constexpr int GPW = 32 / LPM;                        // matrices per warp
  constexpr int HALVES = LPM / 8;                      // lanes sharing a trailing row
  extern __shared__ __align__(16) uint32_t smem[];
  const int r = g.r, S = g.S;
  int32_t* ids = reinterpret_cast<int32_t*>(smem);                  // r*r ids
  uint32_t* mats = smem + ((r * r + 3) & ~3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LPM, l = lane % LPM;
  const unsigned omask = (LPM == 32 ? 0xffffffffu : ((1u << LPM) - 1u)) << (grp * LPM);
  const int my = warp * GPW + grp;                     // matrix slot within the CTA
  uint32_t* A = mats + (size_t)my * g.MS;
  uint32_t* PB = A + r * S;                            // [B][16] panel [D | I], then V[s][S] (R-scaled, negated)
  uint32_t* ZPR = PB + OCT_B * PBW;                    // [B+1]   prod_{s<S} z_s * R
  uint32_t* ZETAR = ZPR + OCT_B + 1;                   // [B]     prod_{s<s'<B} z_s' * R
  uint32_t* ZR = ZETAR + OCT_B;                        // [B]     z_s * R
  uint32_t* CC = ZR + OCT_B;                           // [B][B]  -R^2 * C (U12 transform)
  const uint32_t p = m.p;
  const int cend = (r + 3) & ~3;

  for (int e = threadIdx.x; e < r * r; e += blockDim.x) ids[e] = ids_g[e];
  // padding columns [r, S) are zeroed once: fills write only the r*r real
  // entries and the elimination keeps padding at zero (0*ZPR + sum tau*0)
  for (int w = threadIdx.x; w < g.M * g.MS; w += blockDim.x) mats[w] = 0;
  const int64_t iters = (nodes + g.M - 1) / g.M;

  for (int64_t it = blockIdx.x; it < iters; it += gridDim.x) {
    __syncthreads();
    if constexpr (DFT8) oct_fill_dft8(src, mats, g, ids, it, node_lo);
    else oct_fill(src, mats, g, ids, it, node_lo, nodes);
    __syncthreads();
    int64_t node;
    if constexpr (DFT8) node = oct_node_dft8(it, my, g, src.NL);
    else node = oct_node_linear(it, my, g, nodes);
    if (node < 0) continue;

    uint32_t preR = m.r1, inflR = m.r1;   // Montgomery forms of prod z and prod z^(r-1-k)
    bool ok = true;
    for (int K = 0; K < r && ok; K += OCT_B) {
      const int Bk = (r - K) < OCT_B ? (r - K) : OCT_B;
      // ---------------- P phase: factor the augmented diagonal block [D | I] ----------------
      // PB = [D | I] (8 x 16, dense): D = rows/cols K..K+Bk-1 of the matrix, I = identity.
      // Division-free rank-1 steps leave, for every pivot row s, its final values
      // restricted to the block (PB[s][s+1..7]) and the transform C with
      // final row s = sum_{q<=s} C[s][q] * original row K+q (PB[s][8..15]);
      // every finished pivot row is stored as NPR (-R * value).
      for (int w = l; w < OCT_B * PBW; w += LPM) {
        const int q = w / PBW, c = w - q * PBW;
        uint32_t v = 0;
        if (q < Bk) v = c < Bk ? A[(K + q) * S + K + c] : (c - OCT_B == q ? 1u : 0u);
        PB[w] = v;
      }
      __syncwarp(omask);
      for (int s = 0; s < Bk; ++s) {
        const uint32_t z = PB[s * PBW + s];
        if (z == 0) { ok = false; break; }
        const uint32_t zR = to_mont(z, m);
        preR = mont(preR, zR, m);
        if (K + s + 1 < r) inflR = mont(inflR, preR, m);
        if (l == 0) ZR[s] = zR;
        const int a0 = (s + 1) & ~3;
        const int nch = (PBW - a0) >> 2;
        uint32_t* prow = PB + s * PBW;
        for (int ch = l; ch < nch; ch += LPM) {
          const int c = a0 + 4 * ch;
          uint4 v = *reinterpret_cast<const uint4*>(prow + c);
          uint32_t t0 = to_mont(v.x, m), t1 = to_mont(v.y, m), t2 = to_mont(v.z, m), t3 = to_mont(v.w, m);
          t0 = t0 ? p - t0 : 0u; t1 = t1 ? p - t1 : 0u; t2 = t2 ? p - t2 : 0u; t3 = t3 ? p - t3 : 0u;
          if (c + 0 > s) v.x = t0;
          if (c + 1 > s) v.y = t1;
          if (c + 2 > s) v.z = t2;
          if (c + 3 > s) v.w = t3;
          *reinterpret_cast<uint4*>(prow + c) = v;
        }
        __syncwarp(omask);
        const int items = (Bk - 1 - s) * nch;
        for (int idx = l; idx < items; idx += LPM) {
          const int jj = idx / nch, cc = idx - jj * nch;   // nch <= 4: cheap
          uint32_t* rj = PB + (s + 1 + jj) * PBW;
          const int c = a0 + 4 * cc;
          const uint32_t tj = rj[s];
          const uint4 np = *reinterpret_cast<const uint4*>(prow + c);
          uint4 a = *reinterpret_cast<const uint4*>(rj + c);
          const uint32_t n0 = oct_reduce(mad_wide(tj, np.x, mad_wide(a.x, zR, 0ull)), m);
          const uint32_t n1 = oct_reduce(mad_wide(tj, np.y, mad_wide(a.y, zR, 0ull)), m);
          const uint32_t n2 = oct_reduce(mad_wide(tj, np.z, mad_wide(a.z, zR, 0ull)), m);
          const uint32_t n3 = oct_reduce(mad_wide(tj, np.w, mad_wide(a.w, zR, 0ull)), m);
          if (c + 0 > s) a.x = n0;
          if (c + 1 > s) a.y = n1;
          if (c + 2 > s) a.z = n2;
          if (c + 3 > s) a.w = n3;
          *reinterpret_cast<uint4*>(rj + c) = a;
        }
        __syncwarp(omask);
      }
      if (!ok) break;
      if (K + OCT_B >= r) break;       // no trailing rows: elimination done
      // ---------------- U12: the pivot rows right of the block, all in one pass ----------------
      //   NPR_s[c] = -R * sum_{q<=s} C[s][q] a[K+q][c] = REDC(sum_q CC[s][q] a[K+q][c]),
      //   CC = -R^2 C mod p = to_mont(stored -R*C)
      for (int w = l; w < OCT_B * OCT_B; w += LPM) CC[w] = to_mont(PB[(w / OCT_B) * PBW + OCT_B + (w % OCT_B)], m);
      __syncwarp(omask);
      {
        uint32_t cc[OCT_B * (OCT_B + 1) / 2];
#pragma unroll
        for (int s = 0; s < OCT_B; ++s)
#pragma unroll
          for (int q = 0; q <= s; ++q) cc[s * (s + 1) / 2 + q] = CC[s * OCT_B + q];
        for (int c = K + OCT_B + l; c < r; c += LPM) {
          uint32_t a[OCT_B];
#pragma unroll
          for (int q = 0; q < OCT_B; ++q) a[q] = A[(K + q) * S + c];
#pragma unroll
          for (int s = 0; s < OCT_B; ++s) {
            uint64_t acc = 0;
#pragma unroll
            for (int q = 0; q <= s; ++q) acc = mad_wide(cc[s * (s + 1) / 2 + q], a[q], acc);
            A[(K + s) * S + c] = oct_reduce(acc, m);
          }
        }
      }
      // ---------------- block scalars (lane q <-> pivot q) ----------------
      // V[q][s] = NPR_q[K+s] * prod_{q<s'<s} z_s'  (in place in PB, q < s < 8)
      if (l < OCT_B) {
        const int q = l;
        uint32_t zz = m.r1;            // prod_{q<s'<s} z_s' * R
        for (int s = q + 1; s < OCT_B; ++s) {
          PB[q * PBW + s] = mont(PB[q * PBW + s], zz, m);
          zz = mont(zz, ZR[s], m);
        }
        ZETAR[q] = zz;
        if (l == 0) {
          uint32_t zp = m.r1;
          ZPR[0] = zp;
          for (int s = 0; s < OCT_B; ++s) { zp = mont(zp, ZR[s], m); ZPR[s + 1] = zp; }
        }
      }
      __syncwarp(omask);
      // ---------------- T phase: trailing rows ----------------
      // lane l: rows c0 + (l % 8) + 8u, column chunks (l / 8) + HALVES*v
      const int c0 = K + OCT_B;
      const uint32_t zpr = ZPR[OCT_B];
      const uint32_t* npr = A + K * S;                  // NPR_q[c] = npr[q * S + c]
      uint32_t vr[OCT_B * (OCT_B - 1) / 2], zp[OCT_B], ze[OCT_B];
#pragma unroll
      for (int q = 0; q < OCT_B; ++q) {
        zp[q] = ZPR[q];
        ze[q] = ZETAR[q];
#pragma unroll
        for (int s2 = 0; s2 < q; ++s2) vr[q * (q - 1) / 2 + s2] = PB[s2 * PBW + q];
      }
      const int half = l >> 3;
      for (int i = c0 + (l & 7); i < r; i += 8) {
        uint32_t* row = A + i * S;
        uint32_t tau[OCT_B];
        oct_chain(row + K, zp, vr, ze, m, tau);
        for (int c = c0 + 4 * half; c < cend; c += 4 * HALVES) {
          const uint4 a4 = *reinterpret_cast<const uint4*>(row + c);
          uint64_t a0 = mad_wide(a4.x, zpr, 0ull), a1 = mad_wide(a4.y, zpr, 0ull);
          uint64_t a2 = mad_wide(a4.z, zpr, 0ull), a3 = mad_wide(a4.w, zpr, 0ull);
#pragma unroll
          for (int q = 0; q < OCT_B; ++q) {
            const uint4 n4 = *reinterpret_cast<const uint4*>(npr + q * S + c);
            a0 = mad_wide(tau[q], n4.x, a0);
            a1 = mad_wide(tau[q], n4.y, a1);
            a2 = mad_wide(tau[q], n4.z, a2);
            a3 = mad_wide(tau[q], n4.w, a3);
          }
          uint4 o;
          o.x = oct_reduce(a0, m);
          o.y = oct_reduce(a1, m);
          o.z = oct_reduce(a2, m);
          o.w = oct_reduce(a3, m);
          *reinterpret_cast<uint4*>(row + c) = o;
        }
      }
      __syncwarp(omask);
    }
    if (l == 0) {
      if (ok) {
        // det = prod z / prod z^(r-1-k); Fermat inverse in Montgomery form:
        // mont_pow(infl*R, p-2) = infl^-1 * R, mont(pre*R, .) = det*R, mont(., 1) = det
        const uint32_t invR = mont_pow(inflR, (uint64_t)p - 2, m);
        out[node] = mont(mont(preR, invR, m), 1u, m);
      } else {
        unsigned long long slot = atomicAdd(flag_count, 1ull);
        flag_nodes[slot] = node_lo + node;
      }
    }
  }
}

inline OctGeom oct_geom(int r, int warps, int lpm, bool dft8) {
  OctGeom g;
  g.r = r;
  g.S = oct_row_stride(r);
  g.MS = ((r * g.S + OCT_SCALARS + 3) & ~3);
  g.M = warps * (32 / lpm);
  g.U = dft8 ? g.M / 8 : 0;
  return g;
}

inline size_t oct_smem(const OctGeom& g) {
  return sizeof(uint32_t) * ((size_t)((g.r * g.r + 3) & ~3) + (size_t)g.M * g.MS);
}

// Choose warps per CTA so that several CTAs share an SM (load/compute overlap)
// and the resident warp count is largest.
inline OctGeom oct_pick(int r, int lpm, bool dft8) {
  const size_t budget = 224 * 1024;
  OctGeom best = oct_geom(r, 32 / (32 / lpm) / 4 * 2, lpm, dft8);
  double best_score = -1;
  for (int warps = 1; warps <= 8; ++warps) {
    OctGeom g = oct_geom(r, warps, lpm, dft8);
    if (dft8 && (g.M % 8)) continue;
    const size_t sm = oct_smem(g) + 1024;
    const int ctas = (int)(budget / sm);
    if (ctas < 1) continue;
    const int resident = ctas * warps > 48 ? 48 : ctas * warps;   // warps per SM
    const double score = resident + 0.01 * ctas;
    if (score > best_score) { best_score = score; best = g; }
  }
  return best;
}

template <class Src, bool DFT8, int LPM>
int launch_octet_geom(PrimeCtx* ctx, const OctGeom& g, Src src, const int32_t* ids, int64_t node_lo,
                      int64_t nodes, uint32_t* out, unsigned long long* flag_count, int64_t* flag_nodes,
                      cudaStream_t st) {
  const size_t smem = oct_smem(g);
  if (cudaFuncSetAttribute(det_octet_kernel<Src, DFT8, LPM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return check_launch("det_octet attribute");
  const int ctas_per_sm = (int)((224 * 1024) / (smem + 1024));
  const int64_t iters = (nodes + g.M - 1) / g.M;
  const int64_t cap = (int64_t)ctx->sms * (ctas_per_sm > 0 ? ctas_per_sm : 1);
  const int grid = (int)(iters < cap ? iters : cap);
  const int threads = g.M * LPM;
  det_octet_kernel<Src, DFT8, LPM><<<grid, threads, smem, st>>>(src, ids, node_lo, nodes, out, flag_count,
                                                                 flag_nodes, g, ctx->m);
  count_launch();
  return check_launch("det_octet");
}

// lanes per matrix: 16 for the larger orders (more resident warps per SM), 8 below
inline int oct_lpm(int r) {
  static const char* env = getenv("PDB_OCT_LPM");
  if (env) return atoi(env) == 16 ? 16 : 8;
  return r >= 24 ? 16 : 8;
}

template <class Src, bool DFT8>
int launch_octet_lpm(PrimeCtx* ctx, int r, Src src, const int32_t* ids, int64_t node_lo, int64_t nodes,
                     uint32_t* out, unsigned long long* fc, int64_t* fn, cudaStream_t st) {
  if (oct_lpm(r) == 16)
    return launch_octet_geom<Src, DFT8, 16>(ctx, oct_pick(r, 16, DFT8), src, ids, node_lo, nodes, out, fc, fn, st);
  return launch_octet_geom<Src, DFT8, 8>(ctx, oct_pick(r, 8, DFT8), src, ids, node_lo, nodes, out, fc, fn, st);
}

inline int launch_octet(PrimeCtx* ctx, int r, StagedSrc src, const int32_t* ids, int64_t node_lo,
                        int64_t nodes, uint32_t* out, unsigned long long* flag_count, int64_t* flag_nodes,
                        cudaStream_t st) {
  return launch_octet_lpm<StagedSrc, false>(ctx, r, src, ids, node_lo, nodes, out, flag_count, flag_nodes, st);
}

inline int launch_octet(PrimeCtx* ctx, int r, FusedSrc src, const int32_t* ids, int64_t node_lo,
                        int64_t nodes, uint32_t* out, unsigned long long* flag_count, int64_t* flag_nodes,
                        cudaStream_t st) {
  const OctGeom g = oct_pick(r, oct_lpm(r), true);
  const bool dft8 = src.E <= 8 && src.NL >= 8 && src.NL % (8 * g.U) == 0 && node_lo % src.NL == 0 &&
                    nodes % src.NL == 0;
  if (dft8)
    return launch_octet_lpm<FusedSrc, true>(ctx, r, src, ids, node_lo, nodes, out, flag_count, flag_nodes, st);
  return launch_octet_lpm<FusedSrc, false>(ctx, r, src, ids, node_lo, nodes, out, flag_count, flag_nodes, st);
}

}  // namespace pdb
