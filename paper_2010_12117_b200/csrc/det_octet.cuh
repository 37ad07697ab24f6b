// det_octet: blocked division-free elimination, 8 lanes per matrix.
//
// Why this shape (measured in profiles/intpipe_r01.json):
//   * IMAD.WIDE (64-bit multiply-accumulate) issues at half rate like
//     IMAD.HI, so a Shoup mul-mod costs 4 fma-heavy slots while a delayed
//     64-bit MAC costs 2.  Accumulating the B+1 products of a rank-B block
//     update in 64 bits and reducing once (Montgomery REDC + Barrett) halves
//     the slot count per elimination update.
//   * Normalised multipliers need one modular inverse per pivot; with only
//     ~32 resident 40x40 matrices per SM the per-step Fermat inverses would
//     cost as much as the updates.  The division-free (condensation) form of
//     the reference (determinant.py:136-169) needs one inverse per matrix;
//     here its per-row scalings are folded into scalars (tau, ZP, V below),
//     so the elimination itself stays at ~(B+1)/B MACs per update.
//
// Algorithm for one block of pivots K..K+B-1 (z_s = pivot s, prow_s its row):
//   row_i after S pivots = ZP[S]*row_i - sum_{s<S} t_s * zeta_s^(S) * prow_s
//   with ZP[S] = prod_{s<S} z_s, zeta_s^(S) = prod_{s<s'<S} z_s', and the
//   multipliers t_s = (row_i after s pivots)[K+s], obtained by the recurrence
//   t_S = ZP[S]*a[i][K+S] + sum_{s<S} t_s * V[s][S],  V[s][S] = -zeta_s^(S) prow_s[K+S].
//   Pivot rows are stored as NPR = -R*prow mod p (R = 2^32) so that every
//   accumulation is  a*ZPR + sum tau*NPR  == R*(new value), which a single
//   REDC turns back into the value.  At most B+1 = 9 products (< 2^60 each
//   for p < 2^30) are accumulated, inside REDC's bound.
//   det = prod z_k / prod z_k^(r-1-k) (one inverse per matrix).
// A zero diagonal pivot aborts the matrix and appends its node to the
// robust kernel's list.
#pragma once
#include "pdb_internal.cuh"

namespace pdb {

constexpr int OCT_B = 8;      // pivots per block
constexpr int OCT_LPM = 8;    // lanes per matrix

struct OctGeom {
  int r;       // matrix order
  int S;       // row stride (words), multiple of 4, >= ceil4(r)
  int MS;      // matrix stride (words) incl. scalar area
  int M;       // matrices per CTA iteration (= 4 * warps)
};

__host__ __device__ inline int oct_row_stride(int r) {
  int S = (r + 3) & ~3;
  while (((S >> 2) & 1) == 0) S += 4;  // S/4 odd -> 8 rows hit 8 distinct 16B bank groups
  return S;
}

// scalar area per matrix: V table (B*B), ZPR (B+1), ZETA (B), ZETAs (B), z (B)
constexpr int OCT_SCALARS = OCT_B * OCT_B + (OCT_B + 1) + 3 * OCT_B;

__device__ __forceinline__ uint32_t oct_reduce(uint64_t acc, const Mod32& m) {
  return canon32(redc(acc, m), m);
}

template <class Src>
__global__ void __launch_bounds__(256)
det_octet_kernel(Src src, const int32_t* __restrict__ ids_g, int64_t node_lo, int64_t nodes,
                 uint32_t* __restrict__ out, unsigned long long* __restrict__ flag_count,
                 int64_t* __restrict__ flag_nodes, OctGeom g, Mod32 m) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int r = g.r, S = g.S;
  int32_t* ids = reinterpret_cast<int32_t*>(smem);                  // r*r ids
  uint32_t* mats = smem + ((r * r + 3) & ~3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int oct = lane >> 3, l = lane & 7;
  const unsigned omask = 0xffu << (oct * 8);
  const int my = warp * 4 + oct;                       // matrix slot within the CTA
  uint32_t* A = mats + (size_t)my * g.MS;
  uint32_t* V = A + r * S;                             // [B][B]
  uint32_t* ZPR = V + OCT_B * OCT_B;                   // [B+1]
  uint32_t* ZETA = ZPR + OCT_B + 1;                    // [B]
  uint32_t* ZETAs = ZETA + OCT_B;                      // [B]
  uint32_t* Z = ZETAs + OCT_B;                         // [B] raw pivots of this block
  const uint32_t p = m.p;
  const int nwarps = blockDim.x >> 5;

  for (int e = threadIdx.x; e < r * r; e += blockDim.x) ids[e] = ids_g[e];

  for (int64_t base = (int64_t)blockIdx.x * g.M; base < nodes; base += (int64_t)gridDim.x * g.M) {
    __syncthreads();
    // ---- load: warp w fills positions w, w+nw, ...; lane = matrix slot ----
    const int nload = (int)((nodes - base) < g.M ? (nodes - base) : g.M);
    for (int pos = warp; pos < r * S; pos += nwarps) {
      const int i = pos / S, j = pos - i * S;
      if (lane < g.M) {
        uint32_t v = 0;
        if (j < r && lane < nload) v = src.get(ids[i * r + j], node_lo + base + lane);
        mats[(size_t)lane * g.MS + pos] = v;
      }
    }
    __syncthreads();
    if (my >= nload) continue;
    const int64_t node = node_lo + base + my;

    uint32_t pre = 1, infl = 1;
    bool ok = true;
    for (int K = 0; K < r && ok; K += OCT_B) {
      const int Bk = (r - K) < OCT_B ? (r - K) : OCT_B;
      if (l == 0) ZPR[0] = m.r1;
      __syncwarp(omask);
      // ---------------- pivot rows ----------------
      for (int s = 0; s < Bk; ++s) {
        const int k = K + s;
        // multipliers t_0..t_{s-1} of row k (every lane, redundantly)
        uint32_t t[OCT_B], tau[OCT_B];
#pragma unroll
        for (int q = 0; q < OCT_B; ++q) {
          if (q < s) {
            uint64_t acc = (uint64_t)A[k * S + K + q] * ZPR[q];
#pragma unroll
            for (int s2 = 0; s2 < OCT_B; ++s2)
              if (s2 < q) acc += (uint64_t)t[s2] * V[s2 * OCT_B + q];
            t[q] = oct_reduce(acc, m);
          }
        }
        // tau_q = t_q * prod_{q<s'<s} z_s'
        uint32_t zeta = 1;
#pragma unroll
        for (int q = OCT_B - 1; q >= 0; --q) {
          if (q < s) {
            tau[q] = mul_mod(t[q], zeta, m);
            zeta = mul_mod(zeta, Z[q], m);
          }
        }
        const uint32_t zpr = ZPR[s];
        for (int c = k + l; c < r; c += OCT_LPM) {
          uint64_t acc = (uint64_t)A[k * S + c] * zpr;
#pragma unroll
          for (int q = 0; q < OCT_B; ++q)
            if (q < s) acc += (uint64_t)tau[q] * A[(K + q) * S + c];
          const uint32_t v = oct_reduce(acc, m);
          if (c == k) {
            A[k * S + c] = v;
          } else {
            const uint32_t vr = shoup_mul(v, m.r1, m.r1s, p);
            A[k * S + c] = vr ? p - vr : 0u;     // NPR_s[c] = -R * prow_s[c]
          }
        }
        __syncwarp(omask);
        const uint32_t z = A[k * S + k];
        if (z == 0) { ok = false; break; }
        pre = mul_mod(pre, z, m);
        if (k + 1 < r) infl = mul_mod(infl, pre, m);
        if (l == 0) {
          Z[s] = z;
          ZPR[s + 1] = mul_mod(ZPR[s], z, m);
        }
        // V[q][s+1] = NPR_q[K+s+1] * prod_{q<s'<=s} z_s'  (column s+1 of the table)
        if (s + 1 < Bk && l <= s) {
          uint32_t prod = 1;
          for (int s2 = l + 1; s2 < s; ++s2) prod = mul_mod(prod, A[(K + s2) * S + K + s2], m);
          if (l < s) prod = mul_mod(prod, z, m);
          V[l * OCT_B + s + 1] = mul_mod(A[(K + l) * S + K + s + 1], prod, m);
        }
        __syncwarp(omask);
      }
      if (!ok) break;
      // zeta_q = prod_{q<s'<Bk} z_s'  (Shoup constants for the trailing rows)
      if (l == 0) {
        uint32_t zeta = 1;
        for (int q = Bk - 1; q >= 0; --q) {
          ZETA[q] = zeta;
          ZETAs[q] = shoup_companion_fast(zeta, m);
          zeta = mul_mod(zeta, Z[q], m);
        }
      }
      __syncwarp(omask);
      // ---------------- trailing rows (lanes split rows) ----------------
      // Trailing rows exist only when r - K > B, i.e. for full blocks (Bk == OCT_B),
      // so everything below is unrolled over the compile-time block size.
      const int c0 = K + OCT_B;
      const int cend = (r + 3) & ~3;
      const uint32_t zpr = ZPR[OCT_B];
      const uint32_t* npr = A + K * S;                  // NPR_q[c] = npr[q * S + c]
      for (int i = c0 + l; i < r; i += OCT_LPM) {
        uint32_t* row = A + i * S;
        uint32_t t[OCT_B], tau[OCT_B];
#pragma unroll
        for (int q = 0; q < OCT_B; ++q) {
          uint64_t acc = mad_wide(row[K + q], ZPR[q], 0ull);
#pragma unroll
          for (int s2 = 0; s2 < q; ++s2) acc = mad_wide(t[s2], V[s2 * OCT_B + q], acc);
          t[q] = oct_reduce(acc, m);
          tau[q] = shoup_mul(t[q], ZETA[q], ZETAs[q], p);
        }
        for (int c = c0; c < cend; c += 4) {
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
        out[node - node_lo] = mul_mod(pre, inv_mod(infl, m), m);
      } else {
        unsigned long long slot = atomicAdd(flag_count, 1ull);
        flag_nodes[slot] = node;
      }
    }
  }
}

inline OctGeom oct_geom(int r, int warps) {
  OctGeom g;
  g.r = r;
  g.S = oct_row_stride(r);
  g.MS = ((r * g.S + OCT_SCALARS + 3) & ~3);
  g.M = 4 * warps;
  return g;
}

inline size_t oct_smem(const OctGeom& g) {
  return sizeof(uint32_t) * ((size_t)((g.r * g.r + 3) & ~3) + (size_t)g.M * g.MS);
}

template <class Src>
int launch_octet(PrimeCtx* ctx, int r, Src src, const int32_t* ids, int64_t node_lo, int64_t nodes,
                 uint32_t* out, unsigned long long* flag_count, int64_t* flag_nodes, cudaStream_t st) {
  // largest CTA (<= 8 warps) such that two CTAs fit on an SM
  int warps = 8;
  OctGeom g = oct_geom(r, warps);
  while (warps > 1 && oct_smem(g) > 112 * 1024) g = oct_geom(r, --warps);
  const size_t smem = oct_smem(g);
  static bool attr_set[2] = {false, false};
  (void)attr_set;
  if (cudaFuncSetAttribute(det_octet_kernel<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return check_launch("det_octet attribute");
  int64_t ctas = (nodes + g.M - 1) / g.M;
  int64_t cap = (int64_t)ctx->sms * 2;
  int grid = (int)(ctas < cap ? ctas : cap);
  det_octet_kernel<Src><<<grid, warps * 32, smem, st>>>(src, ids, node_lo, nodes, out, flag_count,
                                                        flag_nodes, g, ctx->m);
  count_launch();
  return check_launch("det_octet");
}

}  // namespace pdb
