// Determinants mod p of the r x r matrices at every evaluation node.
//
// The value is algorithm independent (reference determinant.py:1-8), so the
// kernels are free to choose their elimination order; they all return the
// exact det(M) mod p in [0, p).  Three kernels:
//
//  * det_small<R>   R <= 8: one lane per matrix, the matrix in registers,
//                   division-free elimination with diagonal pivots.
//  * det_gj         9 <= r <= 128 and odd p < 2^30: a lane group (8/16/32
//                   lanes) per matrix in shared memory, blocked Schur
//                   complements with an 8x8 Gauss-Jordan pivot block and
//                   delayed (64-bit accumulate + Montgomery) reduction
//                   (det_gj.cuh).
//  * det_robust     any r <= 128, any p < 2^31: one warp per matrix (shared
//                   memory) with the reference's exact pivot rule (first
//                   nonzero column of row i, determinant.py:136-169) and full
//                   division-free updates.
//
// The fast kernels only take diagonal pivots; a matrix whose diagonal pivot
// vanishes is appended to a node list and recomputed by det_robust, so every
// input (singular, structured, permuted) gets the exact answer.
#include <string>
#include <vector>
#include "pdb_internal.cuh"
#include "det_gj.cuh"

#ifndef PDB_GJ_LANES
#define PDB_GJ_LANES 16   // lanes per matrix up to order 40 (see gj_lanes); 8 and 32 build for experiments
#endif

namespace pdb {

struct FlagList {
  unsigned long long* count;
  int64_t* nodes;
};

__device__ __forceinline__ void flag_node(FlagList f, int64_t node) {
  unsigned long long slot = atomicAdd(f.count, 1ull);
  f.nodes[slot] = node;
}

// ---------------------------------------------------------------- robust ----
// The reference's exact rule (determinant.py:136-169), one warp per matrix with
// the matrix in shared memory: row i's pivot is its first nonzero column
// (found by ballots), the rows below get the division-free update
// z*row_k - t*row_i in parallel over (row, column) pairs, and
// det = prod z / prod z^(r-1-i) * (-1)^(inversions of the pivot columns).
// Any p < 2^31 (Barrett products: p = 2 and p >= 2^30 included).  Used for the
// rare nodes whose diagonal pivot vanished in the fast kernels, and for whole
// grids when no fast kernel applies.
constexpr int ROBUST_WARPS = 4;   // most warps per CTA (fewer for large orders: smem)

template <class Src>
__global__ void __launch_bounds__(32 * ROBUST_WARPS)
det_robust(Src src, const int32_t* __restrict__ ids, int r, const int64_t* __restrict__ list,
           const unsigned long long* __restrict__ list_count, int64_t count, int64_t node_lo,
           uint32_t* __restrict__ out, Mod32 m,
           uint32_t* __restrict__ trail_vals = nullptr, int32_t* __restrict__ trail_cols = nullptr) {
  extern __shared__ uint32_t rsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* A = rsm + (size_t)warp * (r * r + r);
  uint32_t* T = A + r * r;   // multiplier column of the current step
  const int64_t total = list ? (int64_t)*list_count : count;
  const uint32_t p = m.p;
  const int wpc = blockDim.x >> 5;
  const int64_t wstride = (int64_t)gridDim.x * wpc;
  for (int64_t idx = blockIdx.x * (int64_t)wpc + warp; idx < total; idx += wstride) {
    const int64_t node = list ? list[idx] : node_lo + idx;   // compact index
    const int64_t at = src.node(node);
    for (int e = lane; e < r * r; e += 32) A[e] = src.at(ids[e], at) % p;
    __syncwarp();
    uint32_t pre = 1 % p, infl = 1 % p;
    uint64_t used0 = 0, used1 = 0;   // pivot columns so far (r <= 128)
    int parity = 0;
    bool alive = true;
    for (int i = 0; i < r; ++i) {
      const uint32_t* row = A + i * r;
      int c = -1;
      for (int j0 = 0; j0 < r && c < 0; j0 += 32) {
        const unsigned nz = __ballot_sync(0xffffffffu, j0 + lane < r && row[j0 + lane] != 0);
        if (nz) c = j0 + __ffs(nz) - 1;
      }
      if (c < 0) { alive = false; break; }
      const uint32_t z = row[c];
      if (trail_vals && lane == 0) { trail_vals[i] = z; trail_cols[i] = c; }
      // earlier pivot columns to the right of c flip the permutation sign
      parity ^= (c < 64 ? __popcll(used0 >> c) + __popcll(used1) : __popcll(used1 >> (c - 64))) & 1;
      if (c < 64) used0 |= 1ull << c;
      else used1 |= 1ull << (c - 64);
      pre = mul_mod(pre, z, m);
      if (i + 1 < r) infl = mul_mod(infl, pre, m);
      // rows below: (r-1-i) x r updates with the multiplier column saved first
      const int rows = r - 1 - i;
      for (int k = lane; k < rows; k += 32) T[k] = A[(i + 1 + k) * r + c];
      __syncwarp();
      const int items = rows * r;
      for (int w = lane; w < items; w += 32) {
        const int kk = w / r, j = w - (w / r) * r;
        uint32_t* a = A + (i + 1 + kk) * r + j;
        *a = sub_mod(mul_mod(z, *a, m), mul_mod(T[kk], row[j], m), p);
      }
      __syncwarp();
    }
    if (lane == 0) {
      uint32_t det = 0;
      if (alive) {
        det = mul_mod(pre, inv_mod(infl, m), m);
        if (parity && det) det = p - det;
      }
      out[node - node_lo] = det;
    }
    __syncwarp();
  }
}

// One CTA (all its warps) per flagged node, odd p < 2^31: the same pivot rule
// and elimination as det_robust, but each step's (r-1-i) x r updates are
// spread over the CTA and done as one REDC of two products (the pivot and
// the multipliers in Montgomery form, the entries plain).  The flagged nodes
// of a fused launch are rare and few (~1 per 10^7 nodes), so what matters is
// the latency of one determinant: ~5 us instead of ~190 us for r = 40 with a
// warp and Barrett products.
template <class Src>
__global__ void __launch_bounds__(256)
det_robust_cta(Src src, const int32_t* __restrict__ ids, int r, const int64_t* __restrict__ list,
               const unsigned long long* __restrict__ list_count, int64_t node_lo, uint32_t* __restrict__ out,
               Mod32 m) {
  extern __shared__ uint32_t rsm[];
  uint32_t* A = rsm;          // r x r, plain canonical residues
  uint32_t* T = A + r * r;    // multiplier column of the step, Montgomery forms (negated)
  __shared__ int s_c;
  __shared__ uint32_t s_z;
  const int64_t total = (int64_t)*list_count;
  const uint32_t p = m.p;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  for (int64_t idx = blockIdx.x; idx < total; idx += gridDim.x) {
    const int64_t node = list[idx];
    const int64_t at = src.node(node);
    __syncthreads();
    for (int e = tid; e < r * r; e += nt) A[e] = src.at(ids[e], at) % p;
    __syncthreads();
    uint32_t pre = 1 % p, infl = 1 % p;
    uint64_t used0 = 0, used1 = 0;
    int parity = 0;
    bool alive = true;
    for (int i = 0; i < r; ++i) {
      const uint32_t* row = A + i * r;
      if (tid < 32) {   // first nonzero column of row i
        int c = -1;
        for (int j0 = 0; j0 < r && c < 0; j0 += 32) {
          const unsigned nz = __ballot_sync(0xffffffffu, j0 + lane < r && row[j0 + lane] != 0);
          if (nz) c = j0 + __ffs(nz) - 1;
        }
        if (lane == 0) { s_c = c; s_z = c >= 0 ? row[c] : 0u; }
      }
      __syncthreads();
      const int c = s_c;
      if (c < 0) { alive = false; break; }
      const uint32_t z = s_z;
      if (tid == 0) {
        parity ^= (c < 64 ? __popcll(used0 >> c) + __popcll(used1) : __popcll(used1 >> (c - 64))) & 1;
        if (c < 64) used0 |= 1ull << c;
        else used1 |= 1ull << (c - 64);
        pre = mul_mod(pre, z, m);
        if (i + 1 < r) infl = mul_mod(infl, pre, m);
      }
      const uint32_t zR = to_mont(z, m);
      const int rows = r - 1 - i;
      for (int k = tid; k < rows; k += nt) {
        const uint32_t t = to_mont(A[(i + 1 + k) * r + c], m);
        T[k] = t ? p - t : 0u;
      }
      __syncthreads();
      const int items = rows * r;
      for (int w = tid; w < items; w += nt) {
        const int kk = w / r, j = w - (w / r) * r;
        uint32_t* a = A + (i + 1 + kk) * r + j;
        *a = csub(redc(mad_wide(zR, *a, mad_wide(T[kk], row[j], 0ull)), m), p);
      }
      __syncthreads();
    }
    if (tid == 0) {
      uint32_t det = 0;
      if (alive) {
        det = mul_mod(pre, inv_mod(infl, m), m);
        if (parity && det) det = p - det;
      }
      out[node - node_lo] = det;
    }
  }
}

// ----------------------------------------------------------------- small ----
// One lane per matrix, D matrices per lane (D = 4 for r <= 4, 2 for r <= 6):
// the entries are read as Montgomery forms of A' = A R^-1 (no conversion), the
// division-free elimination row_i <- z row_i - t row_k is one REDC of two
// products, and the D x 32 inflations of a warp share one Fermat inversion
// (prefix products within the lane, then across the warp by shuffles).
// det A = det A' * R^r is applied by the last Montgomery product (Rr = R^r).
// Valid for odd p < 2^31: two products < 2 p^2 keep REDC's bound and its
// output below 2p, one conditional subtraction makes it canonical.
template <int R, class Src>
__global__ void __launch_bounds__(128)
det_small(Src src, const int32_t* __restrict__ ids_g, int64_t node_lo, int64_t nodes,
          uint32_t* __restrict__ out, FlagList flags, Mod32 m, uint32_t Rr) {
#ifndef PDB_SMALL_D4
#define PDB_SMALL_D4 4
#endif
  constexpr int D = R <= 4 ? PDB_SMALL_D4 : (R <= 6 ? 2 : 1);
  __shared__ int32_t ids[R * R];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) ids[e] = ids_g[e];
  __syncthreads();
  const uint32_t p = m.p, one = m.r1;
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count: every lane takes part in the batched inversion
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * D;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) * D; base < nodes; base += stride) {
    uint32_t a[D][R][R];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t idx = base + d * 32 + lane;
      const int64_t node = src.node(node_lo + (idx < nodes ? idx : 0));
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) a[d][i][j] = src.at(ids[i * R + j], node);
    }
    uint32_t pre[D], infl[D];
    bool ok[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      pre[d] = one;
      infl[d] = one;
      ok[d] = true;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const uint32_t z = a[d][k][k];
        ok[d] = ok[d] && z != 0;
        pre[d] = gj_mont(pre[d], z, m);
        if (k + 1 < R) infl[d] = gj_mont(infl[d], pre[d], m);
#pragma unroll
        for (int i = k + 1; i < R; ++i) {
          const uint32_t nt = p - a[d][i][k];   // in (0, p]
#pragma unroll
          for (int j = k + 1; j < R; ++j)
            a[d][i][j] = gj_red2(mad_wide(a[d][k][j], nt, mad_wide(a[d][i][j], z, 0ull)), m);
        }
      }
    }
    // batched inversion: lane-local prefix products, then across the warp
    uint32_t lp[D];
    uint32_t run = one;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const bool use = base + d * 32 + lane < nodes && ok[d];
      run = gj_mont(run, use ? infl[d] : one, m);
      lp[d] = run;
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
    uint32_t inv_total = one;   // total^(p-2), square and multiply
    {
      uint32_t b = total;
      for (uint32_t e = p - 2; e; e >>= 1) {
        if (e & 1) inv_total = gj_mont(inv_total, b, m);
        b = gj_mont(b, b, m);
      }
    }
    uint32_t left = __shfl_up_sync(0xffffffffu, pre_x, 1);
    uint32_t right = __shfl_down_sync(0xffffffffu, suf_x, 1);
    if (lane == 0) left = one;
    if (lane == 31) right = one;
    uint32_t inv = gj_mont(gj_mont(left, right, m), inv_total, m);   // 1 / (this lane's product)
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      const int64_t idx = base + d * 32 + lane;
      const bool valid = idx < nodes;
      const bool use = valid && ok[d];
      const uint32_t inv_d = d ? gj_mont(inv, lp[d - 1], m) : inv;   // 1 / infl[d]
      if (use) inv = gj_mont(inv, infl[d], m);
      if (valid) {
        if (ok[d]) out[idx] = gj_mont(gj_mont(pre[d], inv_d, m), Rr, m);
        else flag_node(flags, node_lo + idx);
      }
    }
  }
}

// 2^(32 r) mod p: the Montgomery scale of an r x r determinant.
static uint32_t mont_scale(const Mod32& m, int r) {
  uint64_t acc = 1 % m.p, b = m.r1;
  for (int e = r; e; e >>= 1) {
    if (e & 1) acc = (uint64_t)((unsigned __int128)acc * b % m.p);
    b = (uint64_t)((unsigned __int128)b * b % m.p);
  }
  return (uint32_t)acc;
}

template <class Src>
static int launch_small(int r, Src src, const int32_t* ids, int64_t lo, int64_t n, uint32_t* out,
                        FlagList f, Mod32 m, int grid, cudaStream_t st) {
  switch (r) {
#define PDB_SMALL(R) case R: det_small<R, Src><<<grid, 128, 0, st>>>(src, ids, lo, n, out, f, m, mont_scale(m, R)); count_launch(); break;
    PDB_SMALL(1) PDB_SMALL(2) PDB_SMALL(3) PDB_SMALL(4)
    PDB_SMALL(5) PDB_SMALL(6) PDB_SMALL(7) PDB_SMALL(8)
#undef PDB_SMALL
    default: return -1;
  }
  return 0;
}

size_t det_scratch_bytes(int r, int64_t nodes) {
  (void)r;   // flag count + flagged node list + one denominator per node + the row table
  return 256 + sizeof(int64_t) * (size_t)nodes + sizeof(uint32_t) * ((size_t)nodes + 3) +
         sizeof(int64_t) * ((size_t)nodes / 8 + 2) + 16;
}

// Full outer index of every compact last-axis row a fused launch touches (pruned maps).
__global__ void fused_row_table(NodeMap map, int64_t orow0, int64_t rows, int64_t klast, int lognl,
                                int64_t* __restrict__ table) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < rows; j += (int64_t)gridDim.x * blockDim.x)
    table[j] = map.full((orow0 + j) * klast) >> lognl;
}

static void prepare_src(PrimeCtx*, StagedSrc&, char*, int64_t, int64_t, cudaStream_t) {}

static void prepare_src(PrimeCtx* ctx, FusedSrc& src, char* tail, int64_t node_lo, int64_t nodes, cudaStream_t st) {
  (void)node_lo;
  if (!src.map.nd || src.ulast < 1) return;
  const int64_t klast = 8 * (int64_t)src.ulast;
  const int64_t rows = (nodes + klast - 1) / klast + 1;
  int64_t* table = reinterpret_cast<int64_t*>((reinterpret_cast<uintptr_t>(tail) + 15) & ~uintptr_t(15));
  const int64_t blocks = (rows + 255) / 256;
  const int g = (int)(blocks < (int64_t)ctx->sms * 4 ? blocks : (int64_t)ctx->sms * 4);
  fused_row_table<<<g, 256, 0, st>>>(src.map, src.orow0, rows, klast, __builtin_ctz((unsigned)src.NL), table);
  count_launch();
  src.orow_full = table;
}

template <class Src>
static void launch_robust(PrimeCtx* ctx, Src src, const int32_t* ids, int r, const int64_t* list,
                          const unsigned long long* list_count, int64_t count, int64_t node_lo, uint32_t* out,
                          cudaStream_t st, uint32_t* trail_vals = nullptr, int32_t* trail_cols = nullptr) {
  const size_t per_warp = sizeof(uint32_t) * (size_t)(r * r + r);
  if (list && !trail_vals && ctx->m.odd() && per_warp <= 96 * 1024) {
    // flagged nodes of a fast launch: one CTA per node (latency, not throughput)
    if (per_warp > 48 * 1024)
      cudaFuncSetAttribute(det_robust_cta<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per_warp);
    det_robust_cta<Src><<<ctx->sms, 256, per_warp, st>>>(src, ids, r, list, list_count, node_lo, out, ctx->m);
    count_launch();
    return;
  }
  int warps = (int)((200u * 1024u) / per_warp);
  warps = warps < 1 ? 1 : (warps > ROBUST_WARPS ? ROBUST_WARPS : warps);
  const size_t smem = per_warp * warps;
  cudaFuncSetAttribute(det_robust<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // flagged lists are short (a few nodes per 10^7): one wave; whole grids: 8 CTAs per SM
  const int64_t want = list ? (int64_t)ctx->sms : (count + warps - 1) / warps;
  const int64_t cap = (int64_t)ctx->sms * 8;
  const int grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  det_robust<Src><<<grid, 32 * warps, smem, st>>>(src, ids, r, list, list_count, count, node_lo, out,
                                                  ctx->m, trail_vals, trail_cols);
  count_launch();
}

template <class Src, bool DFT8, int LPM, bool P31, int RPC, bool PAIR = false>
static int launch_gj_geom(PrimeCtx* ctx, const GjGeom& g, Src src, const int32_t* ids, int64_t node_lo,
                          int64_t nodes, uint32_t* out, uint32_t* den, unsigned long long* fc, int64_t* fn,
                          cudaStream_t st) {
  const size_t smem = gj_smem(g);
  if (cudaFuncSetAttribute(det_gj_kernel<Src, DFT8, LPM, P31, RPC, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return check_launch("det_gj attribute");
  int ctas_per_sm = 0;
  const int threads = g.M * LPM;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, det_gj_kernel<Src, DFT8, LPM, P31, RPC, PAIR>, threads, smem);
  if (ctas_per_sm < 1) ctas_per_sm = 1;
  static const char* cenv = getenv("PDB_GJ_CTAS");   // experiments: cap resident CTAs per SM
  if (cenv && *cenv && atoi(cenv) > 0 && atoi(cenv) < ctas_per_sm) ctas_per_sm = atoi(cenv);
  const int64_t iters = DFT8 ? (nodes / 8 + g.U - 1) / g.U : (nodes + g.M - 1) / g.M;
  const int64_t cap = (int64_t)ctx->sms * ctas_per_sm;
  const int grid = (int)(iters < cap ? iters : cap);
  if (grid < 1) return 0;
  const int kt = ktimer_start(st);
  det_gj_kernel<Src, DFT8, LPM, P31, RPC, PAIR><<<grid, threads, smem, st>>>(src, ids, node_lo, nodes, out, den, fc, fn, g, ctx->m);
  ktimer_stop(kt, st);
  count_launch();
  if (int rc = check_launch("det_gj")) return rc;
  const int64_t fblocks = (nodes + 256 * GJ_FIN_D - 1) / (256 * GJ_FIN_D);
  const int fgrid = (int)(fblocks < (int64_t)ctx->sms * 8 ? fblocks : (int64_t)ctx->sms * 8);
  det_gj_finalize<<<fgrid, 256, 0, st>>>(out, den, nodes, mont_scale(ctx->m, g.r), ctx->m);
  count_launch();
  return check_launch("det_gj_finalize");
}

// Lanes per matrix: 16 up to order 40 (measured sweep, r = 10..40) and at 56 / 64;
// 32 at padded order 48 and from 72 on, where few matrices fit in shared memory
// and more lanes per matrix hide latency (profiles/README_r01.md: r = 44 +33 %,
// 96 +28 %, 128 +160 %; r = 64 -57 %, its 64-word rows share banks).
static int gj_lanes(int r) {
  const int RP = (r + 7) & ~7;
  return (RP == 48 || RP >= 72) ? 32 : PDB_GJ_LANES;
}

// Paired pivot blocks (det_gj_kernel<..., PAIR>) accumulate 17 products of
// canonical residues: 17 (p-1)^2 < 2^64, and after hi(acc) -= 2p when hi >= 2p,
// hi + p < 2^32 (REDC's bound).  p < 1.0417e9: every prime the reference plans from
// its default prime_start = 10**9 for up to thousands of primes.
static bool gj_pair_ok(uint32_t p) {
  if (getenv("PDB_GJ_NO_PAIR")) return false;
  const unsigned __int128 pm = p - 1;
  const unsigned __int128 acc = 17 * pm * pm;
  if (acc >> 64) return false;
  const uint64_t hi = (uint64_t)(acc >> 32);
  const uint64_t hi2 = hi >= 2ull * p ? hi - 2ull * p : hi;
  const uint64_t hmax = hi2 > 2ull * p - 1 ? hi2 : 2ull * p - 1;
  return hmax + p < (1ull << 32);
}

template <class Src, bool DFT8>
static int launch_gj_mode(PrimeCtx* ctx, int r, Src src, const int32_t* ids, int64_t node_lo, int64_t nodes,
                         uint32_t* out, uint32_t* den, unsigned long long* fc, int64_t* fn, cudaStream_t st) {
  // 2^30 <= p < 2^31 (not fast) reduces pairs of products
  if (gj_lanes(r) == 32 && PDB_GJ_LANES != 32) {
    const GjGeom g = gj_pick(r, 32, DFT8);
    if (ctx->m.fast()) return launch_gj_geom<Src, DFT8, 32, false, 0>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn, st);
    return launch_gj_geom<Src, DFT8, 32, true, 0>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn, st);
  }
  const GjGeom g = gj_pick(r, PDB_GJ_LANES, DFT8);
  // compile-time orders: 40 (C5) and 16 (C3/C4) for both sources, 24 and 32 for
  // staged grids; the fused DFT-8 fill of the compile-time kernels assumes
  // 256-thread CTAs, the staged ones take any CTA size
  const bool rpc = (!DFT8 || g.M * PDB_GJ_LANES == 256) && !getenv("PDB_GJ_NO_RPC");
  if (ctx->m.fast()) {
    if (g.RP == 40 && rpc && gj_pair_ok(ctx->m.p))
      return launch_gj_geom<Src, DFT8, PDB_GJ_LANES, false, 40, true>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn,
                                                                      st);
    if (g.RP == 40 && rpc)
      return launch_gj_geom<Src, DFT8, PDB_GJ_LANES, false, 40>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn, st);
    if (g.RP == 16 && rpc)
      return launch_gj_geom<Src, DFT8, PDB_GJ_LANES, false, 16>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn, st);
    if constexpr (!DFT8) {
      if (g.RP == 24 && rpc)
        return launch_gj_geom<Src, DFT8, PDB_GJ_LANES, false, 24>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn, st);
      if (g.RP == 32 && rpc)
        return launch_gj_geom<Src, DFT8, PDB_GJ_LANES, false, 32>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn, st);
    }
    return launch_gj_geom<Src, DFT8, PDB_GJ_LANES, false, 0>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn, st);
  }
  if (g.RP == 40 && rpc)
    return launch_gj_geom<Src, DFT8, PDB_GJ_LANES, true, 40>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn, st);
  if (g.RP == 16 && rpc)
    return launch_gj_geom<Src, DFT8, PDB_GJ_LANES, true, 16>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn, st);
  return launch_gj_geom<Src, DFT8, PDB_GJ_LANES, true, 0>(ctx, g, src, ids, node_lo, nodes, out, den, fc, fn, st);
}

static int launch_gj(PrimeCtx* ctx, int r, StagedSrc src, const int32_t* ids, int64_t node_lo, int64_t nodes,
                     uint32_t* out, uint32_t* den, unsigned long long* fc, int64_t* fn, cudaStream_t st) {
  return launch_gj_mode<StagedSrc, false>(ctx, r, src, ids, node_lo, nodes, out, den, fc, fn, st);
}

static int launch_gj(PrimeCtx* ctx, int r, FusedSrc src, const int32_t* ids, int64_t node_lo, int64_t nodes,
                     uint32_t* out, uint32_t* den, unsigned long long* fc, int64_t* fn, cudaStream_t st) {
  const GjGeom g = gj_pick(r, gj_lanes(r), true);
  // whole compact last-axis rows of 8 * ulast nodes (u-pairs may straddle rows)
  const int64_t klast = 8 * (int64_t)src.ulast;
  const bool dft8 = src.E <= 8 && src.NL >= 8 && src.ulast >= 1 &&
                    node_lo % klast == 0 && nodes % klast == 0;
  if (dft8) return launch_gj_mode<FusedSrc, true>(ctx, r, src, ids, node_lo, nodes, out, den, fc, fn, st);
  return launch_gj_mode<FusedSrc, false>(ctx, r, src, ids, node_lo, nodes, out, den, fc, fn, st);
}

template <class Src>
int det_run(PrimeCtx* ctx, Src src, const int32_t* ids, int r, int64_t node_lo, int64_t nodes,
            uint32_t* out, void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (r < 1 || r > PDB_MAX_ORDER) {
    set_error("unsupported matrix order %d (1..%d)", r, PDB_MAX_ORDER);
    return -2;
  }
  if (nodes == 0) return 0;
  if (scratch_bytes < det_scratch_bytes(r, nodes)) {
    set_error("det scratch too small: %zu < %zu", scratch_bytes, det_scratch_bytes(r, nodes));
    return -2;
  }
  char* base = static_cast<char*>(scratch);
  FlagList flags{reinterpret_cast<unsigned long long*>(base), reinterpret_cast<int64_t*>(base + 256)};
  uint32_t* den = reinterpret_cast<uint32_t*>(base + 256 + sizeof(int64_t) * (size_t)nodes);
  prepare_src(ctx, src, reinterpret_cast<char*>(den + nodes + 3), node_lo, nodes, st);
  const Mod32 m = ctx->m;
  bool fast = false;
  if (cudaMemsetAsync(flags.count, 0, sizeof(unsigned long long), st) != cudaSuccess)
    return check_launch("det memset");
  if (r <= 8 && m.odd()) {
    const int per_lane = r <= 4 ? PDB_SMALL_D4 : (r <= 6 ? 2 : 1);   // det_small's D
    int64_t blocks = (nodes + 128 * per_lane - 1) / (128 * per_lane);
    int grid = (int)(blocks < (int64_t)ctx->sms * 32 ? blocks : (int64_t)ctx->sms * 32);
    launch_small(r, src, ids, node_lo, nodes, out, flags, m, grid, st);
    fast = true;
  } else if (m.odd() && m.p < (1u << 31)) {   // det_gj: p < 2^30 fast mode, [2^30, 2^31) paired mode
    if (launch_gj(ctx, r, src, ids, node_lo, nodes, out, den, flags.count, flags.nodes, st) == 0) fast = true;
  }
  if (int rc = check_launch("det fast path")) return rc;
  if (fast) launch_robust(ctx, src, ids, r, flags.nodes, flags.count, 0, node_lo, out, st);
  else launch_robust(ctx, src, ids, r, nullptr, nullptr, nodes, node_lo, out, st);
  return check_launch("det_robust");
}

int condense_run(PrimeCtx* ctx, const uint32_t* mat, int r, uint32_t* trail_vals, int32_t* trail_cols,
                 uint32_t* det_out, void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (r < 1 || r > PDB_MAX_ORDER) {
    set_error("unsupported matrix order %d (1..%d)", r, PDB_MAX_ORDER);
    return -2;
  }
  const size_t need = sizeof(int32_t) * r * r + 256 + sizeof(uint32_t) * (size_t)r * r * 128;
  if (scratch_bytes < need) {
    set_error("condense scratch too small");
    return -2;
  }
  std::vector<int32_t> ids(r * r);
  for (int e = 0; e < r * r; ++e) ids[e] = e;
  int32_t* d_ids = static_cast<int32_t*>(scratch);
  cudaMemcpyAsync(d_ids, ids.data(), sizeof(int32_t) * r * r, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(trail_cols, 0xff, sizeof(int32_t) * r, st);
  cudaStreamSynchronize(st);
  StagedSrc src{mat, 1};
  launch_robust(ctx, src, d_ids, r, nullptr, nullptr, 1, 0, det_out, st, trail_vals, trail_cols);
  return check_launch("condense");
}

template int det_run<StagedSrc>(PrimeCtx*, StagedSrc, const int32_t*, int, int64_t, int64_t,
                                uint32_t*, void*, size_t, cudaStream_t);
template int det_run<FusedSrc>(PrimeCtx*, FusedSrc, const int32_t*, int, int64_t, int64_t,
                               uint32_t*, void*, size_t, cudaStream_t);

}  // namespace pdb
