// Batched multivariate number-theoretic transforms (natural order in and out).
//
// Semantics follow the reference's `_multi` (transform.py:119-143): every
// axis of a row-major tensor gets the length-N_a transform
//     out[k] = sum_j x[j] * w^(jk),  w = omega^(2^(q - log2 N_a))
// (inverse: w^-1 and a final * N_a^-1 when N_a > 1).  The reference rotates
// the tensor after each axis pass; here every axis is transformed in place
// through its stride, so no transposition pass exists at all.
//
// Kernel: one CTA owns a tile of LO lines x TI neighbouring inner indices
// (TI consecutive words per row -> coalesced loads even for strided axes),
// loads it into shared memory in bit-reversed row order and runs the log2 N
// radix-2 DIT stages there with Shoup twiddles.  Lines that are entirely
// zero (outside the coefficient box on not-yet-transformed axes) are skipped
// ("pruning"): for an entry with (d+1)^vn coefficients only the first pass
// touches (d+1)^(vn-1) lines per entry.
#include <cstdlib>
#include "pdb_internal.cuh"
#include "dft8.cuh"

namespace pdb {

template <bool INV>
__global__ void __launch_bounds__(256)
ntt_axis_smem(uint32_t* __restrict__ data, AxisGeom g, int N, int logN, int logTI, int logLO,
              const uint32_t* __restrict__ tw, const uint32_t* __restrict__ tws,
              uint32_t ninv, uint32_t ninvs, Mod32 m) {
  // N, TI = 2^logTI inner columns and LO = 2^logLO lines per tile are powers of two:
  // all tile index arithmetic is shifts and masks.
  extern __shared__ uint32_t sm[];
  __shared__ int64_t line_base[16];
  const int TI = 1 << logTI, LO = 1 << logLO;
  const int64_t tchunks = (g.inner + TI - 1) >> logTI;
  const int64_t ntiles = ((g.active_outer + LO - 1) >> logLO) * tchunks;
  const int tile_words = N << (logTI + logLO);
  const int pairs = tile_words >> 1;
  const uint32_t p = m.p;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t oc0 = (tile / tchunks) << logLO;
    const int64_t t0 = (tile - (tile / tchunks) * tchunks) << logTI;
    if (threadIdx.x < LO) {
      const int64_t oc = oc0 + threadIdx.x;
      line_base[threadIdx.x] = oc < g.active_outer ? outer_offset(oc, g) * (int64_t)N * g.inner + t0 : -1;
    }
    __syncthreads();
    // load (bit-reversed rows)
    for (int w = threadIdx.x; w < tile_words; w += blockDim.x) {
      const int t = w & (TI - 1);
      const int n = (w >> logTI) & (N - 1);
      const int lo = w >> (logTI + logN);
      const int64_t base = line_base[lo];
      uint32_t v = 0;
      if (base >= 0 && t0 + t < g.inner) v = data[base + (int64_t)n * g.inner + t];
      sm[(((lo << logN) + bitrev(n, logN)) << logTI) + t] = v;
    }
    __syncthreads();
    for (int lh = 0; lh < logN; ++lh) {
      const int h = 1 << lh;
      const int lstride = logN - 1 - lh;   // twiddle index q * N / (2h)
      for (int w = threadIdx.x; w < pairs; w += blockDim.x) {
        const int t = w & (TI - 1);
        const int j = (w >> logTI) & ((N >> 1) - 1);
        const int lo = w >> (logTI + logN - 1);
        const int q = j & (h - 1);
        const int a = ((j - q) << 1) + q;
        const int ia = (((lo << logN) + a) << logTI) + t;
        const int ib = ia + (h << logTI);
        const uint32_t u = sm[ia];
        const uint32_t x = sm[ib];
        const uint32_t v = shoup_mul(x, __ldg(tw + (q << lstride)), __ldg(tws + (q << lstride)), p);
        sm[ia] = add_mod(u, v, p);
        sm[ib] = sub_mod(u, v, p);
      }
      __syncthreads();
    }
    for (int w = threadIdx.x; w < tile_words; w += blockDim.x) {
      const int t = w & (TI - 1);
      const int n = (w >> logTI) & (N - 1);
      const int lo = w >> (logTI + logN);
      const int64_t base = line_base[lo];
      if (base >= 0 && t0 + t < g.inner) {
        uint32_t v = sm[(((lo << logN) + n) << logTI) + t];
        if (INV && N > 1) v = shoup_mul(v, ninv, ninvs, p);
        data[base + (int64_t)n * g.inner + t] = v;
      }
    }
    __syncthreads();
  }
}

// ---- register-radix axis transform (N = R1 * R2 <= 256) --------------------
// Four-step decomposition n = R2 n1 + n2, k = k1 + R1 k2:
//   X[k1 + R1 k2] = sum_{n2} w_R2^(n2 k2) [ w_N^(n2 k1) sum_{n1} x[R2 n1 + n2] w_R1^(n1 k1) ].
// The tile (LO lines x TI inner columns, 16-byte global loads) is staged in
// shared memory once; pass 1 runs R2 DFT-R1s per line-column in registers and
// writes the twiddled results back to the slots it read, pass 2 runs R1
// DFT-R2s in registers and stores the outputs straight to global memory (N^-1
// fused for the inverse).  Two shared-memory round trips and two barriers per
// tile instead of log2(N) (ntt_axis_smem); twiddles are per-thread registers
// (w_R1, w_R2 powers) plus one table load per twiddled element.  Shared layout
// for TI = 1 (contiguous lines): one pad word per R2 words and a line stride
// of 16 (mod 32) words, so both passes read conflict-free.

#ifndef PDB_RR_MINB1
#define PDB_RR_MINB1 3  // contiguous-line tiles (TIC = 1): 80 registers, no spills
#endif
#ifndef PDB_RR_MINB
#define PDB_RR_MINB 4   // resident 256-thread CTAs per SM the register budget is sized for (4: 64 registers, measured best)
#endif

// X[k] = sum_n x[n] om^(nk), R-point radix-2 DIT in registers; tw[m] = om^m.
template <int R>
__device__ __forceinline__ void dft_reg(uint32_t (&x)[R], const uint32_t* tw, const uint32_t* tws, uint32_t p) {
  constexpr int LR = R == 1 ? 0 : (R == 2 ? 1 : (R == 4 ? 2 : (R == 8 ? 3 : 4)));
  uint32_t y[R];
#pragma unroll
  for (int i = 0; i < R; ++i) y[LR ? (int)(__brev((unsigned)i) >> (32 - LR)) : 0] = x[i];
#pragma unroll
  for (int h = 1; h < R; h <<= 1) {
#pragma unroll
    for (int j = 0; j < R; j += 2 * h) {
#pragma unroll
      for (int q = 0; q < h; ++q) {
        const int m = q * (R / (2 * h));
        const uint32_t u = y[j + q];
        const uint32_t v = m ? shoup_mul(y[j + q + h], tw[m], tws[m], p) : y[j + q + h];
        y[j + q] = add_mod(u, v, p);
        y[j + q + h] = sub_mod(u, v, p);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) x[i] = y[i];
}

// shared-memory slot of (line lo, axis index n, column t); LS = words per line.
// TI = 1: one pad word per R2 words (pass 2 reads R2 consecutive slots per
// thread).  1 < TI < 32: 16 pad words per R2 rows, so the two k1 (or n2) rows
// a warp touches in one instruction fall in opposite bank halves.
template <int R2>
__device__ __forceinline__ int rr_pos(int lo, int n, int t, int TI, int LS) {
  return TI == 1 ? lo * LS + n + n / R2 : lo * LS + n * TI + t + (TI < 32 ? (n / R2) * 16 : 0);
}

// TIC: compile-time tile width (1 = contiguous lines, 32 = 128-byte rows; 0 =
// runtime), so every shared-memory slot of a thread's R-element column folds
// into a base register plus immediate offsets.
template <bool INV, int R1, int R2, int TIC = 0>
__global__ void __launch_bounds__(256, TIC == 1 ? PDB_RR_MINB1 : PDB_RR_MINB)
ntt_axis_rr(uint32_t* __restrict__ data, AxisGeom g, int logTI_rt, int logLO, int LS,
            const uint32_t* __restrict__ full, const uint32_t* __restrict__ fulls,
            const uint32_t* __restrict__ invn, const uint32_t* __restrict__ invns, uint32_t p) {
  constexpr int N = R1 * R2;
  extern __shared__ __align__(16) uint32_t sm[];
  // twiddle table of the pass-1 factors (and the DFT constants) for this direction:
  // tw[e] = w_N^(+-e), e < N; the inverse folds N^-1 into every pass-1 factor
  __shared__ uint32_t tw[N], tws[N];
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const int ee = INV ? (N - e) & (N - 1) : e;
    uint32_t v = __ldg(full + ee), vs = __ldg(fulls + ee);
    tw[e] = v;
    tws[e] = vs;
  }
  // the inverse's N^-1 rides on the pass-1 factors: a separate scaled table
  __shared__ uint32_t twn[INV ? N : 1], twns[INV ? N : 1];
  if constexpr (INV) {
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
      twn[e] = __ldg(invn + e);
      twns[e] = __ldg(invns + e);
    }
  }
  const int logTI = TIC == 1 ? 0 : (TIC == 32 ? 5 : logTI_rt);
  const int TI = 1 << logTI, LO = 1 << logLO;
  const int64_t tchunks = (g.inner + TI - 1) >> logTI;
  const int64_t ntiles = ((g.active_outer + LO - 1) >> logLO) * tchunks;
  const int cols = LO * TI;            // line-columns per tile
  constexpr int LOGN = R1 * R2 == 1 ? 0 : __builtin_ctz(R1 * R2);
  __shared__ int64_t line_base[64];
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t oc0 = (tile / tchunks) << logLO;
    const int64_t t0 = (tile - (tile / tchunks) * tchunks) << logTI;
    if (threadIdx.x < LO) {
      const int64_t oc = oc0 + threadIdx.x;
      line_base[threadIdx.x] = oc < g.active_outer ? outer_offset(oc, g) * (int64_t)N * g.inner + t0 : -1;
    }
    __syncthreads();
    // load: 16-byte vectors along the contiguous direction (t, or n when TI = 1)
    if (TI >= 4 && (g.inner & 3) == 0) {
      for (int w = threadIdx.x; w < (N << (logTI + logLO)) / 4; w += blockDim.x) {
        const int t = (w << 2) & (TI - 1);
        const int n = ((w << 2) >> logTI) & (N - 1);
        const int lo = (w << 2) >> (logTI + LOGN);
        const int64_t base = line_base[lo];
        uint4 v = make_uint4(0, 0, 0, 0);
        if (base >= 0 && t0 + t < g.inner) v = *reinterpret_cast<const uint4*>(data + base + (int64_t)n * g.inner + t);
        *reinterpret_cast<uint4*>(sm + rr_pos<R2>(lo, n, t, TI, LS)) = v;
      }
    } else if (TI == 1 && g.inner == 1 && N >= 4) {
      for (int w = threadIdx.x; w < (N << logLO) / 4; w += blockDim.x) {
        const int n = (w << 2) & (N - 1);
        const int lo = (w << 2) >> LOGN;
        const int64_t base = line_base[lo];
        uint4 v = make_uint4(0, 0, 0, 0);
        if (base >= 0) v = *reinterpret_cast<const uint4*>(data + base + n);
        sm[rr_pos<R2>(lo, n, 0, 1, LS)] = v.x;
        sm[rr_pos<R2>(lo, n + 1, 0, 1, LS)] = v.y;
        sm[rr_pos<R2>(lo, n + 2, 0, 1, LS)] = v.z;
        sm[rr_pos<R2>(lo, n + 3, 0, 1, LS)] = v.w;
      }
    } else {
      for (int w = threadIdx.x; w < (N << (logTI + logLO)); w += blockDim.x) {
        const int t = w & (TI - 1);
        const int n = (w >> logTI) & (N - 1);
        const int lo = w >> (logTI + LOGN);
        const int64_t base = line_base[lo];
        uint32_t v = 0;
        if (base >= 0 && t0 + t < g.inner) v = data[base + (int64_t)n * g.inner + t];
        sm[rr_pos<R2>(lo, n, t, TI, LS)] = v;
      }
    }
    __syncthreads();
    // pass 1: item = (line-column c, n2); DFT-R1 over n1, twiddle w_N^(n2 k1), back in place
    for (int it = threadIdx.x; it < cols * R2; it += blockDim.x) {
      // TI = 1: n2 fastest (consecutive slots of a line); else the column t fastest
      const int c = TI == 1 ? it / R2 : it % cols, n2 = TI == 1 ? it % R2 : it / cols;
      const int t = c & (TI - 1), lo = c >> logTI;
      uint32_t x[R1];
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) x[n1] = sm[rr_pos<R2>(lo, R2 * n1 + n2, t, TI, LS)];
      {
        uint32_t c1[R1 > 1 ? R1 / 2 : 1], c1s[R1 > 1 ? R1 / 2 : 1];
#pragma unroll
        for (int m = 0; m < R1 / 2; ++m) { c1[m] = tw[m * R2]; c1s[m] = tws[m * R2]; }
        dft_reg<R1>(x, c1, c1s, p);
      }
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) {
        const int e = (n2 * k1) & (N - 1);
        if constexpr (INV) x[k1] = shoup_mul(x[k1], twn[e], twns[e], p);
        else if (k1 && n2) x[k1] = shoup_mul(x[k1], tw[e], tws[e], p);
      }
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) sm[rr_pos<R2>(lo, R2 * k1 + n2, t, TI, LS)] = x[k1];
    }
    __syncthreads();
    // pass 2: item = (line-column c, k1); DFT-R2 over n2 -> outputs k1 + R1 k2, straight to HBM
    for (int it = threadIdx.x; it < cols * R1; it += blockDim.x) {
      const int c = TI == 1 ? it / R1 : it % cols, k1 = TI == 1 ? it % R1 : it / cols;
      const int t = c & (TI - 1), lo = c >> logTI;
      uint32_t y[R2];
#pragma unroll
      for (int n2 = 0; n2 < R2; ++n2) y[n2] = sm[rr_pos<R2>(lo, R2 * k1 + n2, t, TI, LS)];
      if constexpr (R2 > 1) {
        uint32_t c2[R2 / 2], c2s[R2 / 2];
#pragma unroll
        for (int m = 0; m < R2 / 2; ++m) { c2[m] = tw[m * R1]; c2s[m] = tws[m * R1]; }
        dft_reg<R2>(y, c2, c2s, p);
      }
      const int64_t base = line_base[lo];
      if (base >= 0 && t0 + t < g.inner) {
        uint32_t* dst = data + base + (int64_t)k1 * g.inner + t;
        const int64_t step = (int64_t)R1 * g.inner;
#pragma unroll
        for (int k2 = 0; k2 < R2; ++k2, dst += step) *dst = y[k2];
      }
    }
    __syncthreads();
  }
}

// ---- global-memory fallback for very long axes (N > PDB_SMEM_NTT_MAX) -------
__global__ void ntt_bitrev_global(uint32_t* __restrict__ data, AxisGeom g, int N, int logN) {
  const int64_t lines = g.active_outer * g.inner;
  const int64_t total = lines * (int64_t)N;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    int64_t line = w / N;
    int n = (int)(w % N);
    int rn = (int)bitrev((uint32_t)n, logN);
    if (rn <= n) continue;
    int64_t oc = line / g.inner, t = line % g.inner;
    int64_t base = outer_offset(oc, g) * (int64_t)N * g.inner + t;
    uint32_t a = data[base + (int64_t)n * g.inner];
    uint32_t b = data[base + (int64_t)rn * g.inner];
    data[base + (int64_t)n * g.inner] = b;
    data[base + (int64_t)rn * g.inner] = a;
  }
}

__global__ void ntt_stage_global(uint32_t* __restrict__ data, AxisGeom g, int N, int h,
                                 const uint32_t* __restrict__ tw, const uint32_t* __restrict__ tws,
                                 Mod32 m, int last, int inv, uint32_t ninv, uint32_t ninvs) {
  const int64_t lines = g.active_outer * g.inner;
  const int64_t total = lines * (int64_t)(N / 2);
  const int stride = N / (2 * h);
  const uint32_t p = m.p;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    int64_t line = w / (N / 2);
    int j = (int)(w % (N / 2));
    int64_t oc = line / g.inner, t = line % g.inner;
    int64_t base = outer_offset(oc, g) * (int64_t)N * g.inner + t;
    int q = j & (h - 1);
    int a = ((j - q) << 1) + q;
    int64_t ia = base + (int64_t)a * g.inner, ib = ia + (int64_t)h * g.inner;
    uint32_t u = data[ia], x = data[ib];
    uint32_t v = shoup_mul(x, tw[q * stride], tws[q * stride], p);
    uint32_t ra = add_mod(u, v, p), rb = sub_mod(u, v, p);
    if (last && inv) {
      ra = shoup_mul(ra, ninv, ninvs, p);
      rb = shoup_mul(rb, ninv, ninvs, p);
    }
    data[ia] = ra;
    data[ib] = rb;
  }
}

// ---- sparse forward axis: input nonzero only on rows j < E <= 8 ------------
// out[k] = sum_{j<E} x_j w^(jk) for every k = u + (N/8) v: each thread owns V
// consecutive inner columns (V = 4: 16-byte loads of the E input rows and
// 16-byte stores of the outputs) and evaluates 8 outputs per column and u by
// a twisted 8-point DFT.  Reads E/N of the axis instead of all of it and does
// ~(E + 4)/8 mul-mods per output instead of log2(N)/2.  The entries'
// coefficient boxes make this the common case of forward passes.  A CTA's
// threads split the N/8 values of u of one tile of TI columns; the E rows are
// read before any output of the tile is written (all writers of rows < E of
// these columns are in this CTA, __syncthreads in between).
// Pruned node sets (executor.kept_u): ukeep > 0 computes only the outputs
// u + (N/8) v with u < ukeep; tiles whose first inner index (the next axis,
// already evaluated, stride kdiv words) is not a kept node of that axis
// (u' = index mod kn8 >= ku) are skipped -- no determinant reads them.
template <int E, int V>
__global__ void __launch_bounds__(256)
ntt_axis_sparse(uint32_t* __restrict__ data, AxisGeom g, int N, int TI, const uint32_t* __restrict__ full,
                const uint32_t* __restrict__ fulls, uint32_t p, int ukeep, int64_t kdiv, int kn8, int ku) {
  const int N8 = ukeep > 0 ? ukeep : N / 8;
  const int64_t tchunks = (g.inner + TI - 1) / TI;
  const int64_t ntiles = g.active_outer * tchunks;
  uint32_t w[4], ws[4];
  w[0] = ws[0] = 0;
#pragma unroll
  for (int v = 1; v < 4; ++v) { w[v] = __ldg(full + v * (N / 8)); ws[v] = __ldg(fulls + v * (N / 8)); }
  const int cols = TI / V;                       // column groups per tile
  const int cg = threadIdx.x % cols;
  const int ug = threadIdx.x / cols, ugs = blockDim.x / cols;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t oc = tile / tchunks;
    const int64_t t0 = (tile - oc * tchunks) * TI + (int64_t)cg * V;
    if (ku > 0 && (int)((((tile - oc * tchunks) * TI) / kdiv) % kn8) >= ku) continue;   // uniform per tile
    const int64_t base = outer_offset(oc, g) * (int64_t)N * g.inner + t0;
    const bool live = t0 < g.inner && ug < ugs;   // V | inner on the vector path
    uint32_t c[V][E];
    if (live) {
#pragma unroll
      for (int j = 0; j < E; ++j) {
        if constexpr (V == 4) {
          const uint4 q = *reinterpret_cast<const uint4*>(data + base + (int64_t)j * g.inner);
          c[0][j] = q.x; c[1][j] = q.y; c[2][j] = q.z; c[3][j] = q.w;
        } else {
          c[0][j] = data[base + (int64_t)j * g.inner];
        }
      }
    }
    __syncthreads();   // every read of rows < E precedes every write
    if (live) {
      for (int u = ug; u < N8; u += ugs) {
        uint32_t tw[8], tws[8];
        int kk = 0;
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          if (l < E) { tw[l] = __ldg(full + kk); tws[l] = __ldg(fulls + kk); }
          else { tw[l] = tws[l] = 0; }
          kk += u;
        }
        uint32_t x[V][8];
#pragma unroll
        for (int q = 0; q < V; ++q) gj_dft8<E>(c[q], tw, tws, w, ws, p, x[q]);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          uint32_t* o = data + base + (int64_t)(u + v * (N / 8)) * g.inner;
          if constexpr (V == 4) *reinterpret_cast<uint4*>(o) = make_uint4(x[0][v], x[1][v], x[2][v], x[3][v]);
          else *o = x[0][v];
        }
      }
    }
    __syncthreads();
  }
}

// Transform one axis of `batch` tensors of shape dims[0..nd) in place.
// ext (may be null) gives, per dim, how many leading indices can be nonzero
// on the dims before `axis` (lines outside that box are skipped).
int ntt_axis(PrimeCtx* ctx, uint32_t* data, int64_t batch, int nd, const int64_t* dims,
             const int64_t* ext, int axis, bool inverse, cudaStream_t st, const int64_t* kept) {
  const int N = (int)dims[axis];
  if (N == 1) return 0;  // length-1 transform is the identity (inverse scale 1)
  const Twiddles* T = ctx_twiddles(ctx, N);
  if (!T) return -1;
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
  const int64_t E = ext ? ext[axis] : N;
  if (!inverse && E >= 1 && E <= 8 && N >= 16 && !getenv("PDB_NTT_DENSE")) {
    // the input is nonzero only on rows < E of this axis: evaluate, don't transform.
    // Tiles of TI inner columns, V = 4 columns per thread when the rows allow 16-byte access.
    const bool vec = g.inner % 4 == 0 && (reinterpret_cast<uintptr_t>(data) & 15) == 0;
    const int V = vec ? 4 : 1;
    int TI = (int)(g.inner < 32 * V ? g.inner : 32 * V);
    if (vec) TI &= ~3;
    const int cols = TI / V;
    int ugs = 256 / cols;                       // u-groups per CTA: at most N/8
    if (ugs > N / 8) ugs = N / 8;
    const int threads = ugs * cols;
    const int64_t tiles = g.active_outer * ((g.inner + TI - 1) / TI);
    const int grid = (int)(tiles < (int64_t)ctx->sms * 16 ? tiles : (int64_t)ctx->sms * 16);
    const uint32_t p = (uint32_t)ctx->p;
    // kept node sets: outputs u < kept[axis]; tiles of non-kept next-axis nodes skipped
    const int ukeep = kept && kept[axis] > 0 ? (int)kept[axis] : 0;
    int64_t kdiv = 1;
    int kn8 = 1, ku = 0;
    if (kept && axis + 1 < nd && kept[axis + 1] > 0 && dims[axis + 1] >= 16) {
      for (int d = axis + 2; d < nd; ++d) kdiv *= dims[d];
      kn8 = (int)(dims[axis + 1] / 8);
      ku = (int)kept[axis + 1];
      if (kdiv % TI) ku = 0;   // a tile must not straddle two next-axis nodes
    }
    switch (E * 2 + (vec ? 1 : 0)) {
#define PDB_SPARSE(EE)                                                                                        \
  case EE * 2: ntt_axis_sparse<EE, 1><<<grid, threads, 0, st>>>(data, g, N, TI, T->full, T->full_s, p, ukeep, kdiv, kn8, ku); break; \
  case EE * 2 + 1: ntt_axis_sparse<EE, 4><<<grid, threads, 0, st>>>(data, g, N, TI, T->full, T->full_s, p, ukeep, kdiv, kn8, ku); break;
      PDB_SPARSE(1) PDB_SPARSE(2) PDB_SPARSE(3) PDB_SPARSE(4)
      PDB_SPARSE(5) PDB_SPARSE(6) PDB_SPARSE(7) PDB_SPARSE(8)
#undef PDB_SPARSE
      default: break;
    }
    count_launch();
    return check_launch("ntt_axis_sparse");
  }
  const uint32_t* tw = inverse ? T->inv : T->fwd;
  const uint32_t* tws = inverse ? T->inv_s : T->fwd_s;
  if (N >= 2 && N <= 256 && !getenv("PDB_NTT_RADIX2")) {
    // register-radix kernel: N = R1 * R2 (R1 = min(N, 16)); tiles of ~4096 words
    // tiles of ~4096-8192 words: up to 32 inner columns (128-byte rows), lines to fill
    int logTI = 0;
    while (logTI < 5 && ((int64_t)2 << logTI) <= g.inner) ++logTI;
    int logLO = 0;
    while (logLO < 6 && ((int64_t)N << (logTI + logLO + 1)) <= 4096 && ((int64_t)2 << logLO) <= g.active_outer)
      ++logLO;
    const int R1 = N < 16 ? N : 16, R2 = N / R1;
    int LS;       // words per line in shared memory (rr_pos)
    if (logTI == 0) {
      LS = N + N / R2;
      LS += ((16 - LS % 32) + 32) % 32;   // consecutive lines in opposite bank halves
    } else {
      LS = (N << logTI) + (logTI < 5 ? (N / R2) * 16 : 0);
    }
    const int64_t tiles = ((g.active_outer + (1 << logLO) - 1) >> logLO) * ((g.inner + (1 << logTI) - 1) >> logTI);
    const size_t smem = sizeof(uint32_t) * ((size_t)LS << logLO);
    int grid = (int)(tiles < (int64_t)ctx->sms * 16 ? tiles : (int64_t)ctx->sms * 16);
    const uint32_t* full = T->full;
    const uint32_t* fulls = T->full_s;
    const uint32_t p = (uint32_t)ctx->p;
#define PDB_RR_T(A, B, C)                                                                                          \
  if (inverse)                                                                                                    \
    ntt_axis_rr<true, A, B, C><<<grid, 256, smem, st>>>(data, g, logTI, logLO, LS, full, fulls, T->inv_full_n,   \
                                                        T->inv_full_ns, p);                                      \
  else                                                                                                            \
    ntt_axis_rr<false, A, B, C><<<grid, 256, smem, st>>>(data, g, logTI, logLO, LS, full, fulls, T->inv_full_n,  \
                                                         T->inv_full_ns, p);
#define PDB_RR(A, B)                                                                                             \
  if (R1 == A && R2 == B) { PDB_RR_T(A, B, 0) }
#define PDB_RR3(A, B)                                                                                            \
  if (R1 == A && R2 == B) {                                                                                       \
    if (logTI == 0) { PDB_RR_T(A, B, 1) }                                                                         \
    else if (logTI == 5) { PDB_RR_T(A, B, 32) }                                                                   \
    else { PDB_RR_T(A, B, 0) }                                                                                    \
  }
    PDB_RR(2, 1) PDB_RR(4, 1) PDB_RR(8, 1) PDB_RR(16, 1)
    PDB_RR3(16, 2) PDB_RR3(16, 4) PDB_RR3(16, 8) PDB_RR3(16, 16)
#undef PDB_RR3
#undef PDB_RR
#undef PDB_RR_T
    count_launch();
    return check_launch("ntt_axis_rr");
  }
  if (N <= PDB_SMEM_NTT_MAX) {
    int logTI = 0;   // inner columns per tile: a power of two <= min(inner, 32)
    while (logTI < 5 && (int64_t)2 << logTI <= g.inner && ((int64_t)N << (logTI + 1)) <= PDB_SMEM_NTT_MAX) ++logTI;
    int logLO = 0;   // lines per tile (<= 16): fill ~4096 words
    while (logLO < 4 && ((int64_t)N << (logTI + logLO + 1)) <= 4096 && ((int64_t)2 << logLO) <= g.active_outer)
      ++logLO;
    const int64_t tiles = ((g.active_outer + (1 << logLO) - 1) >> logLO) * ((g.inner + (1 << logTI) - 1) >> logTI);
    const size_t smem = ((size_t)N << (logTI + logLO)) * sizeof(uint32_t);
    int grid = (int)(tiles < (int64_t)ctx->sms * 16 ? tiles : (int64_t)ctx->sms * 16);
    if (inverse)
      ntt_axis_smem<true><<<grid, 256, smem, st>>>(data, g, N, logN, logTI, logLO, tw, tws, T->ninv, T->ninv_s,
                                                    ctx->m);
    else
      ntt_axis_smem<false><<<grid, 256, smem, st>>>(data, g, N, logN, logTI, logLO, tw, tws, T->ninv, T->ninv_s,
                                                     ctx->m);
    count_launch();  // one launch on either branch
  } else {
    const int64_t total = g.active_outer * g.inner * (int64_t)N;
    int grid = (int)((total / 2 + 255) / 256);
    if (grid > ctx->sms * 32) grid = ctx->sms * 32;
    ntt_bitrev_global<<<grid, 256, 0, st>>>(data, g, N, logN);
    for (int h = 1; h < N; h <<= 1)
      ntt_stage_global<<<grid, 256, 0, st>>>(data, g, N, h, tw, tws, ctx->m, h == N / 2, inverse,
                                             T->ninv, T->ninv_s);
    count_launch(1 + logN);
  }
  return check_launch("ntt_axis");
}

}  // namespace pdb
