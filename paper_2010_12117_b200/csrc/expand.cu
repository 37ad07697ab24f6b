// Determinants at the pruned node set -> the full evaluation grid.
//
// The reference evaluates det(M) at every node of the grid (pipeline.py:374-392)
// and interpolates with a full inverse NTT.  The determinant has degree <= D_a
// in variable a (pipeline.py:184-196), and on an axis of N nodes
//     f(x) = sum_{l<8} x^l g_l(x^8),   deg g_l <= floor(D_a / 8) < U,
// so the values of f at the nodes u + (N/8) v with u < U (v < 8) fix every g_l
// at the first U of the N/8 points y_u = w^(8u) -- hence f at every node.
// Per line, with z_l(u) = (1/8) sum_v f(w^(u + N/8 v)) w8^(-lv) = w^(ul) g_l(y_u):
//     y_l(u') = sum_{u<U} w^(l(u'-u)) L_u(y_u') z_l(u),   u' = U .. N/8-1
//     f(w^(u' + N/8 v)) = sum_l y_l(u') w8^(lv),
// L_u the Lagrange basis on y_0..y_{U-1}.  The extended values are exactly
// the determinants the reference computes at those nodes (the polynomial
// identity holds mod p), so the grid -- and every artifact built from it --
// is bit-identical; only ~prod_a 8 U_a / N_a of the determinants are computed
// (C5: 176^3 of 256^3 = 33 %).
//
// grid_expand: scatter the compact determinants into the grid, then extend
// along each pruned axis from the last to the first; the lines of axis a run
// over the kept nodes of the axes before it and every node of the axes after.
#include <map>
#include <vector>

#include "pdb_internal.cuh"

namespace pdb {

struct ExpandTables {
  int N = 0, U = 0;
  uint32_t* dev = nullptr;   // [64] iDFT-8 (incl. 1/8), [64] DFT-8, [8][N/8-U][U] extension; Montgomery forms
};

static std::mutex g_xlock;
static std::map<std::tuple<const PrimeCtx*, int, int>, ExpandTables> g_tables;
// direct-interpolation tables per (prime, N, U, B) (grid_interpolate, below)
struct InterpTables {
  uint32_t* dev = nullptr;
};
static std::map<std::tuple<const PrimeCtx*, int, int, int>, InterpTables> g_itables;

static uint64_t mulm(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)((unsigned __int128)a * b % p); }
static uint64_t powm(uint64_t a, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  a %= p;
  for (; e; e >>= 1, a = mulm(a, a, p))
    if (e & 1) r = mulm(r, a, p);
  return r;
}

static const ExpandTables* expand_tables(PrimeCtx* ctx, int N, int U) {
  std::lock_guard<std::mutex> guard(g_xlock);
  auto key = std::make_tuple((const PrimeCtx*)ctx, N, U);
  auto it = g_tables.find(key);
  if (it != g_tables.end()) return &it->second;
  const uint64_t p = ctx->p;
  const int l = 31 - __builtin_clz((unsigned)N);
  const uint64_t w = powm(ctx->omega, 1ull << (ctx->q - l), p);   // w_N
  const uint64_t w8 = powm(w, N / 8, p), w8i = powm(w8, p - 2, p);
  const uint64_t inv8 = powm(8, p - 2, p);
  const uint64_t R = ((uint64_t)1 << 32) % p;
  const int N8 = N / 8, T = N8 - U;
  std::vector<uint32_t> h(128 + (size_t)8 * T * U);
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      h[a * 8 + b] = (uint32_t)mulm(mulm(powm(w8i, (uint64_t)a * b, p), inv8, p), R, p);   // [l][v]
      h[64 + a * 8 + b] = (uint32_t)mulm(powm(w8, (uint64_t)a * b, p), R, p);             // [v][l]
    }
  // Lagrange basis on y_u = w^(8u), u < U, evaluated at y_u', u' = U..N8-1
  std::vector<uint64_t> wp(N), y(N8), bw(U);
  wp[0] = 1 % p;
  for (int j = 1; j < N; ++j) wp[j] = mulm(wp[j - 1], w, p);
  for (int j = 0; j < N8; ++j) y[j] = wp[8 * j];
  for (int u = 0; u < U; ++u) {
    uint64_t d = 1;
    for (int j = 0; j < U; ++j)
      if (j != u) d = mulm(d, (y[u] + p - y[j]) % p, p);
    bw[u] = powm(d, p - 2, p);   // barycentric weight
  }
  for (int t = 0; t < T; ++t) {
    const uint64_t yt = y[U + t];
    uint64_t ell = 1;
    for (int j = 0; j < U; ++j) ell = mulm(ell, (yt + p - y[j]) % p, p);
    for (int u = 0; u < U; ++u) {
      const uint64_t Lu = mulm(mulm(ell, bw[u], p), powm((yt + p - y[u]) % p, p - 2, p), p);
      for (int ll = 0; ll < 8; ++ll) {
        const uint64_t tw = wp[((uint64_t)ll * (uint64_t)(U + t - u)) % N];
        h[128 + ((size_t)ll * T + t) * U + u] = (uint32_t)mulm(mulm(tw, Lu, p), R, p);
      }
    }
  }
  ExpandTables X;
  X.N = N;
  X.U = U;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaMalloc(&X.dev, h.size() * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemcpy(X.dev, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("expand table allocation: %s", cudaGetErrorString(e));
    return nullptr;
  }
  return &(g_tables[key] = X);
}

void expand_release(const PrimeCtx* ctx) {
  std::lock_guard<std::mutex> guard(g_xlock);
  for (auto it = g_itables.begin(); it != g_itables.end();) {
    if (std::get<0>(it->first) == ctx) {
      cudaFree(it->second.dev);
      it = g_itables.erase(it);
    } else {
      ++it;
    }
  }
  for (auto it = g_tables.begin(); it != g_tables.end();) {
    if (std::get<0>(it->first) == ctx) {
      cudaFree(it->second.dev);
      it = g_tables.erase(it);
    } else {
      ++it;
    }
  }
}

// sum_i a[i] * bR[i] mod p (bR Montgomery forms), canonical; up to 8 products per
// reduction for p < 2^30, 2 otherwise
__device__ __forceinline__ uint32_t dot_mont(const uint32_t* a, int sa, const uint32_t* bR, int n, const Mod32& m) {
  const int cap = m.fast() ? 8 : 2;
  uint32_t s = 0;
  for (int i0 = 0; i0 < n; i0 += cap) {
    uint64_t acc = 0;
    const int i1 = i0 + cap < n ? i0 + cap : n;
    for (int i = i0; i < i1; ++i) acc = mad_wide(a[(size_t)i * sa], __ldg(bR + i), acc);
    s = add_mod(s, canon32(redc(acc, m), m), m.p);
  }
  return s;
}

__global__ void grid_scatter(const uint32_t* __restrict__ compact, uint32_t* __restrict__ grid, int64_t n,
                             NodeMap map) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    grid[map.full(c)] = compact[c];
}

// One CTA per tile of TI columns; column j = (line j / inner, position j % inner);
// a line's element n sits at outer(line) + n * inner + j % inner.
__global__ void __launch_bounds__(256)
grid_extend(uint32_t* __restrict__ grid, NodeMap outer_map, int64_t lines, int64_t inner, int N, int U, int TI,
            const uint32_t* __restrict__ tab, Mod32 m) {
  extern __shared__ uint32_t xs[];
  const int N8 = N / 8, T = N8 - U, K = 8 * U;
  uint32_t* kept = xs;                  // [K][TI]   kept values, row k = v U + u
  uint32_t* zs = kept + K * TI;         // [8][U][TI]
  __shared__ int64_t cbase[32];
  const int64_t cols = lines * inner;
  const int64_t tiles = (cols + TI - 1) / TI;
  const bool rowfast = inner < TI;      // coalesce along the line when lines are short-strided
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t j0 = tile * TI;
    __syncthreads();
    if (threadIdx.x < TI) {
      const int64_t j = j0 + threadIdx.x;
      cbase[threadIdx.x] = j < cols ? outer_map.full(j / inner) * N * inner + j % inner : -1;
    }
    __syncthreads();
    for (int w = threadIdx.x; w < K * TI; w += blockDim.x) {
      const int k = rowfast ? w % K : w / TI, t = rowfast ? w / K : w % TI;
      const int u = k % U, v = k / U;
      const int64_t b = cbase[t];
      kept[k * TI + t] = b >= 0 ? grid[b + (int64_t)(u + N8 * v) * inner] : 0u;
    }
    __syncthreads();
    for (int w = threadIdx.x; w < 8 * U * TI; w += blockDim.x) {   // z_l(u) = iDFT8
      const int t = w % TI, lu = w / TI, l = lu / U, u = lu % U;
      zs[(l * U + u) * TI + t] = dot_mont(kept + u * TI + t, U * TI, tab + l * 8, 8, m);
    }
    __syncthreads();
    for (int w = threadIdx.x; w < T * TI; w += blockDim.x) {
      const int t = rowfast ? w / T : w % TI, tt = rowfast ? w % T : w / TI;
      const int64_t b = cbase[t];
      if (b < 0) continue;
      uint32_t yl[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) yl[l] = dot_mont(zs + (l * U) * TI + t, TI, tab + 128 + ((size_t)l * T + tt) * U, U, m);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        // 8 products: one reduction for p < 2^30, pairs otherwise
        const uint32_t* f = tab + 64 + v * 8;
        uint32_t s = 0;
#pragma unroll
        for (int h = 0; h < 8; h += 2) {
          uint64_t acc = mad_wide(yl[h], __ldg(f + h), mad_wide(yl[h + 1], __ldg(f + h + 1), 0ull));
          if (m.fast()) {
#pragma unroll
            for (int q = h + 2; q < 8; ++q) acc = mad_wide(yl[q], __ldg(f + q), acc);
            s = canon32(redc(acc, m), m);
            break;
          }
          s = add_mod(s, canon32(redc(acc, m), m), m.p);
        }
        grid[b + (int64_t)(U + tt + N8 * v) * inner] = s;
      }
    }
  }
}

// ---- direct interpolation from the kept nodes (no full determinant grid) ----
// With z_l(u) = (1/8) sum_v f(w^(u + N/8 v)) w8^(-lv) = w^(ul) g_l(y_u) (see the
// top of this file), the coefficients of f on an axis are
//     c_(8i + l) = g_(l,i) = sum_{u<U} Vinv[i][u] w^(-ul) z_l(u),   8i + l < B,
// Vinv the inverse of the U x U Vandermonde matrix of y_u = w^(8u).  One pass
// per axis (last to first) over a shrinking box: the axis goes from its 8U
// kept nodes to its B = D_a + 1 coefficients, the coefficients the inverse NTT
// of the extended grid gives there (the rest of that axis is zero by the
// degree bound).  Tables per (prime, N, U, B): [64] iDFT-8 incl. 1/8 (shared
// with the extension), then Q[l][i][u] = Vinv[i][u] w^(-ul), i < ceil(B/8).

static const uint32_t* interp_tables(PrimeCtx* ctx, int N, int U, int B) {
  std::lock_guard<std::mutex> guard(g_xlock);
  auto key = std::make_tuple((const PrimeCtx*)ctx, N, U, B);
  auto it = g_itables.find(key);
  if (it != g_itables.end()) return it->second.dev;
  const uint64_t p = ctx->p;
  const int l2 = 31 - __builtin_clz((unsigned)N);
  const uint64_t w = powm(ctx->omega, 1ull << (ctx->q - l2), p);
  const uint64_t wi = powm(w, p - 2, p);
  const uint64_t w8 = powm(w, N / 8, p), w8i = powm(w8, p - 2, p);
  const uint64_t inv8 = powm(8, p - 2, p);
  const uint64_t R = ((uint64_t)1 << 32) % p;
  const int I = (B + 7) / 8;
  std::vector<uint32_t> h(64 + (size_t)8 * I * U);
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) h[a * 8 + b] = (uint32_t)mulm(mulm(powm(w8i, (uint64_t)a * b, p), inv8, p), R, p);
  // Vinv: row i of the inverse holds the y^i coefficients of the Lagrange basis
  std::vector<uint64_t> y(U);
  for (int u = 0; u < U; ++u) y[u] = powm(w, 8ull * u, p);
  std::vector<uint64_t> vinv((size_t)U * U);
  for (int u = 0; u < U; ++u) {
    std::vector<uint64_t> poly(1, 1);   // prod_{j != u} (Y - y_j), low degree first
    uint64_t den = 1;
    for (int j = 0; j < U; ++j) {
      if (j == u) continue;
      std::vector<uint64_t> nx(poly.size() + 1, 0);
      for (size_t d = 0; d < poly.size(); ++d) {
        nx[d + 1] = (nx[d + 1] + poly[d]) % p;
        nx[d] = (nx[d] + mulm(poly[d], (p - y[j]) % p, p)) % p;
      }
      poly.swap(nx);
      den = mulm(den, (y[u] + p - y[j]) % p, p);
    }
    const uint64_t di = powm(den, p - 2, p);
    for (int i = 0; i < U; ++i) vinv[(size_t)i * U + u] = mulm(poly[i], di, p);
  }
  for (int l = 0; l < 8; ++l)
    for (int i = 0; i < I; ++i)
      for (int u = 0; u < U; ++u) {
        const uint64_t q = mulm(vinv[(size_t)i * U + u], powm(wi, (uint64_t)u * l, p), p);
        h[64 + ((size_t)l * I + i) * U + u] = (uint32_t)mulm(q, R, p);
      }
  InterpTables X;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  cudaError_t e = cudaMalloc(&X.dev, h.size() * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemcpy(X.dev, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("interpolation table allocation: %s", cudaGetErrorString(e));
    return nullptr;
  }
  return (g_itables[key] = X).dev;
}

// Output addressing of one pass: the columns (every index but the axis) are
// the mixed radix over ext[b != a]; ostride[b] the output stride of axis b.
struct InterpGeom {
  int nd, a;
  int64_t ext[PDB_MAP_DIMS];
  int64_t ostride[PDB_MAP_DIMS];
};

// sum_{u<U} a[u] * bR[u] (bR Montgomery forms, a in registers), canonical; at
// most 8 products per reduction for p < 2^30 (9 p^2 < REDC bound), 2 otherwise.
template <int UM>
__device__ __forceinline__ uint32_t dot_reg(const uint32_t (&a)[UM], const uint32_t* bR, int U, const Mod32& m) {
  uint32_t s = 0;
  if (m.fast()) {
#pragma unroll
    for (int g = 0; g < UM; g += 8) {
      if (g >= U) break;
      uint64_t acc = 0;
#pragma unroll
      for (int i = g; i < g + 8 && i < UM; ++i)
        if (i < U) acc = mad_wide(a[i], bR[i], acc);
      s = add_mod(s, canon32(redc(acc, m), m), m.p);
    }
  } else {
#pragma unroll
    for (int i = 0; i < UM; i += 2) {
      if (i >= U) break;
      uint64_t acc = mad_wide(a[i], bR[i], 0ull);
      if (i + 1 < U) acc = mad_wide(a[i + 1], bR[i + 1], acc);
      s = add_mod(s, canon32(redc(acc, m), m), m.p);
    }
  }
  return s;
}

// One CTA per tile of TI columns: kept values [K][TI] -> z [8][U][TI] -> coefficients.
// UM >= U is a compile-time bound: a thread holds one column's 8 values of a u
// (the iDFT-8) or U values of a residue class l (the Vandermonde solve) in
// registers; the tables sit in shared memory and are read as warp broadcasts.
template <int UM>
__global__ void __launch_bounds__(256)
grid_interp(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, InterpGeom gm, int64_t cols, int64_t inner,
            int U, int B, int TI, const uint32_t* __restrict__ tab, Mod32 m) {
  extern __shared__ uint32_t xs[];
  const int K = 8 * U, I = (B + 7) / 8;
  uint32_t* kept = xs;                  // [K][TI]
  uint32_t* zs = kept + K * TI;         // [8][U][TI]
  uint32_t* tq = zs + 8 * U * TI;       // [64] iDFT-8, then Q[8][I][U]
  __shared__ int64_t cin[32], cout_[32];
  for (int w = threadIdx.x; w < 64 + 8 * I * U; w += blockDim.x) tq[w] = __ldg(tab + w);
  const int64_t tiles = (cols + TI - 1) / TI;
  const bool rowfast = inner < TI;
  const uint32_t* Q = tq + 64;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t j0 = tile * TI;
    __syncthreads();
    if (threadIdx.x < TI) {
      const int64_t j = j0 + threadIdx.x;
      if (j < cols) {
        const int64_t o = j / inner, t = j - (j / inner) * inner;
        cin[threadIdx.x] = o * K * inner + t;
        int64_t off = 0, c = j;
        for (int b = gm.nd - 1; b >= 0; --b) {
          if (b == gm.a) continue;
          const int64_t e = gm.ext[b];
          off += (c % e) * gm.ostride[b];
          c /= e;
        }
        cout_[threadIdx.x] = off;
      } else {
        cin[threadIdx.x] = -1;
      }
    }
    __syncthreads();
    for (int w = threadIdx.x; w < K * TI; w += blockDim.x) {
      const int k = rowfast ? w % K : w / TI, t = rowfast ? w / K : w % TI;
      const int64_t b = cin[t];
      kept[k * TI + t] = b >= 0 ? __ldg(in + b + (int64_t)k * inner) : 0u;
    }
    __syncthreads();
    // z_l(u) = iDFT-8 over v (1/8 folded): item (u, t) holds the 8 values of its u
    for (int w = threadIdx.x; w < U * TI; w += blockDim.x) {
      const int t = w % TI, u = w / TI;
      uint32_t x[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) x[v] = kept[(v * U + u) * TI + t];
#pragma unroll
      for (int l = 0; l < 8; ++l) zs[(l * U + u) * TI + t] = dot_reg<8>(x, tq + l * 8, 8, m);
    }
    __syncthreads();
    // coefficients c_(8i + l), 8i + l < B: item (l, t) holds z_l(0..U) of its column
    for (int w = threadIdx.x; w < 8 * TI; w += blockDim.x) {
      const int t = w % TI, l = w / TI;
      if (cin[t] < 0) continue;
      uint32_t z[UM];
#pragma unroll
      for (int u = 0; u < UM; ++u) z[u] = u < U ? zs[(l * U + u) * TI + t] : 0u;
      uint32_t* o = out + cout_[t];
      const int64_t os = gm.ostride[gm.a];
      for (int i = 0; 8 * i + l < B; ++i)
        o[(int64_t)(8 * i + l) * os] = dot_reg<UM>(z, Q + (l * I + i) * U, U, m);
    }
  }
}

// compact determinants (map's kept nodes) -> coefficients c[j_0..j_{d-1}], j_a <
// box[a], written at grid positions sum j_a stride_a of the dims grid; the rest
// of the grid is not touched.  Every axis must be pruned (kept_u > 0).
// scratch: as many words as the compact array; compact is overwritten.
int grid_interpolate(PrimeCtx* ctx, uint32_t* compact, uint32_t* scratch, uint32_t* grid, const NodeMap& map,
                     const int64_t* dims, const int64_t* box, cudaStream_t st) {
  const int nd = map.nd;
  if (nd == 0) { set_error("grid_interpolate needs a pruned node map"); return -2; }
  int64_t ext[PDB_MAP_DIMS], full_stride[PDB_MAP_DIMS];
  for (int a = 0; a < nd; ++a) {
    if (!map.u[a]) { set_error("grid_interpolate: axis %d is not pruned", a); return -2; }
    if (box[a] < 1 || box[a] > 8 * map.u[a]) {
      set_error("grid_interpolate: box %lld on axis %d exceeds 8 U = %d", (long long)box[a], a, 8 * map.u[a]);
      return -2;
    }
    ext[a] = map.klen[a];
  }
  full_stride[nd - 1] = 1;
  for (int a = nd - 2; a >= 0; --a) full_stride[a] = full_stride[a + 1] * dims[a + 1];
  const uint32_t* src = compact;
  for (int a = nd - 1; a >= 0; --a) {
    const int N = (int)dims[a], U = map.u[a], B = (int)box[a];
    const uint32_t* tab = interp_tables(ctx, N, U, B);
    if (!tab) return -1;
    InterpGeom gm;
    gm.nd = nd;
    gm.a = a;
    int64_t cols = 1, inner = 1;
    for (int b = 0; b < nd; ++b) {
      gm.ext[b] = ext[b];
      if (b != a) cols *= ext[b];
      if (b > a) inner *= ext[b];
    }
    const bool last = a == 0;
    uint32_t* dst = last ? grid : (src == compact ? scratch : compact);
    if (last) {
      for (int b = 0; b < nd; ++b) gm.ostride[b] = full_stride[b];
    } else {   // compact output: ext with ext[a] -> B
      int64_t stv = 1;
      for (int b = nd - 1; b >= 0; --b) {
        gm.ostride[b] = stv;
        stv *= (b == a ? B : ext[b]);
      }
    }
    if (U > 32) { set_error("grid_interpolate: kept u %d > 32", U); return -2; }
    int TI = 32;
    const size_t tabw = 64 + (size_t)8 * ((B + 7) / 8) * U;
    while (TI > 1 && ((size_t)(8 * U + 8 * U) * TI + tabw) * 4 > 96 * 1024) TI >>= 1;
    const size_t smem = ((size_t)(8 * U + 8 * U) * TI + tabw) * sizeof(uint32_t);
    const int64_t tiles = (cols + TI - 1) / TI;
    const int g = (int)(tiles < (int64_t)ctx->sms * 8 ? tiles : (int64_t)ctx->sms * 8);
#define PDB_INTERP(UM)                                                                                          \
  {                                                                                                             \
    if (smem > 48 * 1024)                                                                                       \
      cudaFuncSetAttribute(grid_interp<UM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);            \
    grid_interp<UM><<<g, 256, smem, st>>>(src, dst, gm, cols, inner, U, B, TI, tab, ctx->m);                    \
  }
    if (U <= 8) PDB_INTERP(8)
    else if (U <= 16) PDB_INTERP(16)
    else if (U <= 24) PDB_INTERP(24)
    else PDB_INTERP(32)
#undef PDB_INTERP
    count_launch();
    if (int rc = check_launch("grid_interp")) return rc;
    ext[a] = B;
    src = dst;
  }
  return 0;
}

int grid_expand(PrimeCtx* ctx, const uint32_t* compact, uint32_t* grid, const NodeMap& map, const int64_t* dims,
                cudaStream_t st) {
  int64_t n = 1;
  for (int a = 0; a < map.nd; ++a) n *= map.klen[a];
  if (map.nd == 0) {
    set_error("grid_expand needs a pruned node map");
    return -2;
  }
  {
    const int64_t blocks = (n + 255) / 256;
    const int g = (int)(blocks < (int64_t)ctx->sms * 16 ? blocks : (int64_t)ctx->sms * 16);
    grid_scatter<<<g, 256, 0, st>>>(compact, grid, n, map);
    count_launch();
    if (int rc = check_launch("grid_scatter")) return rc;
  }
  for (int a = map.nd - 1; a >= 0; --a) {
    if (!map.u[a]) continue;
    const int N = (int)dims[a], U = map.u[a];
    const ExpandTables* X = expand_tables(ctx, N, U);
    if (!X) return -1;
    NodeMap om = map;            // the axes before a: kept nodes only
    om.nd = a;
    int64_t lines = 1, inner = 1;
    for (int b = 0; b < a; ++b) lines *= map.klen[b];
    for (int b = a + 1; b < map.nd; ++b) inner *= dims[b];
    // om.full(line): the line's row-major index over dims[0..a) (units of N * inner words)
    for (int b = 0; b < a; ++b) om.stride[b] = map.stride[b] / ((int64_t)N * inner);
    int TI = 32;
    while (TI > 1 && (size_t)(8 * U + 8 * U) * TI * 4 > 96 * 1024) TI >>= 1;
    const size_t smem = (size_t)(8 * U + 8 * U) * TI * sizeof(uint32_t);
    const int64_t tiles = (lines * inner + TI - 1) / TI;
    const int g = (int)(tiles < (int64_t)ctx->sms * 8 ? tiles : (int64_t)ctx->sms * 8);
    if (smem > 48 * 1024) cudaFuncSetAttribute(grid_extend, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    grid_extend<<<g, 256, smem, st>>>(grid, om, lines, inner, N, U, TI, X->dev, ctx->m);
    count_launch();
    if (int rc = check_launch("grid_extend")) return rc;
  }
  return 0;
}

}  // namespace pdb
