/*
 * polydet_b200 — C ABI of the B200 modular-determinant hot path.
 *
 * The reference (arXiv 2010.12117, package `polydet`) has no native code and
 * no FFI: its hot path is four numpy functions called from the Python
 * executor.  Each entry point below replaces one of them; the Python package
 * `paper_2010_12117_b200` binds this library with ctypes and keeps the
 * reference's Python signatures on top:
 *
 *   pdb_ntt_multi_u32        <- transform.py:119-159  ntt_forward_multi / ntt_inverse_multi
 *   pdb_reduce_scatter_u32   <- tensor.py:214-237     reduce_mod + pad_to (per entry, per prime)
 *   pdb_det_batch_u32        <- determinant.py:92-133 det_grid (with entry_ids indirection)
 *   pdb_eval_det_fused_u32   <- pipeline.py:349-392   _fft_stage's last axis fused into _det_stage
 *   pdb_crt_mrc_u32          <- crt.py:94-130         combine_tensor (digits + Horner + signed lift)
 *   pdb_prime_ctx_*          <- transform.py:19-72    TwiddleTable (per-prime root tables)
 *
 * Conventions
 *  - Every pointer argument named data/grids/partial/out/residues/limbs/neg/
 *    scratch/mag/pos/entry_ids is a DEVICE pointer owned by the caller; the
 *    library allocates nothing in hot calls (only pdb_prime_ctx_* allocate
 *    their twiddle tables).  `primes` in pdb_crt_mrc_u32 is a HOST array.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream); calls are
 *    stream-ordered and do not synchronise unless stated.
 *  - Return 0 on success, <0 on error; pdb_last_error() gives a thread-local
 *    message.  -2 = invalid argument (maps to ValueError), -1 = CUDA error.
 *  - Residues are u32 in [0, p); this library handles primes p < 2^31
 *    (the reference's default planning range, prime_start = 10^9).
 */
#ifndef POLYDET_B200_H
#define POLYDET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pdb_prime_ctx pdb_prime_ctx;

const char* pdb_last_error(void);
int32_t pdb_version(void);
/* Kernels launched by this library since load (process-wide counter). */
int64_t pdb_launch_count(void);
int32_t pdb_device_sm_count(int32_t device);

/* Prime p = c * 2^q + 1 with omega of exact order 2^q (reference PrimeSpec,
 * modular.py:81-108).  Builds the Shoup/Montgomery constants. */
int32_t pdb_prime_ctx_create(uint64_t p, uint64_t omega, int32_t q, pdb_prime_ctx** out);
int32_t pdb_prime_ctx_destroy(pdb_prime_ctx* ctx);
/* Build (synchronously) the device twiddle tables for transform length n. */
int32_t pdb_prime_ctx_prepare(pdb_prime_ctx* ctx, int64_t n);

/* In-place natural-order NTT of `batch` row-major tensors of shape dims[0..ndim)
 * along every axis whose bit is set in axis_mask (inverse: w^-1 and * N^-1
 * per axis with N > 1).  extents (may be NULL) = per axis, how many leading
 * indices can be nonzero before that axis is transformed: lines outside the
 * box are skipped (they are zero and stay zero).  Axes are processed from the
 * last to the first.  Errors: length not a power of two or above 2^q
 * ("unsupported length"). */
int32_t pdb_ntt_multi_u32(pdb_prime_ctx* ctx, uint32_t* data, int64_t batch, int32_t ndim,
                          const int64_t* dims, const int64_t* extents, uint32_t axis_mask,
                          int32_t inverse, void* stream);

/* Forward transform for a pruned node set (executor.kept_u): as pdb_ntt_multi_u32
 * (forward), except that an axis with kept_u[a] > 0 (N_a >= 16, 8 kept_u[a] < N_a)
 * evaluates only its nodes u + (N_a/8) v, u < kept_u[a], and passes skip the
 * lines of non-kept nodes of the next axis.  Positions of non-kept nodes are
 * left unwritten: only the fused determinant of the kept nodes reads the result. */
int32_t pdb_ntt_forward_kept_u32(pdb_prime_ctx* ctx, uint32_t* data, int64_t batch, int32_t ndim,
                                 const int64_t* dims, const int64_t* extents, const int64_t* kept_u,
                                 uint32_t axis_mask, void* stream);

/* dst[pos[i]] = (sign_i * sum_l mag[i*limbs + l] 2^(32 l)) mod p. */
int32_t pdb_reduce_scatter_u32(pdb_prime_ctx* ctx, const uint32_t* mag, const uint8_t* neg,
                               const int64_t* pos, int64_t count, int32_t limbs, uint32_t* dst,
                               void* stream);

/* det mod p of M(node) for node in [node_lo, node_lo + nodes), where
 * M(node)[i][j] = grids[entry_ids[i*r + j] * grid_stride + node]; out[node - node_lo]. */
size_t pdb_det_scratch_bytes(int32_t r, int64_t nodes);
int32_t pdb_det_batch_u32(pdb_prime_ctx* ctx, const uint32_t* grids, int64_t grid_stride,
                          const int32_t* entry_ids, int32_t r, int64_t node_lo, int64_t nodes,
                          uint32_t* out, void* scratch, size_t scratch_bytes, void* stream);

/* Same, with the entries evaluated on the fly: partial[(o*ncoef + l)*entries + e]
 * holds entry e (of `entries` unique ones) transformed along every axis but the
 * last, l-th coefficient of the last variable; node = o * n_last + c is
 * evaluated at w_{n_last}^c.  (Layout [outer][ncoef][entries]: the entries are
 * innermost so the kernel's fills read coalesced rows.) */
int32_t pdb_eval_det_fused_u32(pdb_prime_ctx* ctx, const uint32_t* partial, int64_t outer,
                               int32_t ncoef, int32_t entries, int32_t n_last, const int32_t* entry_ids, int32_t r,
                               int64_t node_lo, int64_t nodes, uint32_t* out, void* scratch,
                               size_t scratch_bytes, void* stream);

/* ---- pruned node sets (csrc/expand.cu) --------------------
 * det(M) has degree <= D_a in variable a (the plan's degree bound,
 * pipeline.py:184-196), so on an axis of N >= 16 nodes the determinants at the
 * nodes u + (N/8) v with u < U, v < 8 (any U >= floor(D_a/8) + 1) determine
 * the determinant at every node.  A node map names those kept nodes; kernels
 * taking one index the kept nodes of the grid in a compact row-major order
 * (axis a: 8 U_a positions k = v U_a + u, or all N_a when kept_u[a] == 0).
 * ndim == 0 is the identity (every node, natural order). */
#define PDB_MAP_MAX_DIMS 8
typedef struct pdb_node_map {
  int32_t ndim;                          /* grid rank, <= PDB_MAP_MAX_DIMS; 0 = identity */
  int32_t kept_u[PDB_MAP_MAX_DIMS];      /* U_a (2 <= 8 U_a < N_a), or 0 = the whole axis */
  int64_t dims[PDB_MAP_MAX_DIMS];        /* full grid shape (powers of two) */
} pdb_node_map;

/* Number of kept nodes (the compact grid size); <0 on an invalid map. */
int64_t pdb_node_map_size(const pdb_node_map* map);

/* pdb_det_batch_u32 / pdb_eval_det_fused_u32 over the kept nodes of `map`:
 * node_lo / nodes are compact indices and out[i] = det at compact node
 * node_lo + i.  The fused form's map covers the grid outer x n_last. */
int32_t pdb_det_batch_map_u32(pdb_prime_ctx* ctx, const uint32_t* grids, int64_t grid_stride,
                              const int32_t* entry_ids, int32_t r, const pdb_node_map* map,
                              int64_t node_lo, int64_t nodes, uint32_t* out, void* scratch,
                              size_t scratch_bytes, void* stream);
int32_t pdb_eval_det_fused_map_u32(pdb_prime_ctx* ctx, const uint32_t* partial, int64_t outer,
                                   int32_t ncoef, int32_t entries, int32_t n_last,
                                   const int32_t* entry_ids, int32_t r, const pdb_node_map* map,
                                   int64_t node_lo, int64_t nodes, uint32_t* out, void* scratch,
                                   size_t scratch_bytes, void* stream);

/* compact[pdb_node_map_size(map)] determinants at the kept nodes (every axis
 * pruned) -> the polynomial's coefficients c[j_0..j_{d-1}], j_a < box[a] <= 8 kept_u[a],
 * written at their row-major positions of grid[prod dims]; the rest of grid is
 * not written (the inverse NTT of the full determinant grid is zero there by
 * the degree bound, so a zeroed grid then equals reference _ifft_stage,
 * pipeline.py:395-404).  One pass per axis straight from the kept nodes: no
 * full determinant grid, no inverse NTT.  compact is overwritten; scratch holds
 * as many u32 as compact. */
int32_t pdb_grid_interpolate_u32(pdb_prime_ctx* ctx, uint32_t* compact, uint32_t* scratch, uint32_t* grid,
                                 const pdb_node_map* map, const int64_t* box, void* stream);

/* compact[pdb_node_map_size(map)] determinants at the kept nodes -> grid[prod dims]
 * with every node's determinant (the same values det_grid computes there,
 * determinant.py:92-133).  compact and grid must not overlap. */
int32_t pdb_grid_expand_u32(pdb_prime_ctx* ctx, const uint32_t* compact, uint32_t* grid,
                            const pdb_node_map* map, void* stream);

/* Scalar condensation with the reference's pivot trail (determinant.py:57-84):
 * mat = r*r row-major residues (device); trail_vals[i]/trail_cols[i] = pivot of
 * step i (cols = -1 after an all-zero row); det_out[0] = det.  Scratch needs
 * 4 r^2 + 256 + 512 r^2 bytes. */
int32_t pdb_condense_u32(pdb_prime_ctx* ctx, const uint32_t* mat, int32_t r, uint32_t* trail_vals,
                         int32_t* trail_cols, uint32_t* det_out, void* scratch, size_t scratch_bytes,
                         void* stream);

/* Mixed-radix CRT over nprimes residue rows residues[i*stride + pos], pos < n.
 * limbs[pos*L + l] = |X| little-endian, neg[pos] = X < 0, X in (-P/2, P/2]. */
int32_t pdb_crt_limbs(int32_t nprimes);
size_t pdb_crt_scratch_bytes(int32_t nprimes);
int32_t pdb_crt_mrc_u32(const uint32_t* residues, int32_t nprimes, int64_t n, int64_t stride,
                        const uint32_t* primes, uint32_t* limbs, int32_t L, uint8_t* neg,
                        void* scratch, size_t scratch_bytes, void* stream);

/* Positions whose coefficient is nonzero, i.e. some residue is nonzero
 * (0 <= X < P): index[0..*count) ascending (index has room for n entries;
 * count is a DEVICE int64).  Replaces the reference's zero test of
 * CoeffTensor.terms() (tensor.py:101-107) before the lift. */
size_t pdb_crt_nonzero_scratch_bytes(int64_t n);
int32_t pdb_crt_nonzero_u32(const uint32_t* residues, int32_t nprimes, int64_t n, int64_t stride,
                            int64_t* index, int64_t* count, void* scratch, size_t scratch_bytes,
                            void* stream);
/* pdb_crt_mrc_u32 at the positions index[0..count) (NULL: 0..count-1), compact
 * output limbs[i*L + l], neg[i]; *width (DEVICE int32, may be NULL) = the most
 * limbs any of these coefficients uses.  No host synchronisation. */
int32_t pdb_crt_mrc_sel_u32(const uint32_t* residues, int32_t nprimes, int64_t stride,
                            const uint32_t* primes, const int64_t* index, int64_t count, uint32_t* limbs,
                            int32_t L, uint8_t* neg, int32_t* width, void* stream);

/* Result materialisation (reference crt.py:122-130 builds Python ints): the
 * |X| limb rows [count][width] (row stride `stride` u32) re-cut into CPython's
 * 30-bit digits [count][ndigits] (ndigits >= ceil(32 width / 30), <= 255) plus
 * the significant digit count per row, on the device; the host then makes each
 * int with one allocation and one copy.  No host synchronisation. */
int32_t pdb_limbs_to_digits30(const uint32_t* limbs, int64_t count, int32_t width, int64_t stride,
                              uint32_t* digits, int32_t ndigits, uint8_t* digit_count, void* stream);

/* Integer-pipe peak of an update primitive (no memory traffic), in updates/s.
 * variant 0 = Shoup mul-mod + sub-mod, 1 = delayed 64-bit MAC (9 MACs + one REDC,
 * the det kernel's trailing update: updates = MACs), 2 = raw accumulating
 * IMAD.WIDE stream (the integer multiplier's ceiling, MACs/s). */
int32_t pdb_mulmod_peak(uint32_t p, int32_t variant, double* updates_per_second, void* stream);

/* Profiling hook (no reference counterpart): while enabled, every det_gj kernel
 * launch is bracketed by CUDA events on its launch stream.  pdb_kernel_timing
 * enables (1) or disables (0) it and clears the record; pdb_kernel_timing_read
 * waits for the recorded launches and returns their summed device time. */
int32_t pdb_kernel_timing(int32_t enable);
int32_t pdb_kernel_timing_read(double* ms, int64_t* launches);

/* ---- the wide path: primes 2^31 <= p < 2^62 --------------
 * u64 twins of the entry points above for contexts created with p >= 2^31
 * (reference object/int64 dtype paths, tensor.py:152-154).  Residues are u64;
 * the CRT takes any mix of odd primes < 2^62 (test_crt.py:147-153).  The u32
 * entry points reject wide contexts and vice versa. */
int32_t pdb_prime_ctx_create_wide(uint64_t p, uint64_t omega, int32_t q, pdb_prime_ctx** out);
int32_t pdb_ntt_multi_u64(pdb_prime_ctx* ctx, uint64_t* data, int64_t batch, int32_t ndim,
                          const int64_t* dims, const int64_t* extents, uint32_t axis_mask,
                          int32_t inverse, void* stream);
int32_t pdb_reduce_scatter_u64(pdb_prime_ctx* ctx, const uint32_t* mag, const uint8_t* neg,
                               const int64_t* pos, int64_t count, int32_t limbs, uint64_t* dst,
                               void* stream);
size_t pdb_det_scratch_bytes_u64(int32_t r, int64_t nodes);
int32_t pdb_det_batch_u64(pdb_prime_ctx* ctx, const uint64_t* grids, int64_t grid_stride,
                          const int32_t* entry_ids, int32_t r, int64_t node_lo, int64_t nodes,
                          uint64_t* out, void* scratch, size_t scratch_bytes, void* stream);
int32_t pdb_condense_u64(pdb_prime_ctx* ctx, const uint64_t* mat, int32_t r, uint64_t* trail_vals,
                         int32_t* trail_cols, uint64_t* det_out, void* scratch, size_t scratch_bytes,
                         void* stream);
int32_t pdb_crt_limbs_u64(int32_t nprimes);
size_t pdb_crt_scratch_bytes_u64(int32_t nprimes);
int32_t pdb_crt_mrc_u64(const uint64_t* residues, int32_t nprimes, int64_t n, int64_t stride,
                        const uint64_t* primes, uint32_t* limbs, int32_t L, uint8_t* neg,
                        void* scratch, size_t scratch_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* POLYDET_B200_H */
