"""ctypes binding of libpolydet_b200.so (the C ABI in include/polydet_b200.h).

The library is the ONLY compute path of this package: if it is missing, or
no CUDA device is visible, every call raises DeviceError -- there is no CPU
fallback.  torch is used purely for device memory and streams: tensors are
allocated with torch and handed to the kernels as raw pointers.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import DeviceError
from .fields import MODULUS_LIMIT, U32_KERNEL_MODULUS

LIB_NAME = "libpolydet_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME
U32_LIMIT = U32_KERNEL_MODULUS   # u32 kernels: p < 2^31
WIDE_LIMIT = MODULUS_LIMIT       # u64 kernels (the wide path): p < 2^62


def needs_wide(p: int) -> bool:
    return p >= U32_LIMIT

_lib = None
_lock = threading.Lock()

_c_i32, _c_i64, _c_u32, _c_u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
_c_size, _c_vp = ctypes.c_size_t, ctypes.c_void_p

MAP_MAX_DIMS = 8


class NodeMapC(ctypes.Structure):
    """pdb_node_map (include/polydet_b200.h): the kept nodes of a pruned grid."""
    _fields_ = [("ndim", ctypes.c_int32), ("kept_u", ctypes.c_int32 * MAP_MAX_DIMS),
                ("dims", ctypes.c_int64 * MAP_MAX_DIMS)]


_c_map = ctypes.POINTER(NodeMapC)

_SIGNATURES = {
    "pdb_last_error": (ctypes.c_char_p, []),
    "pdb_version": (_c_i32, []),
    "pdb_launch_count": (_c_i64, []),
    "pdb_device_sm_count": (_c_i32, [_c_i32]),
    "pdb_prime_ctx_create": (_c_i32, [_c_u64, _c_u64, _c_i32, ctypes.POINTER(_c_vp)]),
    "pdb_prime_ctx_destroy": (_c_i32, [_c_vp]),
    "pdb_prime_ctx_prepare": (_c_i32, [_c_vp, _c_i64]),
    "pdb_ntt_multi_u32": (_c_i32, [_c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_vp, _c_u32, _c_i32, _c_vp]),
    "pdb_reduce_scatter_u32": (_c_i32, [_c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_vp]),
    "pdb_det_scratch_bytes": (_c_size, [_c_i32, _c_i64]),
    "pdb_det_batch_u32": (_c_i32, [_c_vp, _c_vp, _c_i64, _c_vp, _c_i32, _c_i64, _c_i64, _c_vp,
                                   _c_vp, _c_size, _c_vp]),
    "pdb_eval_det_fused_u32": (_c_i32, [_c_vp, _c_vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_vp, _c_i32, _c_i64,
                                        _c_i64, _c_vp, _c_vp, _c_size, _c_vp]),
    "pdb_node_map_size": (_c_i64, [_c_map]),
    "pdb_det_batch_map_u32": (_c_i32, [_c_vp, _c_vp, _c_i64, _c_vp, _c_i32, _c_map, _c_i64, _c_i64, _c_vp,
                                       _c_vp, _c_size, _c_vp]),
    "pdb_eval_det_fused_map_u32": (_c_i32, [_c_vp, _c_vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_vp, _c_i32, _c_map,
                                            _c_i64, _c_i64, _c_vp, _c_vp, _c_size, _c_vp]),
    "pdb_grid_expand_u32": (_c_i32, [_c_vp, _c_vp, _c_vp, _c_map, _c_vp]),
    "pdb_condense_u32": (_c_i32, [_c_vp, _c_vp, _c_i32, _c_vp, _c_vp, _c_vp, _c_vp, _c_size, _c_vp]),
    "pdb_crt_limbs": (_c_i32, [_c_i32]),
    "pdb_crt_scratch_bytes": (_c_size, [_c_i32]),
    "pdb_crt_mrc_u32": (_c_i32, [_c_vp, _c_i32, _c_i64, _c_i64, _c_vp, _c_vp, _c_i32, _c_vp, _c_vp,
                                 _c_size, _c_vp]),
    "pdb_crt_nonzero_scratch_bytes": (_c_size, [_c_i64]),
    "pdb_crt_nonzero_u32": (_c_i32, [_c_vp, _c_i32, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp, _c_size, _c_vp]),
    "pdb_crt_mrc_sel_u32": (_c_i32, [_c_vp, _c_i32, _c_i64, _c_vp, _c_vp, _c_i64, _c_vp, _c_i32, _c_vp, _c_vp,
                                     _c_vp]),
    "pdb_mulmod_peak": (_c_i32, [_c_u32, _c_i32, ctypes.POINTER(ctypes.c_double), _c_vp]),
    "pdb_kernel_timing": (_c_i32, [_c_i32]),
    "pdb_ntt_forward_kept_u32": (_c_i32, [_c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_vp, _c_vp, _c_u32, _c_vp]),
    "pdb_grid_interpolate_u32": (_c_i32, [_c_vp, _c_vp, _c_vp, _c_vp, _c_map, _c_vp, _c_vp]),
    "pdb_limbs_to_digits30": (_c_i32, [_c_vp, _c_i64, _c_i32, _c_i64, _c_vp, _c_i32, _c_vp, _c_vp]),
    "pdb_kernel_timing_read": (_c_i32, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_c_i64)]),
    # the wide path (2^31 <= p < 2^62): u64 twins
    "pdb_prime_ctx_create_wide": (_c_i32, [_c_u64, _c_u64, _c_i32, ctypes.POINTER(_c_vp)]),
    "pdb_ntt_multi_u64": (_c_i32, [_c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_vp, _c_u32, _c_i32, _c_vp]),
    "pdb_reduce_scatter_u64": (_c_i32, [_c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i32, _c_vp, _c_vp]),
    "pdb_det_scratch_bytes_u64": (_c_size, [_c_i32, _c_i64]),
    "pdb_det_batch_u64": (_c_i32, [_c_vp, _c_vp, _c_i64, _c_vp, _c_i32, _c_i64, _c_i64, _c_vp,
                                   _c_vp, _c_size, _c_vp]),
    "pdb_condense_u64": (_c_i32, [_c_vp, _c_vp, _c_i32, _c_vp, _c_vp, _c_vp, _c_vp, _c_size, _c_vp]),
    "pdb_crt_limbs_u64": (_c_i32, [_c_i32]),
    "pdb_crt_scratch_bytes_u64": (_c_size, [_c_i32]),
    "pdb_crt_mrc_u64": (_c_i32, [_c_vp, _c_i32, _c_i64, _c_i64, _c_vp, _c_vp, _c_i32, _c_vp, _c_vp,
                                 _c_size, _c_vp]),
}


def exported_symbols():
    """Names the header declares (checked by the CPU test suite)."""
    return sorted(_SIGNATURES)


def load_library():
    """Load (once) and type the shared library; raise DeviceError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("PDB_LIBRARY", str(LIB_PATH))
        if not Path(path).is_file():
            raise DeviceError(
                "%s not built (run __graft_entry__.build() or `make -C "
                "paper_2010_12117_b200/csrc`); there is no CPU fallback" % path)
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


_host = None


def host_module():
    """The native host module (csrc/host_ints.cpp): result materialisation."""
    global _host
    if _host is None:
        try:
            from . import _pdb_host
        except ImportError as exc:
            raise DeviceError("_pdb_host native module not built (run __graft_entry__.build() or `make -C "
                              "paper_2010_12117_b200/csrc`): %s" % exc) from exc
        _host = _pdb_host
    return _host


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the determinant pipeline runs only on the GPU")
    return torch


def check(rc: int, what: str = ""):
    if rc == 0:
        return
    msg = load_library().pdb_last_error().decode(errors="replace")
    if rc == -2:
        raise ValueError(msg)
    raise DeviceError("%s failed: %s" % (what or "kernel", msg))


def stream_handle(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def host_i64(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (ctypes.c_int64 * max(len(vals), 1))(*vals)


class PrimeContext:
    """Device twiddle tables + constants of one prime (reference TwiddleTable)."""

    def __init__(self, p: int, omega: int, q: int, device: int, wide: bool = None):
        if p >= WIDE_LIMIT:
            raise ValueError("modulus %d exceeds the device kernels (p < 2^62)" % p)
        wide = needs_wide(p) if wide is None else bool(wide)
        lib = load_library()
        torch = _torch()
        handle = ctypes.c_void_p()
        create = lib.pdb_prime_ctx_create_wide if wide else lib.pdb_prime_ctx_create
        with torch.cuda.device(device):
            check(create(p, omega, q, ctypes.byref(handle)), "prime context")
        self.handle = handle
        self.wide = wide
        self.p, self.omega, self.q, self.device = p, omega, q, device
        self._lib = lib

    def prepare(self, n: int):
        import torch
        with torch.cuda.device(self.device):
            check(self._lib.pdb_prime_ctx_prepare(self.handle, int(n)), "twiddle tables")

    def __del__(self):
        try:
            if self.handle:
                self._lib.pdb_prime_ctx_destroy(self.handle)
        except Exception:
            pass


_contexts: dict = {}


def prime_context(spec, device=None, wide=None) -> PrimeContext:
    """Cached context of one prime; wide=True forces the u64 kernels (a prime
    set mixing p < 2^31 and p >= 2^31 shares one residue width)."""
    torch = _torch()
    dev = torch.cuda.current_device() if device is None else int(device)
    wide = needs_wide(spec.p) if wide is None else bool(wide) or needs_wide(spec.p)
    key = (spec.p, spec.omega, spec.q, dev, wide)
    with _lock:
        ctx = _contexts.get(key)
    if ctx is None:
        ctx = PrimeContext(spec.p, spec.omega, spec.q, dev, wide)
        with _lock:
            _contexts[key] = ctx
    return ctx


# -- thin typed wrappers (device tensors in, nothing returned) ------------------------

def ntt_multi(ctx: PrimeContext, data, batch: int, dims, extents, axes, inverse: bool, stream=None):
    lib = load_library()
    nd = len(dims)
    mask = 0
    for a in axes:
        mask |= 1 << a
    ext = host_i64(extents) if extents is not None else None
    fn = lib.pdb_ntt_multi_u64 if ctx.wide else lib.pdb_ntt_multi_u32
    check(fn(ctx.handle, ptr(data), int(batch), nd, host_i64(dims), ext, mask, int(bool(inverse)),
             stream_handle(stream)), "ntt")


def ntt_forward_kept(ctx: PrimeContext, data, batch: int, dims, extents, kept_u, axes, stream=None):
    """Forward NTT evaluating only the kept nodes of a pruned node set (u32 path)."""
    lib = load_library()
    mask = 0
    for a in axes:
        mask |= 1 << a
    ext = host_i64(extents) if extents is not None else None
    check(lib.pdb_ntt_forward_kept_u32(ctx.handle, ptr(data), int(batch), len(dims), host_i64(dims), ext,
                                       host_i64(kept_u), mask, stream_handle(stream)), "ntt")


def reduce_scatter(ctx: PrimeContext, mag, neg, pos, count: int, limbs: int, dst, stream=None):
    lib = load_library()
    fn = lib.pdb_reduce_scatter_u64 if ctx.wide else lib.pdb_reduce_scatter_u32
    check(fn(ctx.handle, ptr(mag), ptr(neg), ptr(pos), int(count), int(limbs), ptr(dst), stream_handle(stream)),
          "reduce_scatter")


def det_scratch_bytes(r: int, nodes: int, wide: bool = False) -> int:
    lib = load_library()
    fn = lib.pdb_det_scratch_bytes_u64 if wide else lib.pdb_det_scratch_bytes
    return int(fn(int(r), int(nodes)))


def det_batch(ctx: PrimeContext, grids, grid_stride: int, ids, r: int, node_lo: int, nodes: int,
              out, scratch, stream=None):
    lib = load_library()
    fn = lib.pdb_det_batch_u64 if ctx.wide else lib.pdb_det_batch_u32
    check(fn(ctx.handle, ptr(grids), int(grid_stride), ptr(ids), int(r), int(node_lo), int(nodes), ptr(out),
             ptr(scratch), scratch.numel() * scratch.element_size(), stream_handle(stream)), "det")


def eval_det_fused(ctx: PrimeContext, partial, outer: int, ncoef: int, entries: int, n_last: int, ids, r: int,
                   node_lo: int, nodes: int, out, scratch, stream=None):
    """partial: [outer][ncoef][entries] u32 (see include/polydet_b200.h)."""
    lib = load_library()
    check(lib.pdb_eval_det_fused_u32(ctx.handle, ptr(partial), int(outer), int(ncoef), int(entries), int(n_last),
                                     ptr(ids), int(r), int(node_lo), int(nodes), ptr(out), ptr(scratch),
                                     scratch.numel() * scratch.element_size(), stream_handle(stream)),
          "fused det")


def node_map(dims, kept_u):
    """pdb_node_map for a grid of shape dims keeping u < kept_u[a] on each axis
    with kept_u[a] > 0 (None for the identity)."""
    if not any(kept_u):
        return None
    if len(dims) > MAP_MAX_DIMS:
        raise ValueError("node maps support at most %d axes" % MAP_MAX_DIMS)
    m = NodeMapC()
    m.ndim = len(dims)
    for a, (n, u) in enumerate(zip(dims, kept_u)):
        m.dims[a] = int(n)
        m.kept_u[a] = int(u)
    return m


def node_map_size(m) -> int:
    n = int(load_library().pdb_node_map_size(ctypes.byref(m)))
    if n < 0:
        check(-2, "node map")
    return n


def det_batch_map(ctx: PrimeContext, grids, grid_stride: int, ids, r: int, nmap, node_lo: int, nodes: int,
                  out, scratch, stream=None):
    """det_batch over compact nodes [node_lo, node_lo + nodes) of `nmap` (u32 path)."""
    lib = load_library()
    check(lib.pdb_det_batch_map_u32(ctx.handle, ptr(grids), int(grid_stride), ptr(ids), int(r), ctypes.byref(nmap),
                                    int(node_lo), int(nodes), ptr(out), ptr(scratch),
                                    scratch.numel() * scratch.element_size(), stream_handle(stream)), "det")


def eval_det_fused_map(ctx: PrimeContext, partial, outer: int, ncoef: int, entries: int, n_last: int, ids, r: int,
                       nmap, node_lo: int, nodes: int, out, scratch, stream=None):
    lib = load_library()
    check(lib.pdb_eval_det_fused_map_u32(ctx.handle, ptr(partial), int(outer), int(ncoef), int(entries),
                                         int(n_last), ptr(ids), int(r), ctypes.byref(nmap), int(node_lo),
                                         int(nodes), ptr(out), ptr(scratch),
                                         scratch.numel() * scratch.element_size(), stream_handle(stream)),
          "fused det")


def grid_interpolate(ctx: PrimeContext, compact, scratch, grid, nmap, box, stream=None):
    """Kept-node determinants -> coefficients in the box (written into grid; compact is overwritten)."""
    lib = load_library()
    b = (ctypes.c_int64 * len(box))(*[int(x) for x in box])
    check(lib.pdb_grid_interpolate_u32(ctx.handle, ptr(compact), ptr(scratch), ptr(grid), ctypes.byref(nmap), b,
                                       stream_handle(stream)), "grid interpolate")


def grid_expand(ctx: PrimeContext, compact, grid, nmap, stream=None):
    """Determinants at the kept nodes of nmap -> every node of the grid."""
    lib = load_library()
    check(lib.pdb_grid_expand_u32(ctx.handle, ptr(compact), ptr(grid), ctypes.byref(nmap), stream_handle(stream)),
          "grid expand")


def condense(ctx: PrimeContext, mat, r: int, trail_vals, trail_cols, det_out, scratch, stream=None):
    lib = load_library()
    fn = lib.pdb_condense_u64 if ctx.wide else lib.pdb_condense_u32
    check(fn(ctx.handle, ptr(mat), int(r), ptr(trail_vals), ptr(trail_cols), ptr(det_out), ptr(scratch),
             scratch.numel() * scratch.element_size(), stream_handle(stream)), "condense")


def crt_limbs(nprimes: int, wide: bool = False) -> int:
    lib = load_library()
    return int((lib.pdb_crt_limbs_u64 if wide else lib.pdb_crt_limbs)(int(nprimes)))


def crt_scratch_bytes(nprimes: int, wide: bool = False) -> int:
    lib = load_library()
    return int((lib.pdb_crt_scratch_bytes_u64 if wide else lib.pdb_crt_scratch_bytes)(int(nprimes)))


def crt_mrc(residues, nprimes: int, n: int, stride: int, primes, limbs, L: int, neg, scratch, stream=None,
            wide: bool = False):
    lib = load_library()
    if wide:
        hp = (ctypes.c_uint64 * nprimes)(*[int(p) for p in primes])
        fn = lib.pdb_crt_mrc_u64
    else:
        hp = (ctypes.c_uint32 * nprimes)(*[int(p) for p in primes])
        fn = lib.pdb_crt_mrc_u32
    check(fn(ptr(residues), int(nprimes), int(n), int(stride), hp, ptr(limbs), int(L), ptr(neg), ptr(scratch),
             scratch.numel() * scratch.element_size(), stream_handle(stream)), "crt")


def crt_nonzero(residues, nprimes: int, n: int, stride: int, index, count, stream=None):
    """Ascending positions < n with a nonzero residue row -> index; device count."""
    lib = load_library()
    torch = _torch()
    scratch = scratch_tensor(lib.pdb_crt_nonzero_scratch_bytes(int(n)), residues.device)
    check(lib.pdb_crt_nonzero_u32(ptr(residues), int(nprimes), int(n), int(stride), ptr(index), ptr(count),
                                  ptr(scratch), scratch.numel() * scratch.element_size(), stream_handle(stream)),
          "crt nonzero")
    del torch


def crt_mrc_sel(residues, nprimes: int, stride: int, primes, index, count: int, limbs, L: int, neg, width,
                stream=None):
    """CRT lift at positions index[0..count) (index None: 0..count-1), compact output."""
    lib = load_library()
    hp = (ctypes.c_uint32 * nprimes)(*[int(p) for p in primes])
    check(lib.pdb_crt_mrc_sel_u32(ptr(residues), int(nprimes), int(stride), hp,
                                  ptr(index) if index is not None else None, int(count), ptr(limbs), int(L),
                                  ptr(neg), ptr(width) if width is not None else None, stream_handle(stream)),
          "crt")


def launch_count() -> int:
    """Kernels this process has launched through the library (all devices)."""
    return int(load_library().pdb_launch_count())


def limbs_to_digits30(limbs, count: int, width: int, stride: int, digits, ndigits: int, digit_count,
                      stream=None):
    """Limb rows [count][width] (row stride `stride`) -> 30-bit digit rows [count][ndigits] + counts."""
    check(load_library().pdb_limbs_to_digits30(ptr(limbs), int(count), int(width), int(stride), ptr(digits),
                                               int(ndigits), ptr(digit_count), stream_handle(stream)),
          "limbs to digits")


def kernel_timing(enable: bool) -> None:
    """Start (clearing the record) or stop CUDA-event timing of every det_gj launch."""
    check(load_library().pdb_kernel_timing(1 if enable else 0), "kernel timing")


def kernel_timing_read():
    """(summed device ms, launches) of the det_gj launches recorded since kernel_timing(True)."""
    ms, n = ctypes.c_double(), ctypes.c_int64()
    check(load_library().pdb_kernel_timing_read(ctypes.byref(ms), ctypes.byref(n)), "kernel timing")
    return ms.value, n.value


def mulmod_peak(p: int, variant: int) -> float:
    lib = load_library()
    _torch()
    out = ctypes.c_double()
    check(lib.pdb_mulmod_peak(int(p), int(variant), ctypes.byref(out), stream_handle()), "peak")
    return out.value


# -- host <-> device helpers ---------------------------------------------------------

def to_device_u32(values, device=None):
    """numpy residues (any int dtype, values < 2^32) -> int32-typed device tensor."""
    torch = _torch()
    arr = np.ascontiguousarray(np.asarray(values).astype(np.uint32, copy=False)).view(np.int32)
    return torch.from_numpy(arr).to(device or torch.cuda.current_device())


def to_host_u32(t) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint32)


def word_dtype(wide: bool):
    """Device residue word: int32 (u32 kernels) or int64 (u64 kernels, values < 2^62)."""
    torch = _torch()
    return torch.int64 if wide else torch.int32


def to_device_words(values, wide: bool, device=None):
    """Residues (numpy, any int or object dtype) -> device tensor of the path's word."""
    if not wide:
        return to_device_u32(values, device)
    torch = _torch()
    arr = np.asarray(values)
    arr = np.array([int(v) for v in arr.reshape(-1)], dtype=np.int64).reshape(arr.shape) if arr.dtype == object \
        else np.array(arr, dtype=np.int64)
    return torch.from_numpy(arr).to(device or torch.cuda.current_device())


def to_host_words(t, wide: bool) -> np.ndarray:
    """Device residues -> numpy uint32 / uint64."""
    if not wide:
        return to_host_u32(t)
    return t.detach().cpu().numpy().view(np.uint64)


def scratch_tensor(nbytes: int, device=None):
    torch = _torch()
    words = max((int(nbytes) + 15) // 16 * 4, 4)
    return torch.empty(words, dtype=torch.int32, device=device or torch.cuda.current_device())
