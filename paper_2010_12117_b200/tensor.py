"""Reference module name `polydet.tensor` (tensor.py): coefficient tensors and
polynomial matrices, re-exported from this package's layout module."""

from .layout import (  # noqa: F401
    CoeffTensor,
    DegreeVector,
    ModTensor,
    PolyMatrix,
    axis_rotate,
    encode,
    normalize_terms,
    pad_shape,
    pad_to,
    poly_matrix,
    reduce_mod,
    residue_dtype,
    tensor_from_terms,
)
