"""Reference module name `polydet.workspace` (workspace.py): checkpoint/resume
artifacts, re-exported from this package's checkpoint module."""

from .checkpoint import Workspace, decode_array, digest_of, encode_array, stable_json  # noqa: F401
