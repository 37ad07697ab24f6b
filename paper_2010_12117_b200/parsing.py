"""Reference module name `polydet.parsing`: the result printer only (the text
grammar of input documents is out of scope)."""

from .formatting import format_polynomial  # noqa: F401
