"""Error taxonomy of the drop-in (mirrors /root/reference/pkg/src/hhsar/errors.py:9-27).

The reference maps ConfigError / IoFormatError / NumericDomainError to CLI
exit codes 2 / 3 / 4 (cli.py:483-494).  The same class names and the same
hierarchy are kept so callers that catch the reference's exceptions by name
keep working.  When the reference package ``hhsar`` is already imported in the
process (the ``install()`` operator shim), its classes are reused so an
``except hhsar.NumericDomainError`` clause also catches errors raised here.
"""

from __future__ import annotations

import sys

_ref = sys.modules.get("hhsar.errors")

if _ref is not None:  # share identity with the reference's exception classes
    HhsarError = _ref.HhsarError
    ConfigError = _ref.ConfigError
    IoFormatError = _ref.IoFormatError
    NumericDomainError = _ref.NumericDomainError
else:
    class HhsarError(Exception):
        """Base class for every error raised by the package."""

    class ConfigError(HhsarError):
        """Bad argument, configuration or geometry supplied by the caller."""

    class IoFormatError(HhsarError):
        """Malformed, truncated or inconsistent file content."""

    class NumericDomainError(HhsarError):
        """Inputs outside the mathematical domain of an operation (delays
        outside the profile window, unreachable lattices, ...)."""


class NativeUnavailableError(RuntimeError):
    """The sm_100a CUDA library is missing or no B200 is visible.

    There is deliberately no CPU fallback: the product path fails loudly.
    """


EXIT_CODES = {ConfigError: 2, IoFormatError: 3, NumericDomainError: 4}
