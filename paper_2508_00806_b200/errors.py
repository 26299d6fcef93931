"""Exception taxonomy of the compressor path.

Names and meaning follow the reference package's ``actplan.errors``
(/root/reference/pkg/src/actplan/errors.py:6-34) so that callers catching the
reference exceptions catch ours by the same name.  The device kernels report
data-dependent failures as bits of a 32-bit error word (see
``include/adacc.h``); :func:`raise_for_error_word` maps those bits back onto
these types.
"""

from __future__ import annotations


class ActplanError(Exception):
    """Base class (errors.py:6)."""


class ParseError(ActplanError):
    """Malformed profile / plan file (errors.py:10)."""


class ValidationError(ActplanError):
    """A documented invariant is violated: bad shape, group size ... (errors.py:14)."""


class NonFiniteInputError(ActplanError):
    """An activation is NaN/inf after the float16 cast (errors.py:21)."""


class CorruptPayloadError(ActplanError):
    """An ADC1 wire payload fails structural validation (errors.py:25)."""


class NonBinaryMaskError(ActplanError):
    """A dropout mask holds values other than 0 and 1 (errors.py:29)."""


class TooManyOutliersError(ActplanError):
    """More than half of all channels were flagged as outliers (errors.py:33)."""


class OutlierCapacityError(ActplanError):
    """More outlier channels than the caller-sized side buffer can hold.

    Not a reference error: the reference allocates on the host after it knows
    k.  The device path writes into caller-owned buffers sized for ``k_cap``
    and reports overflow instead; the Python wrapper grows the buffer and
    re-runs, so this never escapes :func:`compress`.
    """


class CudaError(ActplanError):
    """A CUDA launch / runtime failure reported through the C-ABI."""


# Error-word bits written by the kernels (mirrors include/adacc.h).
ERR_NONFINITE = 1 << 0
ERR_TOO_MANY_OUTLIERS = 1 << 1
ERR_K_CAP = 1 << 2
ERR_NONBINARY = 1 << 3


def raise_for_error_word(word: int, *, rows: int = 0, cols: int = 0, k: int = 0) -> None:
    """Raise the reference exception that corresponds to a device error word.

    Order of precedence follows the reference control flow: the float16 cast
    is checked first (codec.py:167-170), then the outlier-count guard
    (codec.py:324-327).
    """
    if not word:
        return
    if word & ERR_NONFINITE:
        raise NonFiniteInputError(
            "activation values must be finite in half precision (NaN, infinity, or overflow found)"
        )
    if word & ERR_NONBINARY:
        raise NonBinaryMaskError("mask bytes must be 0 or 1")
    if word & ERR_TOO_MANY_OUTLIERS:
        raise TooManyOutliersError(
            f"{k} of {cols} channels flagged as outliers; refusing to compress"
        )
    if word & ERR_K_CAP:
        raise OutlierCapacityError(f"{k} outlier channels exceed the side-buffer capacity")
    raise CudaError(f"unknown device error word 0x{word:x}")
