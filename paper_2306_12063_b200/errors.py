"""Exception hierarchy of the codec boundary.

Same names and meanings as the reference's `qcldpc.errors`
(`/root/reference/pkg/src/qcldpc/errors.py:4-37`) so callers that catch the
reference's exceptions keep working after the switch.  Two additions report
conditions only the GPU path can hit (missing native library, device error).
"""


class CodecError(Exception):
    """Root of every error raised by the codec."""


class UnsupportedCode(CodecError):
    """No code is defined for the requested (standard, N, rate)."""


class BadZ(CodecError):
    """Lifting size outside the standard's table."""


class UnsupportedZ(CodecError):
    """The packed encoder needs a lifting size that is a multiple of 8."""


class MalformedHb(CodecError):
    """The h_b column does not have exactly one interior non-negative entry."""


class SizeMismatch(CodecError):
    """An array's length disagrees with the code dimensions."""


class ArithmeticMismatch(CodecError):
    """LLR arithmetic differs from the decoder configuration."""


class DivByZeroSigma(CodecError):
    """A zero noise variance cannot be turned into channel LLRs."""


class CorruptFile(CodecError):
    """A file's bytes disagree with its declared layout."""


class NativeLibraryError(CodecError):
    """libqcb200.so is missing, stale or failed to load (no CPU fallback)."""


class DeviceError(CodecError):
    """A CUDA call inside libqcb200 failed; the message carries the CUDA error."""
