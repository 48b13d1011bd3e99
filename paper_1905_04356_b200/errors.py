"""Exception hierarchy mirroring the reference (fpmat/errors.py:1-109).

When the reference package is importable these ARE the reference classes, so
callers that catch ``fpmat.errors.X`` keep working after the drop-in; on the
GPU box (no reference) an identical local hierarchy is defined.
"""
_NAMES = [
    "CompositeModulus", "OutOfRange", "LengthMismatch", "NoSuchElement", "CtxMismatch",
    "DegreeTooLarge", "OrderTooSmall", "DuplicatePoints", "NotInvertibleAtZero", "BothZero",
    "DimMismatch", "EnvelopeExceeded", "NotSquare", "ReconstructionFailed", "NoGeometricGrid",
    "SingularAtZero", "SingularMatrix", "InsufficientPrecision", "DimensionCap",
    "FieldTooSmall", "VerificationFailed", "TooLarge", "NotCoprime", "GenericityFailure",
    "SingularEvaluation", "BadParams",
]

try:  # pragma: no cover - depends on the environment
    from fpmat import errors as _ref  # type: ignore

    FpmatError = _ref.FpmatError
    for _n in _NAMES:
        globals()[_n] = getattr(_ref, _n)
except Exception:  # reference not importable: local mirror
    class FpmatError(Exception):
        """Base class for all library errors."""

    for _n in _NAMES:
        globals()[_n] = type(_n, (FpmatError,), {})

__all__ = ["FpmatError"] + _NAMES
