"""B200-native F_p polynomial-matrix multiply and PM-Basis.

Drop-in for the hot path of the reference `fpmat` package (arXiv:1905.04356):
``pm_mul``, ``pm_middle_product`` / ``_pm_middle``, ``Multiplier``,
``mbasis`` / ``pmbasis``, ``m_intbasis`` / ``pm_intbasis`` with the reference's names, argument meaning and
exceptions, computed by hand-written sm_100a kernels in libfpm_b200.so
(csrc/) behind the C ABI declared in include/fpmat_b200.h.
"""
from . import config, errors  # noqa: F401
from .modring import FieldCtx, NttPlan, cached_field, field_new, ntt_forward, ntt_inverse  # noqa: F401
from .polmat import (  # noqa: F401
    STRATEGIES,
    Multiplier,
    PolMat,
    _pm_middle,
    applicable_strategies,
    pm_middle_product,
    pm_mul,
    polmat_from_text,
    polmat_to_text,
    random_polmat,
)
from .appint import eval_polmat_points, m_intbasis, mbasis, mbasis1, pm_intbasis, pmbasis  # noqa: F401

__all__ = [
    "FieldCtx", "NttPlan", "field_new", "cached_field", "ntt_forward", "ntt_inverse",
    "PolMat", "pm_mul", "pm_middle_product", "applicable_strategies", "Multiplier",
    "polmat_to_text", "polmat_from_text", "random_polmat", "mbasis", "mbasis1", "pmbasis",
    "m_intbasis", "pm_intbasis", "eval_polmat_points",
]
