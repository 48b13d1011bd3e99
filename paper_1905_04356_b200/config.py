"""Tuning knobs (mirror of fpmat/config.py:10-24 for the hot path).

As in the reference (config.py:3-5) these only choose which exact algorithm
runs, never the result.
"""
# PM-Basis recursion base case (config.py:18); the GPU output is identical
# for every value (the basis is the product of canonical order-1 steps).
PMBASIS_BASE_ORDER = 32
# reference dispatch constants that affect *semantics* of _pm_middle
# (upoly.py:353, polmat.py:494) -- kept to reproduce the reference bit for bit
MIDDLE_PRODUCT_FFT_MIN = 64
# reference pm_mul dispatch (kept for `applicable_strategies` parity only)
PM_MUL_NAIVE_MAX_DIM = 10
PM_MUL_EVAL_MIN_POINTS = 8
