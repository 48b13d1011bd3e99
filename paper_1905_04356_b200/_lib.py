"""ctypes binding of libfpm_b200.so (include/fpmat_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every compute entry point raises
:class:`FpmBackendError`.  Status codes map 1:1 onto the reference exception
classes (fpmat/errors.py) -- see ``_raise``.
"""
import ctypes
import os
import subprocess
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfpm_b200.so")
# test-only build: the product objects plus the tensor-core self-test hooks
# (csrc/tc_selftest.cu); never loaded by the package itself
SELFTEST_PATH = os.path.join(_HERE, "libfpm_b200_selftest.so")

_lock = threading.Lock()
_lib = None
_ctx = {}
_st_lib = None
_st_ctx = {}


class FpmBackendError(RuntimeError):
    """CUDA library missing / no device / CUDA failure."""


_STATUS = {
    1: errors.DimMismatch,
    2: errors.CtxMismatch,
    3: errors.OrderTooSmall,
    4: errors.FieldTooSmall,
    5: errors.DegreeTooLarge,
    6: errors.EnvelopeExceeded,
    7: errors.LengthMismatch,
    8: errors.OutOfRange,
    9: errors.CompositeModulus,
    10: errors.DuplicatePoints,
    11: errors.NoSuchElement,
    20: ValueError,
    21: NotImplementedError,
}


def build(force=False, verbose=False):
    """Compile the CUDA library in-tree (make -C paper_1905_04356_b200)."""
    args = ["make", "-j8", "-C", _HERE]
    if force:
        subprocess.run(["make", "-C", _HERE, "clean"], check=True,
                       stdout=subprocess.DEVNULL)
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(args, check=True, stdout=out)
    return LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise FpmBackendError(
                f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u32, u64 = (ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong,
                                  ctypes.c_uint32, ctypes.c_uint64)
        pi64 = ctypes.POINTER(ctypes.c_int64)
        pint = ctypes.POINTER(ctypes.c_int)
        sig = {
            "fpm_version": (i32, []),
            "fpm_last_error": (ctypes.c_char_p, []),
            "fpm_launch_count": (i64, []),
            "fpm_context_create": (i32, [i32, ctypes.POINTER(vp)]),
            "fpm_context_destroy": (None, [vp]),
            "fpm_context_set_stream": (i32, [vp, vp]),
            "fpm_context_synchronize": (i32, [vp]),
            "fpm_field_info": (i32, [u64, pint, ctypes.POINTER(ctypes.c_uint64)]),
            "fpm_is_prime": (i32, [u64]),
            "fpm_factorize": (i32, [u64, ctypes.POINTER(ctypes.c_uint64), pint, i32, pint]),
            "fpm_element_order": (i32, [u64, u64, ctypes.POINTER(ctypes.c_uint64)]),
            "fpm_order_at_least": (i32, [u64, u64, ctypes.POINTER(ctypes.c_uint64)]),
            "fpm_ntt_u32": (i32, [vp, u32, i32, i32, vp, vp, i32]),
            "fpm_ntt_u64": (i32, [vp, u64, i32, i32, vp, vp, i32]),
            "fpm_polmat_mul": (i32, [vp, u64, i32, vp, i32, i32, i32, vp, i32, i32, vp]),
            "fpm_product_primes": (i32, [u64, i32, i32, i32, ctypes.POINTER(ctypes.c_uint32),
                                         i32, pint]),
            "fpm_split_residues": (i32, [vp, i32, vp, i64, ctypes.POINTER(ctypes.c_uint32), i32,
                                         vp]),
            "fpm_crt_combine": (i32, [vp, u64, i32, ctypes.POINTER(ctypes.c_uint32), i32, vp,
                                      i64, i32, vp]),
            "fpm_polmat_mul_host": (i32, [vp, u64, i32, vp, i32, i32, i32, vp, i32, i32, vp]),
            "fpm_polmat_middle": (i32, [vp, u64, i32, vp, i32, i32, i32, vp, i32, i32, i64,
                                        i32, i32, vp]),
            "fpm_pm_middle_product": (i32, [vp, u64, i32, vp, i32, i32, i32, vp, i32, i32,
                                            i64, i32, vp]),
            "fpm_mbasis": (i32, [vp, u64, i32, vp, i32, i32, i32, i32, pi64, vp, pint, pi64]),
            "fpm_pmbasis": (i32, [vp, u64, i32, vp, i32, i32, i32, i32, pi64, vp, pint, pi64]),
            "fpm_pmbasis_host": (i32, [vp, u64, i32, vp, i32, i32, i32, i32, pi64, vp, pint,
                                       pi64]),
            "fpm_set_pmbasis_threshold": (i32, [vp, i32]),
            "fpm_set_option": (i32, [ctypes.c_char_p, i64]),
            "fpm_pm_intbasis": (i32, [vp, u64, i32, vp, i32, i32, i32,
                                      ctypes.POINTER(ctypes.c_uint64), pi64, vp, pint, pi64]),
            "fpm_m_intbasis": (i32, [vp, u64, i32, vp, i32, i32, i32,
                                     ctypes.POINTER(ctypes.c_uint64), pi64, vp, pint, pi64]),
            "fpm_polmat_eval_points": (i32, [vp, u64, i32, vp, i32, i32, i32,
                                             ctypes.POINTER(ctypes.c_uint64), i32, vp]),
            "fpm_multiplier_create": (i32, [vp, u64, i32, vp, i32, i32, i32, i32,
                                            ctypes.POINTER(vp)]),
            "fpm_multiplier_apply": (i32, [vp, vp, i32, i32, vp]),
            "fpm_multiplier_destroy": (None, [vp]),
            "fpm_polmat_text_size": (i32, [u64, i32, vp, i32, i32, i32,
                                           ctypes.POINTER(ctypes.c_size_t)]),
            "fpm_polmat_to_text": (i32, [u64, i32, vp, i32, i32, i32, vp,
                                         ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
            "fpm_polmat_text_dims": (i32, [ctypes.c_char_p, ctypes.c_size_t,
                                           ctypes.POINTER(ctypes.c_longlong), pint, pint, pint]),
            "fpm_polmat_from_text": (i32, [ctypes.c_char_p, ctypes.c_size_t, i32, vp, i32]),
            "fpm_profile_enable": (i32, [vp, i32]),
            "fpm_profile_count": (i32, [vp]),
            "fpm_profile_get": (i32, [vp, i32, ctypes.c_char_p, i32,
                                      ctypes.POINTER(ctypes.c_float)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    """Names declared in include/fpmat_b200.h (checked by the CPU tests)."""
    import re

    hdr = os.path.join(os.path.dirname(_HERE), "include", "fpmat_b200.h")
    with open(hdr) as f:
        txt = f.read()
    return sorted(set(re.findall(r"\b(fpm_[a-z0-9_]+)\s*\(", txt)))


def _raise(status, what):
    msg = lib().fpm_last_error().decode(errors="replace")
    exc = _STATUS.get(status)
    if exc is None:
        raise FpmBackendError(f"{what}: status {status}: {msg}")
    raise exc(f"{what}: {msg}")


def check(status, what):
    if status != 0:
        _raise(status, what)


def context(device=None):
    """Process-wide context per device, bound to torch's current stream."""
    import torch

    if not torch.cuda.is_available():
        raise FpmBackendError("no CUDA device: the B200 product path has no CPU fallback")
    if device is None:
        device = torch.cuda.current_device()
    L = lib()
    with _lock:
        h = _ctx.get(device)
        if h is None:
            hp = ctypes.c_void_p()
            with torch.cuda.device(device):
                check(L.fpm_context_create(device, ctypes.byref(hp)), "fpm_context_create")
            h = hp
            _ctx[device] = h
    stream = torch.cuda.current_stream(device).cuda_stream
    check(L.fpm_context_set_stream(h, ctypes.c_void_p(stream)), "fpm_context_set_stream")
    return h


def profile(h, on=True):
    check(lib().fpm_profile_enable(h, 1 if on else 0), "fpm_profile_enable")


def profile_records(h):
    """[(stage name, ms)] recorded since profile(h, True)."""
    L = lib()
    out = []
    buf = ctypes.create_string_buffer(64)
    ms = ctypes.c_float()
    for i in range(L.fpm_profile_count(h)):
        check(L.fpm_profile_get(h, i, buf, 64, ctypes.byref(ms)), "fpm_profile_get")
        out.append((buf.value.decode(), float(ms.value)))
    return out


def launch_count():
    return int(lib().fpm_launch_count())


def set_option(name, value):
    """fpm_set_option: kernel-selection switches for A/B measurements
    (include/fpmat_b200.h); name None resets every option."""
    check(lib().fpm_set_option(None if name is None else name.encode(), int(value)),
          "fpm_set_option")


def selftest_lib():
    """The test-only library (tensor-core kernels called directly)."""
    global _st_lib
    with _lock:
        if _st_lib is None:
            if not os.path.exists(SELFTEST_PATH):
                raise FpmBackendError(f"{SELFTEST_PATH} not built")
            L = ctypes.CDLL(SELFTEST_PATH)
            L.fpm_context_create.restype = ctypes.c_int
            L.fpm_context_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
            L.fpm_context_set_stream.restype = ctypes.c_int
            L.fpm_context_set_stream.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
            _st_lib = L
    return _st_lib


def selftest_context(device=0):
    """A context of the self-test library on torch's current stream."""
    import torch

    L = selftest_lib()
    with _lock:
        h = _st_ctx.get(device)
        if h is None:
            hp = ctypes.c_void_p()
            with torch.cuda.device(device):
                rc = L.fpm_context_create(device, ctypes.byref(hp))
            if rc != 0:
                raise FpmBackendError(f"selftest fpm_context_create: status {rc}")
            h = _st_ctx[device] = hp
    rc = L.fpm_context_set_stream(h, ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream))
    if rc != 0:
        raise FpmBackendError(f"selftest fpm_context_set_stream: status {rc}")
    return h
