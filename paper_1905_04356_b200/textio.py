"""Interchange formats of dense polynomial matrices (host side, native).

Text is the reference CLI format of polmat_to_text / polmat_from_text
(ref polmat.py:617-647), byte for byte, produced and parsed by
libfpm_b200.so on all host threads (fpm_polmat_to_text / _from_text; no GPU
needed).  The binary format (.fpmb) is this library's own: a 32-byte
little-endian header, the per-entry trimmed lengths, then the dense
coefficients, readable with numpy without parsing (and memory-mappable).

Dense layout as everywhere in this package: (m, n, L), coefficient t of
entry (i, j) at [i, j, t], trailing zeros allowed (trimmed on output).
"""
import ctypes
import struct

import numpy as np

from . import _lib

_MAGIC = b"FPMB"
_VERSION = 1
_HEAD = struct.Struct("<4sIQIIII")  # magic, version, p, m, n, L, elem_bytes


def _as_host(M, p):
    """numpy (m, n, L) view of M (numpy array or torch tensor, any device)."""
    if hasattr(M, "detach"):
        M = M.detach().cpu().numpy()
    a = np.asarray(M)
    if a.ndim != 3:
        raise ValueError("expected a dense (m, n, L) matrix")
    eb = 4 if p < (1 << 32) and a.dtype.itemsize <= 4 else 8
    dt = np.uint32 if eb == 4 else np.uint64
    if a.dtype.kind == "i":
        a = a.view(np.uint32 if a.dtype.itemsize == 4 else np.uint64)
    return np.ascontiguousarray(a, dtype=dt), eb


def dense_to_text(M, p):
    """polmat_to_text (polmat.py:617-623) of a dense matrix -> str."""
    a, eb = _as_host(M, p)
    m, n, L = a.shape
    L_ = _lib.lib()
    size = ctypes.c_size_t(0)
    _lib.check(L_.fpm_polmat_text_size(p, eb, a.ctypes.data, m, n, L, ctypes.byref(size)),
               "fpm_polmat_text_size")
    buf = np.empty(size.value, dtype=np.uint8)
    wrote = ctypes.c_size_t(0)
    _lib.check(L_.fpm_polmat_to_text(p, eb, a.ctypes.data, m, n, L, buf.ctypes.data,
                                     size.value, ctypes.byref(wrote)), "fpm_polmat_to_text")
    return buf[: wrote.value].tobytes().decode("ascii")


def dense_from_text(text, elem_bytes=None):
    """polmat_from_text (polmat.py:626-647) -> (p, dense numpy (m, n, L)),
    L = the longest trimmed entry (at least 0)."""
    raw = text.encode() if isinstance(text, str) else bytes(text)
    L_ = _lib.lib()
    p, m, n, L = ctypes.c_longlong(0), ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    _lib.check(L_.fpm_polmat_text_dims(raw, len(raw), ctypes.byref(p), ctypes.byref(m),
                                       ctypes.byref(n), ctypes.byref(L)), "polmat_from_text")
    eb = elem_bytes or (4 if p.value < (1 << 32) else 8)
    out = np.zeros((m.value, n.value, L.value), dtype=np.uint32 if eb == 4 else np.uint64)
    _lib.check(L_.fpm_polmat_from_text(raw, len(raw), eb, out.ctypes.data, L.value),
               "polmat_from_text")
    return int(p.value), out


def save_binary(path, M, p):
    """Write a dense matrix as .fpmb (header, trimmed lengths, coefficients)."""
    a, eb = _as_host(M, p)
    m, n, L = a.shape
    nz = a != 0
    lens = np.where(nz.any(axis=2), L - np.argmax(nz[:, :, ::-1], axis=2), 0).astype(np.uint32)
    with open(path, "wb") as f:
        f.write(_HEAD.pack(_MAGIC, _VERSION, p, m, n, L, eb))
        f.write(lens.tobytes())
        f.write(a.tobytes())


def load_binary(path, mmap=False):
    """Read .fpmb -> (p, dense numpy (m, n, L), trimmed lengths (m, n))."""
    with open(path, "rb") as f:
        head = f.read(_HEAD.size)
    magic, ver, p, m, n, L, eb = _HEAD.unpack(head)
    if magic != _MAGIC or ver != _VERSION or eb not in (4, 8):
        raise ValueError(f"{path}: not an FPMB v{_VERSION} file")
    dt = np.uint32 if eb == 4 else np.uint64
    off = _HEAD.size + 4 * m * n
    lens = np.fromfile(path, dtype=np.uint32, count=m * n, offset=_HEAD.size).reshape(m, n)
    if mmap:
        data = np.memmap(path, dtype=dt, mode="r", offset=off, shape=(m, n, L))
    else:
        data = np.fromfile(path, dtype=dt, count=m * n * L, offset=off).reshape(m, n, L)
    return int(p), data, lens
