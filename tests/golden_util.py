"""Helpers shared by the tests: fixture loading and PolMat-rows <-> dense."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_small = None


def small():
    global _small
    if _small is None:
        with open(os.path.join(GOLDEN, "small.json")) as f:
            _small = json.load(f)
    return _small


def big_goldens():
    out = {}
    path = os.path.join(GOLDEN, "big_goldens.jsonl")
    if os.path.exists(path):
        with open(path) as f:
            for line in f:
                line = line.strip()
                if line:
                    rec = json.loads(line)
                    out[rec["key"]] = rec
    return out


def dense(rows, m, n, L=None, dtype=np.uint64):
    """PolMat rows (trimmed lists) -> dense (m, n, L) array."""
    if L is None:
        L = max([len(e) for r in rows for e in r] + [0])
    out = np.zeros((m, n, max(L, 0)), dtype=dtype)
    for i, r in enumerate(rows):
        for j, e in enumerate(r):
            if e:
                out[i, j, : len(e)] = e
    return out


def rows_from_dense(M):
    M = np.asarray(M)
    rows = []
    for i in range(M.shape[0]):
        row = []
        for j in range(M.shape[1]):
            e = M[i, j]
            nz = np.flatnonzero(e)
            L = int(nz[-1]) + 1 if nz.size else 0
            row.append([int(c) for c in e[:L]])
        rows.append(row)
    return rows


def random_polmat_dense(p, m, n, deg, rng):
    """Dense equivalent of fpmat.polmat.random_polmat (polmat.py:650-659):
    coefficients drawn with rng.randrange(p) in row-major entry order."""
    out = np.zeros((m, n, deg + 1), dtype=np.uint64)
    for i in range(m):
        for j in range(n):
            out[i, j] = [rng.randrange(p) for _ in range(deg + 1)]
    return out
