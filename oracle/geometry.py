"""Wrap-around diagonal geometry and products (float64) — TEST INFRASTRUCTURE ONLY.

Restates reference ``pkg/src/diagsparse/diagcore.py`` (and the scipy "compact"
product of ``bcsr.py:391-409``).  Conventions (diagcore.py:1-8, 106-116):

* W is M x N, C = max(M, N) candidate offsets, each diagonal has L = min(M, N)
  stored values.
* M >= N: value t of offset o sits at ((o + t) mod M, t).
* M <  N: value t of offset o sits at (t, (o + t) mod N).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp


def candidate_count(rows: int, cols: int) -> int:
    """diagcore.py:22-26 — number of distinct wrap-around diagonals."""
    if rows < 1 or cols < 1:
        raise ValueError(f"dimensions must be positive, got {rows}x{cols}")
    return max(rows, cols)


def required_diagonals(rows: int, cols: int, sparsity: float) -> int:
    """diagcore.py:29-48 — K = round_half_up((1-s) M N / min(M,N)) in [1, C]."""
    s = float(sparsity)
    if not (0.0 <= s < 1.0):
        raise ValueError(f"sparsity must be in [0, 1), got {sparsity}")
    k = math.floor((1.0 - s) * rows * cols / min(rows, cols) + 0.5)
    return int(min(max(k, 1), candidate_count(rows, cols)))


def entry_coords(rows: int, cols: int, offsets) -> tuple[np.ndarray, np.ndarray]:
    """diagcore.py:106-116 and layers.py:53-60 — stacked (K, L) row/col indices.

    Row j of each array lists the coordinates of offsets[j] in storage order.
    """
    offs = np.asarray(offsets, dtype=np.int64).reshape(-1, 1)
    t = np.arange(min(rows, cols), dtype=np.int64).reshape(1, -1)
    if rows >= cols:
        return (offs + t) % rows, np.broadcast_to(t, (offs.shape[0], t.shape[1])).copy()
    return np.broadcast_to(t, (offs.shape[0], t.shape[1])).copy(), (offs + t) % cols


def dense_matrix(rows: int, cols: int, offsets, values) -> np.ndarray:
    """diagcore.py:153-159 — scatter the diagonals into a dense M x N array."""
    r, c = entry_coords(rows, cols, offsets)
    out = np.zeros((rows, cols))
    out[r.ravel(), c.ravel()] = np.asarray(values, dtype=np.float64).ravel()
    return out


def transpose_diagonals(rows: int, cols: int, offsets, values):
    """diagcore.py:162-191 — transpose as a pure index remap.

    Rectangular: offsets and values carry over unchanged (diagcore.py:172-177).
    Square: offset s -> (N - s) mod N, values rotated so that new slot
    (s + t) mod N receives old value t, then re-sorted by new offset
    (diagcore.py:179-189).  Returns (offsets_T, values_T) of the N x M matrix.
    """
    offs = [int(o) for o in offsets]
    vals = np.asarray(values, dtype=np.float64)
    if rows != cols:
        return tuple(offs), vals.copy()
    n = rows
    flipped = [(n - s) % n for s in offs]
    perm = np.argsort(flipped)
    out = np.empty_like(vals)
    t = np.arange(n)
    for dst, src in enumerate(perm):
        rotated = np.empty(n)
        rotated[(offs[src] + t) % n] = vals[src]
        out[dst] = rotated
    return tuple(flipped[j] for j in perm), out


def diag_spmm(rows: int, cols: int, offsets, values, X: np.ndarray) -> np.ndarray:
    """diagcore.py:200-238 — Y = W @ X, diagonal by diagonal.

    X is (N, B); the result is (M, B).  Above structural density 1/4 the
    reference multiplies the materialized matrix with BLAS instead
    (diagcore.py:226-228); that switch is kept so timings stay comparable.
    """
    X = np.asarray(X, dtype=np.float64)
    vec = X.ndim == 1
    if vec:
        X = X[:, None]
    if X.shape[0] != cols:
        raise ValueError(f"X has {X.shape[0]} rows, expected {cols}")
    vals = np.asarray(values, dtype=np.float64)
    L = min(rows, cols)
    if 4 * len(offsets) * L >= rows * cols:
        Y = dense_matrix(rows, cols, offsets, vals) @ X
        return Y[:, 0] if vec else Y
    Y = np.zeros((rows, X.shape[1]))
    t = np.arange(L)
    for j, o in enumerate(offsets):
        if rows >= cols:
            Y[(o + t) % rows] += vals[j][:, None] * X
        else:
            Y += vals[j][:, None] * X[(o + t) % cols]
    return Y[:, 0] if vec else Y


def csr_spmm(rows: int, cols: int, offsets, values, X: np.ndarray) -> np.ndarray:
    """bcsr.py:391-409 ("compact" strategy) — Y = W @ X through scipy CSR.

    The reference reorders rows before blocking (bcsr.py:161-224); a row
    permutation does not change any row's sum, so the product is the same
    scipy ``csr_matvecs`` arithmetic on the un-permuted rows.
    """
    r, c = entry_coords(rows, cols, offsets)
    W = sp.csr_matrix(
        (np.asarray(values, dtype=np.float64).ravel(), (r.ravel(), c.ravel())),
        shape=(rows, cols),
    )
    return W @ np.asarray(X, dtype=np.float64)
