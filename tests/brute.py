"""Independent pins for the oracle (test-only; shares nothing with oracle/ or csrc/).

* dense_permute: brute-force dense transpose with numpy (np.transpose has exactly the
  torch.permute semantics the ABI uses) plus a tag channel that recovers the
  permutation vector (SURVEY.md §8(c) pin 4).
* closed forms of the stencil operators under the BASELINE permutations, enumerated
  directly in output order (SURVEY.md §8(c) pin 3).
* certificate: properties that, for unique keys, imply equality with the oracle
  (SURVEY.md §8(c) pin 5).
"""
from __future__ import annotations

import numpy as np


def dense_permute(dims, perm, keys, vals):
    dims = [int(d) for d in dims]
    keys = np.asarray(keys, dtype=np.int64)
    total = int(np.prod(dims)) if dims else 1
    tag = np.zeros(total, dtype=np.int64)
    tag[keys] = np.arange(1, len(keys) + 1)
    t = tag.reshape(dims).transpose(list(perm)).reshape(-1)  # row-major scan of the transpose
    nz = np.nonzero(t)[0]
    src = t[nz] - 1
    return nz.astype(np.uint64), np.asarray(vals)[src], src.astype(np.uint32)


def _ravel(coords, dims):
    return np.ravel_multi_index(tuple(np.asarray(c, dtype=np.int64) for c in coords),
                                tuple(int(d) for d in dims)).astype(np.int64)


def source_positions(keys_in, dims, perm, keys_out):
    """perm vector of an output: for each output key, the position in keys_in of the
    entry it came from (unravel under the new dims, ravel the source coordinates)."""
    dims = [int(d) for d in dims]
    ndims = [dims[p] for p in perm]
    oc = np.unravel_index(np.asarray(keys_out, dtype=np.int64), ndims)
    sc = [None] * len(dims)
    for t, p in enumerate(perm):
        sc[p] = oc[t]
    skeys = _ravel(sc, dims)
    pos = np.searchsorted(np.asarray(keys_in, dtype=np.int64), skeys)
    assert np.all(np.asarray(keys_in)[pos] == skeys)
    return pos.astype(np.uint32)


def closed_form_2d5_transposed(n):
    """5-point Laplacian, perm (0,2,1,3): output tensor B[x, x', y, y'] = A[x, y, x', y'].
    Enumerate x, x' in {x-1, x, x+1}, y, y' (y' = y unless x' = x) in output order."""
    K, V = [], []
    for x in range(n):
        for xp in (x - 1, x, x + 1):
            if not 0 <= xp < n:
                continue
            for y in range(n):
                yps = (y - 1, y, y + 1) if xp == x else (y,)
                for yp in yps:
                    if not 0 <= yp < n:
                        continue
                    K.append(((x * n + xp) * n + y) * n + yp)
                    V.append(-4.0 if (xp == x and yp == y) else 1.0)
    return np.array(K, dtype=np.uint64), np.array(V)


_BIHARM = {(0, 0): 20.0, (1, 0): -8.0, (-1, 0): -8.0, (0, 1): -8.0, (0, -1): -8.0,
           (1, 1): 2.0, (1, -1): 2.0, (-1, 1): 2.0, (-1, -1): 2.0,
           (2, 0): 1.0, (-2, 0): 1.0, (0, 2): 1.0, (0, -2): 1.0}


def closed_form_2d13_swapped(n):
    """13-point biharmonic, perm (1,0,2,3): B[y, x, x', y'] = A[x, y, x', y'].
    Enumerate y, x, then the stencil neighbours sorted by (x', y')."""
    offs = sorted(_BIHARM)
    K, V = [], []
    for y in range(n):
        for x in range(n):
            for dx, dy in offs:
                xp, yp = x + dx, y + dy
                if 0 <= xp < n and 0 <= yp < n:
                    K.append(((y * n + x) * n + xp) * n + yp)
                    V.append(_BIHARM[(dx, dy)])
    return np.array(K, dtype=np.uint64), np.array(V)


def certificate(keys_in, vals_in, dims, perm, keys_out, vals_out, perm_out, reencode):
    """(i) perm_out is a bijection, (ii) keys_out[i] = reencode(keys_in[perm_out[i]]),
    (iii) vals_out[i] == vals_in[perm_out[i]] bitwise, (iv) keys_out strictly
    increasing.  With unique keys these imply equality with the oracle's output."""
    n = len(keys_in)
    p = np.asarray(perm_out, dtype=np.int64)
    assert len(keys_out) == n and len(p) == n
    assert np.array_equal(np.sort(p), np.arange(n)), "perm_out is not a bijection"
    assert np.array_equal(np.asarray(keys_out, dtype=np.uint64),
                          reencode(np.asarray(keys_in, dtype=np.uint64)[p]))
    assert np.array_equal(np.asarray(vals_out).view(np.uint64),
                          np.asarray(vals_in)[p].view(np.uint64))
    ko = np.asarray(keys_out, dtype=np.uint64)
    assert np.all(ko[1:] > ko[:-1]), "keys_out not strictly increasing"


def reencode_np(dims, perm):
    """Key re-encoding via numpy's unravel_index / ravel_multi_index (library routines,
    independent of the oracle's div/mod/Horner code)."""
    dims = [int(d) for d in dims]
    ndims = tuple(dims[p] for p in perm)

    def f(keys):
        c = np.unravel_index(np.asarray(keys, dtype=np.int64), tuple(dims))
        return np.ravel_multi_index(tuple(c[p] for p in perm), ndims).astype(np.uint64)
    return f
