"""Seeded synthetic inputs for the LCO permutation path (BASELINE.json configs C1-C5).

This module is shared by the oracle tests, the GPU parity tests, ``smoke()`` and
``bench.py``.  It holds none of the method's arithmetic (no decode / re-encode /
sort under a permutation): it only draws random keys and builds stencil operator
tensors directly in their canonical (input) order.  Recipes: DESIGN.md "Inputs".

Everything runs in torch int64 / float64 so the same code generates on CPU or on a
GPU; integer streams are bit-identical across devices.  Keys are stored as int64
(every key is < 2^63), the library reads them as uint64.

Random numbers: counter-based SplitMix64, ``x_i = mix(mix(seed) + (i+1)*phi)``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

_PHI = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK64 = (1 << 64) - 1


def _s64(c: int) -> int:
    """uint64 constant -> the int64 with the same bits."""
    c &= _MASK64
    return c - (1 << 64) if c >= (1 << 63) else c


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def _mix(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _srl(z, 30)) * _s64(_M1)
    z = (z ^ _srl(z, 27)) * _s64(_M2)
    return z ^ _srl(z, 31)


def _mix_int(z: int) -> int:
    z &= _MASK64
    z = ((z ^ (z >> 30)) * _M1) & _MASK64
    z = ((z ^ (z >> 27)) * _M2) & _MASK64
    return z ^ (z >> 31)


def splitmix(seed: int, stream: int, start: int, count: int, device="cpu") -> torch.Tensor:
    """count 64-bit draws (as int64 bit patterns) of stream `stream`, counters start.."""
    base = _mix_int(_mix_int(seed) ^ (stream * 0x632BE59BD9B4E019))
    i = torch.arange(start + 1, start + count + 1, dtype=torch.int64, device=device)
    return _mix(i * _s64(_PHI) + _s64(base))


def uniform_keys(seed, start, count, key_range, device="cpu") -> torch.Tensor:
    """Uniform integers in [0, key_range).  Power-of-two ranges take the top bits;
    other ranges reduce the top 63 bits modulo key_range (bias <= key_range/2^63)."""
    r = splitmix(seed, 1, start, count, device)
    if key_range & (key_range - 1) == 0:
        b = key_range.bit_length() - 1
        return _srl(r, 64 - b) if b > 0 else torch.zeros_like(r)
    return _srl(r, 1) % key_range


def uniform_values(seed, count, device="cpu") -> torch.Tensor:
    """U[-1, 1) fp64 with 52 random bits (exact on every device)."""
    r = _srl(splitmix(seed, 2, 0, count, device), 12)
    return r.to(torch.float64) * (2.0 ** -51) - 1.0


def normal_values(seed, count, device="cpu") -> torch.Tensor:
    """N(0,1) fp64 by Box-Muller (transcendentals may differ in the last bit across
    devices; values are only moved by the method, never computed on)."""
    u1 = (_srl(splitmix(seed, 3, 0, count, device), 11).to(torch.float64) + 1.0) * (2.0 ** -53)
    u2 = _srl(splitmix(seed, 4, 0, count, device), 11).to(torch.float64) * (2.0 ** -53)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * torch.pi * u2)


def random_tensor(dims, nnz, seed, values="uniform", device="cpu"):
    """nnz unique keys uniform in [0, prod dims), sorted ascending, plus values.

    Dedup: the key set is the distinct values among the first M
    draws, M the smallest count giving nnz distinct keys."""
    total = 1
    for d in dims:
        total *= int(d)
    if nnz > total:
        raise ValueError("nnz exceeds the number of coordinates")
    drawn = 0
    keys = torch.empty(0, dtype=torch.int64, device=device)
    while keys.numel() < nnz:
        need = nnz - keys.numel()
        fresh = uniform_keys(seed, drawn, need, total, device)
        drawn += need
        keys = torch.unique(torch.cat([keys, fresh]), sorted=True)
    if values == "uniform":
        vals = uniform_values(seed, nnz, device)
    elif values == "normal":
        vals = normal_values(seed, nnz, device)
    else:
        raise ValueError(values)
    return keys, vals


def _stencil(n, ndim, offsets, device):
    """Operator tensor of a constant-coefficient stencil on an n^ndim grid with
    Dirichlet truncation (out-of-grid neighbours dropped).  Modes are
    (grid coords, neighbour coords); offsets must be listed in increasing
    lexicographic order so that the keys come out sorted."""
    grid = torch.arange(n ** ndim, dtype=torch.int64, device=device)
    coords = []
    rem = grid
    for _ in range(ndim):
        coords.append(rem % n)
        rem = rem // n
    coords = coords[::-1]  # row-major: first axis most significant
    keys, vals = [], []
    for off, coef in offsets:
        ok = torch.ones_like(grid, dtype=torch.bool)
        nb = []
        for a in range(ndim):
            c = coords[a] + off[a]
            ok &= (c >= 0) & (c < n)
            nb.append(c)
        k = grid.clone()
        for a in range(ndim):
            k = k * n + nb[a]
        keys.append(torch.where(ok, k, torch.full_like(k, -1)))
        vals.append(torch.full(grid.shape, float(coef), dtype=torch.float64, device=device))
    K = torch.stack(keys, 1).reshape(-1)
    V = torch.stack(vals, 1).reshape(-1)
    keep = K >= 0
    return K[keep].contiguous(), V[keep].contiguous()


def laplacian_2d5(n, device="cpu"):
    """2-D 5-point Laplacian (-4 centre, +1 neighbours), modes (x, y, x', y')."""
    offs = [((-1, 0), 1), ((0, -1), 1), ((0, 0), -4), ((0, 1), 1), ((1, 0), 1)]
    return _stencil(n, 2, offs, device)


def laplacian_3d7(n, device="cpu"):
    """3-D 7-point Laplacian (-6 centre, +1 neighbours), modes (x,y,z,x',y',z')."""
    offs = [((-1, 0, 0), 1), ((0, -1, 0), 1), ((0, 0, -1), 1), ((0, 0, 0), -6),
            ((0, 0, 1), 1), ((0, 1, 0), 1), ((1, 0, 0), 1)]
    return _stencil(n, 3, offs, device)


def biharmonic_2d13(n, device="cpu"):
    """2-D 13-point biharmonic (20 centre, -8 axis-1, 2 diagonal, 1 axis-2)."""
    offs = [((-2, 0), 1), ((-1, -1), 2), ((-1, 0), -8), ((-1, 1), 2), ((0, -2), 1),
            ((0, -1), -8), ((0, 0), 20), ((0, 1), -8), ((0, 2), 1), ((1, -1), 2),
            ((1, 0), -8), ((1, 1), 2), ((2, 0), 1)]
    return _stencil(n, 2, offs, device)


def combinatorial_laplacian(n, device="cpu"):
    """Support pattern of the order-4 combinatorial Laplacian of PAPER.md Eq (2.3),
    a_ijkl = d(y)_ii' delta_jl d(y)_i'k + d(x)_jj' delta_ik d(x)_j'l, with d the
    central-difference FD matrix of Eq (2.1): d.d couples offsets {-2, 0, +2}, so each
    (i, j) has the neighbours (i+-2, j), (i, j+-2) and itself (5 N^2 nonzeros in the
    interior).  Built in sorted order with Dirichlet truncation (the one-sided boundary
    rows of Eq 2.1 change only the values near the edges; values are only moved)."""
    offs = [((-2, 0), 0.25), ((0, -2), 0.25), ((0, 0), -1.0), ((0, 2), 0.25), ((2, 0), 0.25)]
    return _stencil(n, 2, offs, device)


def eq23_term(n, device="cpu"):
    """One of the two terms of PAPER.md Eq (2.3) as stored after its product: the
    d(y) d(y) term c^(y)_{ijkl} = d(y)_ii' delta_jl d(y)_i'k couples (i, j) to
    (i + {-2, 0, 2}, j) with the coefficients of d.d (d the central difference of Eq 2.1):
    1/4, -1/2, 1/4.  The d(x) term in its own index order (j, i, l, k) has the same
    layout, so both operands of the paper's addition come from this generator, and
    term + permute(term, {1,0,3,2}) is the combinatorial Laplacian (same support and
    coefficients as combinatorial_laplacian)."""
    offs = [((-2, 0), 0.25), ((0, 0), -0.5), ((2, 0), 0.25)]
    return _stencil(n, 2, offs, device)


def fill_tensor(n, fill, seed, device="cpu"):
    """Order-4 n^4 tensor with a constant fill factor (PAPER.md:261 '2% fill')."""
    return random_tensor((n,) * 4, int(round(fill * n ** 4)), seed, "uniform", device)


@dataclass
class Workload:
    name: str
    dims: tuple
    perms: list
    keys: torch.Tensor
    vals: torch.Tensor
    recipe: str
    extra: dict = field(default_factory=dict)


def config(name: str, device="cpu", scale: int | None = None) -> Workload:
    """BASELINE.json configs.  `scale` shrinks the grid / nnz for fast tests while
    keeping the structure (None = full size)."""
    if name == "C1":
        dims = (64, 48, 32)
        nnz = 5000 if scale is None else scale
        k, v = random_tensor(dims, nnz, seed=1, values="uniform", device=device)
        return Workload(name, dims, [(2, 0, 1)], k, v,
                        f"64x48x32, {nnz} unique uniform keys, U[-1,1) values, seed 1")
    if name == "C2":
        n = 512 if scale is None else scale
        k, v = laplacian_2d5(n, device)
        return Workload(name, (n,) * 4, [(2, 3, 0, 1), (0, 2, 1, 3)], k, v,
                        f"2-D 5-point Laplacian operator on {n}x{n}, Dirichlet truncation")
    if name == "C3":
        n = 128 if scale is None else scale
        k, v = laplacian_3d7(n, device)
        return Workload(name, (n,) * 6, [(3, 4, 5, 0, 1, 2), (0, 3, 1, 4, 2, 5)], k, v,
                        f"3-D 7-point Laplacian operator on {n}^3, Dirichlet truncation")
    if name == "C4":
        n = 2048 if scale is None else scale
        k, v = biharmonic_2d13(n, device)
        return Workload(name, (n,) * 4, [(1, 0, 2, 3)], k, v,
                        f"2-D 13-point biharmonic operator on {n}x{n}, Dirichlet truncation")
    if name == "C5":
        dims = (4096,) * 5
        nnz = 500_000_000 if scale is None else scale
        k, v = random_tensor(dims, nnz, seed=5, values="normal", device=device)
        return Workload(name, dims, [(4, 3, 2, 1, 0)], k, v,
                        f"4096^5, {nnz} unique uniform keys in [0,2^60), N(0,1) values, seed 5")
    raise ValueError(name)
