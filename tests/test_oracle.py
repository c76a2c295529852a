"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names the passage it pins.  A plausible mistake in the oracle (dropped
term, wrong sign or index, transposed operand, unstable sort, wrong tie rule) fails
at least one of: the paper's worked example (Table 1), the Fig 3 classification and
plan constants, dense brute-force transposes over every permutation of orders 1-5,
closed forms of the stencil operators, the round-trip invariant, and the
duplicate-key stability case.
"""
import itertools
import os

import numpy as np
import pytest

import oracle
import workloads
from tests import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _table(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                rows.append([int(x) for x in line.split()])
    return np.array(rows, dtype=np.int64)


def paper_lex_to_perm(lex):
    """Paper lex order (least significant first) -> row-major torch perm,
    relabelling paper index mu as row-major mode N-1-mu (reading R1)."""
    n = len(lex)
    return tuple(n - 1 - lex[n - 1 - t] for t in range(n))


# ---------------------------------------------------------------- worked examples
def test_table1_linearize():
    """PAPER.md:155-169 Table 1: {i,j,k} -> LIV with LIV = i + 4(j + 4k)."""
    t = _table("table1_lco.txt")
    for i, j, k, liv in t:
        # row-major modes (k, j, i): mode 0 most significant
        assert oracle.linearize([4, 4, 4], [k, j, i]) == liv
        assert oracle.delinearize([4, 4, 4], liv) == [k, j, i]


def test_table1_reversed_permutation():
    """Table 1 tensor permuted to lex {2,1,0}; SPEC.md:88 (18 -> 33) + hand derivation."""
    t = _table("table1_lco.txt")
    exp = _table("table1_reversed.txt")
    keys = t[:, 3].astype(np.uint64)
    vals = np.arange(1.0, 7.0)
    perm = paper_lex_to_perm((2, 1, 0))
    assert perm == (2, 1, 0)
    assert oracle.shuffle([4, 4, 4], perm, [18])[0] == 33
    for fn in (oracle.permute, oracle.rp_permute):
        ko, vo, po = fn([4, 4, 4], perm, keys, vals)
        assert ko.tolist() == exp[:, 1].tolist()
        assert po.tolist() == exp[:, 2].tolist()
        assert vo.tolist() == vals[exp[:, 2]].tolist()


def test_fig3_classification():
    """PAPER.md:243 Fig 3: a_ijk 10x3x2, {0,1,2} -> {1,0,2}: i is a rearrangement
    index, j and k are resting; the final index is always resting."""
    perm = paper_lex_to_perm((1, 0, 2))
    assert perm == (0, 2, 1)  # row-major modes (k, j, i) -> (k, i, j)
    assert oracle.classify(perm) == [0, 1, 0]  # new positions: k resting, i rearr, j resting
    for n in range(1, 7):
        for p in itertools.permutations(range(n)):
            c = oracle.classify(p)
            assert c[-1] == 0
            # crossing rule == "not a suffix minimum"
            assert c == [int(p[t] != min(p[t:])) for t in range(n)]


def test_fig3_rp_regions_and_shaved_key():
    """regions of constant k via LIV div (n_j n_i = 30); inside a region
    the shaved key (LIV' mod 30) div 3 equals i.  Checked on the full dense 10x3x2
    tensor and a random sparse one against brute force."""
    dims = (2, 3, 10)  # row-major (k, j, i)
    perm = (0, 2, 1)
    keys = np.arange(60, dtype=np.uint64)
    new = oracle.shuffle(dims, perm, keys)
    k, j, i = np.unravel_index(keys.astype(np.int64), dims)
    assert np.array_equal(keys // 30, k)
    assert np.array_equal((new % 30) // 3, i)
    rng = np.random.default_rng(3)
    sk = np.sort(rng.choice(60, 25, replace=False)).astype(np.uint64)
    sv = rng.standard_normal(25)
    ek, ev, ep = brute.dense_permute(dims, perm, sk, sv)
    ko, vo, po = oracle.rp_permute(dims, perm, sk, sv)
    assert np.array_equal(ko, ek) and np.array_equal(po, ep) and np.array_equal(vo, ev)


def test_table2_key_modes():
    """PAPER.md:283-289 Table 2: RP's speed tracks how many indices it must rearrange.
    Min {1,0,2,3} rearranges only one index; Median {2,1,3,0} and Max {3,1,2,0} more."""
    r = {name: sum(oracle.classify(paper_lex_to_perm(lex)))
         for name, lex in {"max": (3, 1, 2, 0), "median": (2, 1, 3, 0),
                           "min": (1, 0, 2, 3)}.items()}
    assert r["min"] == 1
    assert r["median"] >= 2 and r["max"] >= 2


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("order", [1, 2, 3, 4, 5])
def test_dense_bruteforce_all_perms(order):
    """Every permutation of orders 1-5 on random shapes (incl. size-1 modes and
    non-powers of two) vs numpy dense transposes (SURVEY.md §8(c) pin 4)."""
    rng = np.random.default_rng(100 + order)
    for trial in range(3):
        dims = tuple(int(x) for x in rng.integers(1, 7 if order < 5 else 5, order))
        total = int(np.prod(dims))
        nnz = int(rng.integers(0, total + 1))
        keys = np.sort(rng.choice(total, nnz, replace=False)).astype(np.uint64)
        vals = rng.standard_normal(nnz)
        for perm in itertools.permutations(range(order)):
            ek, ev, ep = brute.dense_permute(dims, perm, keys, vals)
            for fn in (oracle.permute, oracle.rp_permute):
                ko, vo, po = fn(dims, perm, keys, vals)
                assert np.array_equal(ko, ek), (dims, perm)
                assert np.array_equal(po, ep), (dims, perm)
                assert np.array_equal(vo.view(np.uint64), ev.view(np.uint64))


def test_idx_in_passthrough():
    """perm_out reports idx_in[pi(j)] when an input index vector is given (C4 reading)."""
    rng = np.random.default_rng(7)
    keys = np.sort(rng.choice(4 ** 4, 60, replace=False)).astype(np.uint64)
    idx = (rng.permutation(60) + 1000).astype(np.uint32)
    ko, vo, po = oracle.permute((4, 4, 4, 4), (3, 1, 0, 2), keys, None, idx)
    ek, _, ep = brute.dense_permute((4, 4, 4, 4), (3, 1, 0, 2), keys, np.zeros(60))
    assert np.array_equal(ko, ek) and np.array_equal(po, idx[ep])


# ---------------------------------------------------------------- closed forms
def test_closed_form_symmetric_transpose():
    """C2a / C3a: the Laplacian operators are symmetric, so (2,3,0,1) and (3,4,5,0,1,2)
    return the input keys and values (SURVEY.md §8(c) pin 3)."""
    for w, perm in ((workloads.config("C2", scale=9), (2, 3, 0, 1)),
                    (workloads.config("C3", scale=5), (3, 4, 5, 0, 1, 2))):
        keys, vals = w.keys.numpy().astype(np.uint64), w.vals.numpy()
        ko, vo, po = oracle.permute(w.dims, perm, keys, vals)
        assert np.array_equal(ko, keys) and np.array_equal(vo, vals)
        assert np.array_equal(po, brute.source_positions(keys, w.dims, perm, ko))


def test_closed_form_c2b_c4():
    """C2b (0,2,1,3) and C4 (1,0,2,3) output enumerated directly in output order."""
    w = workloads.config("C2", scale=11)
    keys, vals = w.keys.numpy().astype(np.uint64), w.vals.numpy()
    ek, ev = brute.closed_form_2d5_transposed(11)
    ko, vo, po = oracle.permute(w.dims, (0, 2, 1, 3), keys, vals)
    assert np.array_equal(ko, ek) and np.array_equal(vo, ev)
    assert np.array_equal(po, brute.source_positions(keys, w.dims, (0, 2, 1, 3), ko))
    w = workloads.config("C4", scale=12)
    keys, vals = w.keys.numpy().astype(np.uint64), w.vals.numpy()
    ek, ev = brute.closed_form_2d13_swapped(12)
    ko, vo, po = oracle.rp_permute(w.dims, (1, 0, 2, 3), keys, vals)
    assert np.array_equal(ko, ek) and np.array_equal(vo, ev)


def test_stencil_nnz_counts():
    """Exact nnz of the truncated stencils."""
    assert workloads.config("C2", scale=64).keys.numel() == 5 * 64 ** 2 - 4 * 64
    assert workloads.config("C3", scale=16).keys.numel() == 7 * 16 ** 3 - 6 * 16 ** 2
    assert workloads.config("C4", scale=40).keys.numel() == 13 * 40 ** 2 - (20 * 40 - 4)


# ---------------------------------------------------------------- invariants
def test_roundtrip_and_certificate():
    """permute(p) then permute(p^-1) is the identity with composed perm = iota
    (SPEC.md:207); the certificate holds (SURVEY.md §8(c) pins 5, 6)."""
    w = workloads.config("C1")
    keys, vals = w.keys.numpy().astype(np.uint64), w.vals.numpy()
    perm = (2, 0, 1)
    ko, vo, po = oracle.permute(w.dims, perm, keys, vals)
    brute.certificate(keys, vals, w.dims, perm, ko, vo, po, brute.reencode_np(w.dims, perm))
    ndims = [w.dims[p] for p in perm]
    inv = tuple(int(x) for x in np.argsort(perm))
    k2, v2, p2 = oracle.permute(ndims, inv, ko, vo)
    assert np.array_equal(k2, keys) and np.array_equal(v2, vals)
    assert np.array_equal(po[p2], np.arange(len(keys)))


def test_sort_stability_with_duplicates():
    """Unsorted input with duplicate keys: ties keep input order, which
    is Python's stable sorted() on the re-encoded keys."""
    rng = np.random.default_rng(11)
    dims, perm = (5, 7, 3), (1, 2, 0)
    keys = rng.integers(0, 105, 400).astype(np.uint64)
    vals = rng.standard_normal(400)
    new = brute.reencode_np(dims, perm)(keys)
    order = sorted(range(400), key=lambda i: int(new[i]))
    ko, vo, po = oracle.sort(dims, perm, keys, vals)
    assert po.tolist() == order
    assert np.array_equal(ko, new[order]) and np.array_equal(vo, vals[order])


def test_partition_matches_bruteforce():
    rng = np.random.default_rng(5)
    dims, perm = (8, 8, 8), (2, 1, 0)
    keys = np.sort(rng.choice(512, 200, replace=False)).astype(np.uint64)
    vals = rng.standard_normal(200)
    spl = np.array([100, 300, 301], dtype=np.uint64)
    sk, sv, si, cnt = oracle.partition(dims, perm, keys, vals, 77, spl)
    new = brute.reencode_np(dims, perm)(keys)
    dest = np.searchsorted(spl, new, side="right")
    order = np.argsort(dest, kind="stable")
    assert np.array_equal(sk, keys[order]) and np.array_equal(si, order + 77)
    assert np.array_equal(sv, vals[order])
    assert cnt.tolist() == np.bincount(dest, minlength=4).tolist()


def test_errors():
    with pytest.raises(ValueError):
        oracle.permute((2 ** 32, 2 ** 32), (1, 0), [0])  # product > 2^63-1
    with pytest.raises(ValueError):
        oracle.permute((4, 4), (0, 0), [0])  # not a bijection
    with pytest.raises(ValueError):
        oracle.permute((4, 4), (1, 0), [16])  # key out of range
    with pytest.raises(ValueError):
        oracle.rp_permute((4, 4), (1, 0), [3, 2])  # RP precondition: sorted input
    ko, vo, po = oracle.permute((4, 4), (1, 0), np.zeros(0, np.uint64), np.zeros(0))
    assert len(ko) == 0


# ------------------------------------------------------------------ all-cores oracle
def test_parallel_oracle_dense_bruteforce():
    """oracle.permute_par (the same definition on all cores) vs numpy
    dense transposes over every permutation of order 4."""
    rng = np.random.default_rng(404)
    dims = (3, 5, 4, 6)
    total = int(np.prod(dims))
    keys = np.sort(rng.choice(total, 200, replace=False)).astype(np.uint64)
    vals = rng.standard_normal(200)
    for perm in itertools.permutations(range(4)):
        ek, ev, ep = brute.dense_permute(dims, perm, keys, vals)
        ko, vo, po = oracle.permute_par(dims, perm, keys, vals)
        assert np.array_equal(ko, ek) and np.array_equal(po, ep), perm
        assert np.array_equal(vo.view(np.uint64), ev.view(np.uint64))


def test_parallel_oracle_stable_on_duplicates_large():
    """Large enough that libstdc++'s parallel mergesort engages: ties keep input order
    (PAPER.md:245), i.e. numpy's stable argsort of the re-encoded keys."""
    rng = np.random.default_rng(405)
    dims, perm = (64, 64, 64), (2, 0, 1)
    n = 400_000
    keys = rng.integers(0, 64 ** 3, n).astype(np.uint64)
    vals = rng.standard_normal(n)
    idx = rng.permutation(n).astype(np.uint32)
    new = brute.reencode_np(dims, perm)(keys)
    order = np.argsort(new, kind="stable")
    ko, vo, po = oracle.permute_par(dims, perm, keys, vals, idx)
    assert np.array_equal(ko, new[order]) and np.array_equal(po, idx[order])
    assert np.array_equal(vo, vals[order])
    assert oracle.par_threads() >= 1
    with pytest.raises(ValueError):
        oracle.permute_par((4, 4), (1, 0), [16])


# ------------------------------------------------------------------ index-matched addition
def test_add_self_negation_keeps_explicit_zeros():
    """t + (-1) t over the identity match: t's support with +0.0 everywhere (SPEC add:
    explicit zeros retained)."""
    w = workloads.config("C1")
    k, v = w.keys.numpy().astype(np.uint64), w.vals.numpy()
    kc, vc = oracle.add(w.dims, tuple(range(len(w.dims))), k, v, k, v, -1.0)
    assert np.array_equal(kc, k)
    assert np.array_equal(vc.view(np.uint64), np.zeros(len(k), dtype=np.uint64))


def test_add_disjoint_supports_concatenate():
    rng = np.random.default_rng(3)
    dims = (7, 9, 11)
    total = int(np.prod(dims))
    keys = rng.choice(total, 300, replace=False)
    ka, kb = np.sort(keys[:120]).astype(np.uint64), keys[120:]
    perm = (2, 0, 1)
    # B given in its own order: invert the match on B's keys so that permute(B) = kb
    inv = tuple(int(x) for x in np.argsort(perm))
    dims_b = tuple(dims[i] for i in inv)
    kb_own = np.sort(oracle.shuffle(dims, inv, kb.astype(np.uint64)))
    va, vb = rng.standard_normal(120), rng.standard_normal(180)
    kc, vc = oracle.add(dims_b, perm, ka, va, kb_own, vb, 1.0)
    assert len(kc) == 300 and np.array_equal(kc, np.sort(keys).astype(np.uint64))
    assert bool(np.all(np.diff(kc.astype(np.int64)) > 0))


@pytest.mark.parametrize("order", [2, 3, 4])
def test_add_dense_bruteforce(order):
    """Dense oracle: C = A + s * transpose(B, match) on dense arrays; C's support is the
    union of the supports (explicit zeros where values cancel), values match exactly."""
    rng = np.random.default_rng(40 + order)
    for match in itertools.permutations(range(order)):
        dims_b = tuple(int(x) for x in rng.integers(1, 6, order))
        dims_a = tuple(dims_b[m] for m in match)
        B = np.where(rng.random(dims_b) < 0.4, rng.integers(-3, 4, dims_b).astype(float), 0.0)
        A = np.where(rng.random(dims_a) < 0.4, rng.integers(-3, 4, dims_a).astype(float), 0.0)
        Bm = np.zeros(dims_b, dtype=bool)
        Bm[B != 0] = True
        Am = A != 0
        sign = -1.0 if order % 2 else 1.0
        ka = np.flatnonzero(Am).astype(np.uint64)
        kb = np.flatnonzero(Bm).astype(np.uint64)
        kc, vc = oracle.add(dims_b, match, ka, A.ravel()[ka], kb, B.ravel()[kb], sign)
        dense = A + sign * np.transpose(B, match)
        support = Am | np.transpose(Bm, match)
        assert np.array_equal(kc, np.flatnonzero(support).astype(np.uint64)), (dims_b, match)
        assert np.array_equal(vc, dense.ravel()[kc])


def test_add_laplacian_axis_swap_doubles():
    """Closed form: the 2-D 5-point Laplacian operator (modes x, y, x', y') is symmetric
    under swapping the axes, so with the paper's addition match {1,0,3,2}
    A + permute(A) = 2A exactly, keys unchanged."""
    w = workloads.config("C2", scale=12)
    k, v = w.keys.numpy().astype(np.uint64), w.vals.numpy()
    perm = paper_lex_to_perm((1, 0, 3, 2))
    assert perm == (1, 0, 3, 2)
    kc, vc = oracle.add(w.dims, perm, k, v, k, v, 1.0)
    assert np.array_equal(kc, k) and np.array_equal(vc, 2.0 * v)


def test_add_eq23_assembly():
    """SPEC add example (Eq 2.3, :212-214): the two d.d terms, one re-sorted into
    the {1,0,3,2} order and added, give the combinatorial Laplacian a_ijkl (support of
    5 neighbours per (i, j), diagonal -1/2 - 1/2 = -1, off-diagonal 1/4)."""
    for n in (6, 9):
        k, v = workloads.eq23_term(n)
        k, v = k.numpy().astype(np.uint64), v.numpy()
        kc, vc = oracle.add((n,) * 4, (1, 0, 3, 2), k, v, k, v, 1.0)
        ek, ev = workloads.combinatorial_laplacian(n)
        assert np.array_equal(kc, ek.numpy().astype(np.uint64))
        assert np.array_equal(vc, ev.numpy())


# ------------------------------------------------------------------ matrix datatypes
def test_compress_matches_scipy():
    """CSR / DCSR of a row-major LCO matrix vs scipy.sparse (library routine)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(5)
    for m, n, nnz in ((50, 70, 400), (1000, 30, 200), (7, 9, 0), (1, 1, 1)):
        keys = np.sort(rng.choice(m * n, nnz, replace=False)).astype(np.uint64)
        rows, cols = keys // n, keys % n
        ref = sp.csr_matrix((np.ones(nnz), (rows, cols)), shape=(m, n))
        ptr, minor = oracle.compress(keys, m, n)
        assert np.array_equal(ptr, ref.indptr) and np.array_equal(minor, ref.indices)
        ids, dptr, dminor = oracle.compress(keys, m, n, doubly=True)
        nonempty = np.flatnonzero(np.diff(ref.indptr))
        assert np.array_equal(ids, nonempty) and np.array_equal(dminor, ref.indices)
        assert np.array_equal(dptr, np.append(ref.indptr[nonempty], nnz))


def test_compress_fig5a_diagonal():
    """PAPER.md Fig 5(a): a 10^4 diagonal tensor flattened with rows {i, j}, cols {k, l} is
    a 100 x 100 matrix with 10 nonzeros on a stride-11 diagonal (index-sparse); its DCSR
    holds the 10 present rows only."""
    keys = np.array([i * 1111 for i in range(10)], dtype=np.uint64)  # (i, i, i, i)
    ids, ptr, minor = oracle.compress(keys, 100, 100, doubly=True)
    assert list(ids) == [11 * i for i in range(10)] and list(minor) == [11 * i for i in range(10)]
    assert list(ptr) == list(range(11))
    ptr1, _ = oracle.compress(keys, 100, 100)
    assert len(ptr1) == 101 and ptr1[-1] == 10


def test_sparsity_classes_and_mdt_table():
    """SPEC classify examples and the paper's multiplication table (PAPER.md :340-352,
    transcribed here cell by cell) through the library's host functions."""
    import paper_1802_02619_b200 as lco
    assert lco.sparsity_class(100, 100, 10) == "index-sparse"
    assert lco.sparsity_class(10 ** 4, 10, 10 ** 3) == "row-sparse"
    assert lco.sparsity_class(100, 100, 5000) == "sparse"
    assert lco.sparsity_class(10, 10 ** 4, 10 ** 3) == "column-sparse"
    assert lco.sparsity_class(5, 5, 0) == "sparse"
    paper = {  # A \\ B: sparse, row-sparse, column-sparse, index-sparse
        "sparse": ["CSC/CSR", "CSC", "CSC", "CSC"],
        "column-sparse": ["CSR", "DCSC/DCSR", "DCSC", "DCSC"],
        "row-sparse": ["CSR", "DCSR", "CSCNA/CSRNA", "CSCNA"],
        "index-sparse": ["CSR", "DCSR", "CSRNA", "SOP"],
    }
    cols = ["sparse", "row-sparse", "column-sparse", "index-sparse"]
    for a, row in paper.items():
        for b, want in zip(cols, row):
            assert lco.mdt_choice(a, b) == want, (a, b)
