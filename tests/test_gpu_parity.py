"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Keys and the permutation vector must be identical; values are compared as 64-bit
patterns (they are moved, never computed on).  Sizes span several tiles and a ragged
tail; full BASELINE sizes are checked against the oracle where it finishes in seconds
(C1-C3), and at C4/C5 scale with the certificate (perm bijection, key = re-encode of its
source, value bits, strict increase), which with unique keys implies equality with the
oracle, plus oracle re-encodes of sampled outputs.
"""
import itertools

import numpy as np
import pytest
import torch

import oracle
import paper_1802_02619_b200 as lco
import workloads
from tests import brute

pytestmark = pytest.mark.gpu

TILE = 4096


def _np_u64(t):
    return t.detach().cpu().numpy().view(np.uint64) if t.dtype == torch.int64 else \
        t.detach().cpu().numpy().astype(np.uint64)


def _dev(a, dev, shift):
    """Device copy of a; shift=1 puts it one element into a larger buffer (8-byte but not
    16-byte aligned data pointer)."""
    t = torch.as_tensor(a)
    if not shift:
        return t.to(dev)
    buf = torch.empty(len(t) + 1, dtype=t.dtype, device=dev)
    buf[1:] = t.to(dev)
    return buf[1:]


def check(dims, perm, keys, vals, idx=None, sort=False, dev="cuda:0", return_perm=True,
          hierarchical=False, shift=0):
    """Run the CUDA path and the oracle on the same inputs; compare bit-exactly."""
    k = _dev(np.asarray(keys, dtype=np.uint64).view(np.int64), dev, shift)
    v = None if vals is None else _dev(np.asarray(vals, dtype=np.float64), dev, shift)
    ix = None if idx is None else torch.as_tensor(np.asarray(idx, dtype=np.uint32).view(np.int32)).to(dev)
    p = lco.plan(dims, perm, hierarchical=hierarchical)
    fn = p.sort if sort else p.permute
    ko, vo, po = fn(k, v, ix, return_perm=return_perm)
    torch.cuda.synchronize()
    ofn = oracle.sort if sort else oracle.permute
    ek, ev, ep = ofn(dims, perm, np.asarray(keys, dtype=np.uint64), vals, idx)
    assert np.array_equal(_np_u64(ko), ek), ("keys", dims, perm)
    if vals is not None:
        assert np.array_equal(vo.cpu().numpy().view(np.uint64), ev.view(np.uint64)), ("vals", dims, perm)
    if return_perm:
        assert np.array_equal(po.cpu().numpy().view(np.uint32), ep), ("perm", dims, perm)
    return ko, vo, po


def _rand_sorted(rng, dims, nnz):
    total = int(np.prod(dims))
    if total <= 4 * nnz:
        keys = np.sort(rng.choice(total, min(nnz, total), replace=False))
    else:
        keys = np.unique(rng.integers(0, total, int(nnz * 1.1), dtype=np.int64))[:nnz]
    return keys.astype(np.uint64), rng.standard_normal(len(keys))


# ------------------------------------------------------------------ random shapes
@pytest.mark.parametrize("order", [2, 3, 4, 5])
def test_all_perms_random(order, cuda_device):
    """Every permutation of orders 2-5, multi-tile with a ragged tail, non-pow2 dims."""
    rng = np.random.default_rng(10 + order)
    dims = {2: (1500, 997), 3: (120, 77, 96), 4: (37, 64, 29, 50), 5: (13, 16, 11, 9, 20)}[order]
    keys, vals = _rand_sorted(rng, dims, 3 * TILE + 1234)
    for perm in itertools.permutations(range(order)):
        check(dims, perm, keys, vals)


def test_fig2_shape_nonpow2(cuda_device):
    """Paper Fig 2 shape: order 5, N = 2^10-1 per mode, random support,
    non-power-of-two division on every mode; all 120 perms on a subsample."""
    rng = np.random.default_rng(7)
    dims = (1023,) * 5
    keys, vals = _rand_sorted(rng, dims, 40_000)
    for perm in itertools.permutations(range(5)):
        check(dims, perm, keys, vals)


def test_tile_boundaries_and_tiny(cuda_device):
    rng = np.random.default_rng(3)
    dims, perm = (64, 64, 64), (2, 0, 1)
    for nnz in (1, 2, 31, 32, 33, TILE - 1, TILE, TILE + 1, 2 * TILE, 5 * TILE + 17):
        keys, vals = _rand_sorted(rng, dims, nnz)
        check(dims, perm, keys, vals)


def test_empty(cuda_device):
    p = lco.plan((8, 8), (1, 0))
    k = torch.empty(0, dtype=torch.int64, device=cuda_device)
    v = torch.empty(0, dtype=torch.float64, device=cuda_device)
    ko, vo, po = p.permute(k, v)
    assert ko.numel() == 0 and vo.numel() == 0 and po.numel() == 0


def test_copy_paths(cuda_device):
    rng = np.random.default_rng(4)
    keys, vals = _rand_sorted(rng, (40, 1, 50), 1500)
    check((40, 1, 50), (0, 1, 2), keys, vals)   # identity
    check((40, 1, 50), (1, 0, 2), keys, vals)   # only a size-1 mode moves
    check((2000,), (0,), keys[keys < 2000], vals[keys < 2000])  # order 1


def test_options(cuda_device):
    """idx_in passthrough, keys-only, no perm output."""
    rng = np.random.default_rng(5)
    dims = (100, 90, 80)
    keys, vals = _rand_sorted(rng, dims, 3 * TILE)
    idx = rng.permutation(len(keys)).astype(np.uint32) + 7
    for perm in ((2, 1, 0), (1, 0, 2), (0, 2, 1)):
        check(dims, perm, keys, vals, idx=idx)
        check(dims, perm, keys, None)
        check(dims, perm, keys, vals, return_perm=False)


def test_max_order_and_special_values(cuda_device):
    rng = np.random.default_rng(6)
    dims = (2,) * 16
    keys, _ = _rand_sorted(rng, dims, 20_000)
    vals = np.array([np.nan, -0.0, np.inf, -np.inf, 5e-324] * 4000)[:len(keys)]
    vals[0] = np.frombuffer(np.uint64(0x7ff8dead0000beef).tobytes(), dtype=np.float64)[0]
    for perm in (tuple(range(15, -1, -1)), (1, 0) + tuple(range(2, 16)), (8,) + tuple(range(8)) + tuple(range(9, 16))):
        check(dims, perm, keys, vals)


def test_large_keys_near_limit(cuda_device):
    """prod(dims) close to 2^63-1 with non-pow2 modes."""
    rng = np.random.default_rng(8)
    dims = (3037000499, 3037000499)  # product 9223372030926249001 < 2^63-1
    keys = np.unique(rng.integers(0, 2 ** 63 - 2 ** 40, 30_000, dtype=np.int64)).astype(np.uint64)
    keys = keys[keys < dims[0] * dims[1]]
    check(dims, (1, 0), keys, rng.standard_normal(len(keys)))


# ------------------------------------------------------------------ MSD schedule
def test_msd_two_levels_random(cuda_device):
    """MSD level 1 (8 bits) + segmented level 2 + on-chip leaves (32-bit leaf keys)."""
    rng = np.random.default_rng(21)
    dims = (4096,) * 5
    keys = np.unique(rng.integers(0, 2 ** 60, 2_600_000, dtype=np.int64))[:2_500_000]
    keys = keys.astype(np.uint64)
    assert lco.plan(dims, (4, 3, 2, 1, 0)).info(len(keys))["msd_levels"] == 2
    check(dims, (4, 3, 2, 1, 0), keys, rng.standard_normal(len(keys)))
    check(dims, (3, 4, 0, 2, 1), keys, rng.standard_normal(len(keys)))


def _skewed(rng, n, hot):
    """Sorted unique keys of 4096^5 whose new-order top modes are nearly constant, so
    MSD buckets are far larger than a leaf (exercises the streaming leaf fallback)."""
    c4 = np.full(n, 7)
    c3 = np.where(rng.random(n) < hot, 9, rng.integers(0, 4096, n))
    c2 = rng.integers(0, 2, n)
    c1 = rng.integers(0, 4096, n)
    c0 = rng.integers(0, 4096, n)
    k = np.ravel_multi_index((c0, c1, c2, c3, c4), (4096,) * 5)
    return np.unique(k).astype(np.uint64)


@pytest.mark.parametrize("n", [40_000, 300_000, 3_000_000])
def test_msd_skewed_oversize_leaves(n, cuda_device):
    rng = np.random.default_rng(n)
    keys = _skewed(rng, n, 0.98)
    vals = rng.standard_normal(len(keys))
    check((4096,) * 5, (4, 3, 2, 1, 0), keys, vals)


def test_sort_msd_with_duplicates(cuda_device):
    """lco_sort of unsorted keys with many duplicates through the MSD schedule: equal
    keys keep input order."""
    rng = np.random.default_rng(31)
    dims = (4096,) * 5
    keys = rng.integers(0, 2 ** 60, 1_000_000, dtype=np.int64).astype(np.uint64)
    keys[1::3] = keys[::3][: len(keys[1::3])]  # many duplicates
    perm = (2, 0, 1, 4, 3)
    assert lco.plan(dims, perm).info(len(keys), sort=True)["path"] == "msd"
    check(dims, perm, keys, rng.standard_normal(len(keys)), sort=True)


# ------------------------------------------------------------------ lco_sort
def test_sort_unsorted_with_duplicates(cuda_device):
    rng = np.random.default_rng(9)
    dims = (50, 60, 70)
    keys = rng.integers(0, 50 * 60 * 70, 30_000).astype(np.uint64)  # duplicates likely
    vals = rng.standard_normal(len(keys))
    for perm in ((0, 1, 2), (2, 1, 0), (1, 2, 0)):
        check(dims, perm, keys, vals, sort=True)


def test_sort_equals_permute_on_sorted(cuda_device):
    rng = np.random.default_rng(12)
    dims = (64, 32, 48, 16)
    keys, vals = _rand_sorted(rng, dims, 50_000)
    for perm in ((3, 1, 2, 0), (0, 2, 1, 3)):
        a = check(dims, perm, keys, vals)
        b = check(dims, perm, keys, vals, sort=True)
        assert all(torch.equal(x, y) for x, y in zip(a, b))


# ------------------------------------------------------------------ BASELINE configs
@pytest.mark.parametrize("name,scale", [("C1", None), ("C2", 96), ("C3", 20), ("C4", 100),
                                        ("C5", 300_000), ("C5", 30_000), ("C5", 1_500)])
def test_baseline_configs_scaled(name, scale, cuda_device):
    w = workloads.config(name, scale=scale)
    for perm in w.perms:
        check(w.dims, perm, _np_u64(w.keys), w.vals.numpy())


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_baseline_full_vs_oracle(name, cuda_device):
    w = workloads.config(name)
    for perm in w.perms:
        check(w.dims, perm, _np_u64(w.keys), w.vals.numpy())


def _torch_reencode(keys, dims, perm):
    """Independent re-encode with torch // and % (test-side, not the kernels)."""
    c = []
    k = keys.clone()
    for d in reversed(dims):
        c.append(k % d)
        k = k // d
    c = c[::-1]
    out = torch.zeros_like(keys)
    for p in perm:
        out = out * dims[p] + c[p]
    return out


def certificate_gpu(w, perm, ko, vo, po):
    n = w.keys.numel()
    dev = ko.device
    kin = w.keys.to(dev)
    src = po.long()
    assert torch.equal(torch.sort(src).values, torch.arange(n, device=dev)), "perm not a bijection"
    assert torch.equal(ko, _torch_reencode(kin[src], w.dims, perm)), "key != re-encode(source)"
    assert torch.equal(vo.view(torch.int64), w.vals.to(dev)[src].view(torch.int64)), "vals"
    assert bool((ko[1:] > ko[:-1]).all()), "not strictly increasing"
    # sampled outputs re-encoded by the oracle itself
    g = torch.Generator().manual_seed(1)
    s = torch.randint(0, n, (2000,), generator=g)
    ks = _np_u64(kin[src[s.to(dev)]])
    assert np.array_equal(oracle.shuffle(w.dims, perm, ks), _np_u64(ko[s.to(dev)]))


def test_c4_full_certificate(cuda_device):
    w = workloads.config("C4", device=cuda_device)
    for perm in w.perms:
        ko, vo, po = lco.permute(w.keys, w.vals, w.dims, perm)
        torch.cuda.synchronize()
        certificate_gpu(w, perm, ko, vo, po)
        # closed form: output ordered by (y, x, x', y'); an interior row y holds 13
        # nonzeros per interior x, 9 at x in {0, n-1} and 12 at x in {1, n-2}
        n = w.dims[0]
        y = ko // (n ** 3)
        assert torch.equal(torch.bincount(y, minlength=n).cpu()[2:-2],
                           torch.full((n - 4,), 13 * n - 10, dtype=torch.int64))


def test_c5_full_certificate(cuda_device):
    w = workloads.config("C5", device=cuda_device)
    perm = w.perms[0]
    ko, vo, po = lco.permute(w.keys, w.vals, w.dims, perm)
    torch.cuda.synchronize()
    certificate_gpu(w, perm, ko, vo, po)
    del ko, vo, po
    # full-size oracle parity on a contiguous slice (itself a sorted LCO tensor)
    sl = slice(123_456_789, 123_456_789 + 3_000_000)
    ks, vs = w.keys[sl].contiguous(), w.vals[sl].contiguous()
    ko, vo, po = lco.permute(ks, vs, w.dims, perm)
    ek, ev, ep = oracle.permute(w.dims, perm, _np_u64(ks), vs.cpu().numpy())
    assert np.array_equal(_np_u64(ko), ek) and np.array_equal(po.cpu().numpy().view(np.uint32), ep)
    assert np.array_equal(vo.cpu().numpy().view(np.uint64), ev.view(np.uint64))


# ------------------------------------------------------------------ other entry points
def test_permute_host_matches_device(cuda_device):
    w = workloads.config("C2", scale=64)
    perm = w.perms[0]
    p = lco.plan(w.dims, perm)
    kh, vh = w.keys.pin_memory(), w.vals.pin_memory()
    ko, vo, po = p.permute_host(kh, vh)
    torch.cuda.synchronize()
    ek, ev, ep = oracle.permute(w.dims, perm, _np_u64(w.keys), w.vals.numpy())
    assert np.array_equal(_np_u64(ko), ek) and np.array_equal(po.numpy().view(np.uint32), ep)
    assert np.array_equal(vo.numpy().view(np.uint64), ev.view(np.uint64))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_partition_vs_oracle(world, cuda_device):
    rng = np.random.default_rng(world)
    dims, perm = (256, 128, 64), (2, 0, 1)
    keys, vals = _rand_sorted(rng, dims, 5 * TILE + 99)
    total = int(np.prod(dims))
    spl = np.sort(rng.choice(total, world - 1, replace=False)).astype(np.uint64)
    p = lco.plan(dims, perm)
    k = torch.as_tensor(keys.view(np.int64)).to(cuda_device)
    v = torch.as_tensor(vals).to(cuda_device)
    sk, sv, si, cnt = p.partition(k, v, 1000, torch.as_tensor(spl.view(np.int64)).to(cuda_device))
    ek, ev, ei, ec = oracle.partition(dims, perm, keys, vals, 1000, spl)
    assert np.array_equal(_np_u64(sk), ek) and np.array_equal(si.cpu().numpy().view(np.uint32), ei)
    assert np.array_equal(sv.cpu().numpy().view(np.uint64), ev.view(np.uint64))
    assert cnt.cpu().numpy().tolist() == ec.tolist()


def test_key_histogram(cuda_device):
    rng = np.random.default_rng(2)
    dims, perm = (100, 200, 300), (1, 2, 0)
    keys, _ = _rand_sorted(rng, dims, 50_000)
    p = lco.plan(dims, perm)
    c = p.key_histogram(torch.as_tensor(keys.view(np.int64)).to(cuda_device), 8)
    new = brute.reencode_np(dims, perm)(keys)
    kb = int(np.ceil(np.log2(100 * 200 * 300)))
    exp = np.bincount((new >> np.uint64(kb - 8)).astype(np.int64), minlength=256)
    assert c.cpu().numpy().tolist() == exp.tolist()


def test_validate_flag(cuda_device):
    p = lco.Plan((8, 8), (1, 0), validate=True)
    k = torch.tensor([3, 2, 9], dtype=torch.int64, device=cuda_device)
    with pytest.raises(ValueError, match="UNSORTED"):
        p.permute(k)
    with pytest.raises(ValueError, match="KEY_RANGE"):
        p.permute(torch.tensor([3, 64], dtype=torch.int64, device=cuda_device))
    ko, _, po = p.permute(torch.tensor([2, 3, 9], dtype=torch.int64, device=cuda_device))
    assert ko.tolist() == [9, 16, 24] and po.tolist() == [2, 0, 1]


def test_alias_rejected(cuda_device):
    p = lco.plan((8, 8), (1, 0))
    k = torch.arange(10, dtype=torch.int64, device=cuda_device)
    with pytest.raises(ValueError, match="ALIAS"):
        p.permute(k, out=(k, None, None))


def test_combinatorial_laplacian_all_perms(cuda_device):
    """PAPER.md Eq (2.3) pattern (non-power-of-two N, as P:207 and P:526 use 2^k - 1),
    all 23 permutations, permute and sort both against the oracle (Table 2 workload)."""
    k, v = workloads.combinatorial_laplacian(63)
    keys, vals = _np_u64(k), v.numpy()
    for perm in itertools.permutations(range(4)):
        check((63,) * 4, perm, keys, vals)
        check((63,) * 4, perm, keys, vals, sort=True)


# ------------------------------------------------------------------ segment-local tiles
def _prefix_tensor(rng, seg_sizes, inner_dims):
    """Sorted unique keys of (len(seg_sizes),) + inner_dims where segment s (mode 0 = s)
    holds seg_sizes[s] random nonzeros."""
    inner = int(np.prod(inner_dims))
    keys = []
    for s, m in enumerate(seg_sizes):
        m = min(m, inner)
        keys.append(s * inner + np.sort(rng.choice(inner, m, replace=False)))
    return np.concatenate(keys).astype(np.uint64)


def test_tile_path_random_segments(cuda_device):
    """Identity prefix with small segments: one on-chip sort per tile of whole segments
    (tile boundaries found by binary search on the keys), including ragged segment
    sizes, empty segments and a tail tile."""
    rng = np.random.default_rng(41)
    inner = (37, 64, 29)
    sizes = rng.integers(0, 2500, 300)
    sizes[::17] = 0
    keys = _prefix_tensor(rng, sizes, inner)
    dims = (len(sizes),) + inner
    for perm in [(0, 2, 1, 3), (0, 3, 2, 1), (0, 1, 3, 2), (0, 3, 1, 2)]:
        assert lco.plan(dims, perm).info(len(keys))["path"] == "tile", perm
        check(dims, perm, keys, rng.standard_normal(len(keys)))


def test_tile_path_oversize_segment(cuda_device):
    """A segment larger than an on-chip tile goes to the deferred streaming sort (raw
    input re-encoded on the fly), the other tiles stay on chip."""
    rng = np.random.default_rng(42)
    inner = (128, 96, 16)
    sizes = np.full(400, 300)
    sizes[123] = 60_000
    keys = _prefix_tensor(rng, sizes, inner)
    dims = (len(sizes),) + inner
    assert lco.plan(dims, (0, 3, 1, 2)).info(len(keys))["path"] == "tile"
    check(dims, (0, 3, 1, 2), keys, rng.standard_normal(len(keys)))
    check(dims, (0, 2, 3, 1), keys, None)


def test_tile_path_clustered_q(cuda_device):
    """C2b-like: thousands of nonzeros share each (prefix, middle) value; the tile sort
    takes stable radix passes on q (ties keep input order = suffix order)."""
    w = workloads.config("C2", scale=160)
    dims, perm = w.dims, (0, 2, 1, 3)
    assert lco.plan(dims, perm).info(w.keys.numel())["path"] == "tile"
    check(dims, perm, _np_u64(w.keys), w.vals.numpy())
    check(dims, perm, _np_u64(w.keys), w.vals.numpy(), return_perm=False)


@pytest.mark.parametrize("env", [{}, {"LCO_NO_LEAFS": "1"}, {"LCO_MSD_B1": "9", "LCO_MSD_B2": "9"},
                                 {"LCO_NO_LEAFR": "1"}])
def test_msd_leaf_variants(env, cuda_device, monkeypatch):
    """MSD levels with fully staged CTA leaves (default at 14M), 32-bit-key CTA leaves
    with L2 gathers (default for 1-level ~4K leaves, forced at 14M), 9+9 levels, and
    64-bit-key CTA leaves: all bit-exact."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(43)
    dims = (4096,) * 5
    for n, levels in ((14_000_000, 2), (1_000_000, 1)):
        keys = np.unique(rng.integers(0, 2 ** 60, n + n // 20, dtype=np.int64))[:n]
        keys = keys.astype(np.uint64)
        info = lco.plan(dims, (4, 3, 2, 1, 0)).info(len(keys))
        assert info["msd_levels"] == levels and info["leaf_kind"] == "cta"
        check(dims, (4, 3, 2, 1, 0), keys, rng.standard_normal(len(keys)))
        check(dims, (1, 4, 0, 3, 2), keys, None)


@pytest.mark.parametrize("env", [{}, {"LCO_SAMPLED_TEST": "1"}, {"LCO_NO_SAMPLED": "1"}])
def test_msd_sampled_level1(env, cuda_device, monkeypatch):
    """Sampled level 1 (>= 2^24 nonzeros, two unordered MSD levels): run bases from
    per-digit cursors into sampled, padded bucket capacities; LCO_SAMPLED_TEST halves the
    capacities so every run overflows and the predicated exact path redoes level 1;
    LCO_NO_SAMPLED counts exactly.  All bit-exact vs the oracle."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(97)
    dims = (4096,) * 5
    n = 17_500_000
    keys = np.unique(rng.integers(0, 2 ** 60, n + n // 20, dtype=np.int64))[:n].astype(np.uint64)
    assert lco.plan(dims, (4, 3, 2, 1, 0)).info(len(keys))["msd_levels"] == 2
    check(dims, (4, 3, 2, 1, 0), keys, rng.standard_normal(len(keys)))


# ------------------------------------------------------------------ segmented single pass
@pytest.mark.parametrize("dims,perm,nnz", [((256, 16, 64, 32), (0, 2, 1, 3), 1_000_000),
                                           ((128, 16, 2048, 4), (0, 2, 1, 3), 1_000_000),
                                           ((1000, 8, 16, 64), (0, 3, 1, 2), 5_000_000),
                                           ((128, 8, 8, 128, 8, 8), (0, 3, 1, 2, 4, 5), 1_000_000)])
def test_seg_path(dims, perm, nnz, cuda_device):
    """Identity prefix with large segments and a power-of-two middle of <= 11 bits: one
    stable pass of the middle digit inside every segment (segments found by a count of
    the prefix digit), incl. empty segments and multi-tile segments with ragged tails."""
    rng = np.random.default_rng(51)
    keys, vals = _rand_sorted(rng, dims, nnz)
    keys = keys[(keys // int(np.prod(dims[1:]))) % 5 != 3]  # some empty segments
    vals = vals[: len(keys)]
    info = lco.plan(dims, perm).info(len(keys))
    assert info["path"] == "seg", info["path"]
    check(dims, perm, keys, vals)
    check(dims, perm, keys, None, return_perm=False)


# ------------------------------------------------------------------ hierarchical plan
@pytest.mark.parametrize("order", [4, 5, 6])
def test_hierarchical_all_perms(order, cuda_device):
    """Every permutation with >= 2 runs of rearrangement indices, executed in stages
    (LCO_FLAG_HIERARCHICAL), bit-exact vs the oracle with and without
    values / permutation vector; stage paths vary with the segment sizes."""
    rng = np.random.default_rng(60 + order)
    dims = {4: (64, 64, 48, 64), 5: (24, 16, 20, 16, 24), 6: (8, 12, 8, 10, 8, 12)}[order]
    keys, vals = _rand_sorted(rng, dims, 400_000)
    seen = 0
    for perm in itertools.permutations(range(order)):
        if lco.plan(dims, perm, hierarchical=True).info(len(keys))["path"] != "hier":
            continue
        seen += 1
        check(dims, perm, keys, vals, hierarchical=True)
        if seen % 5 == 0:
            check(dims, perm, keys, None, return_perm=False, hierarchical=True)
    assert seen >= 2


def test_hierarchical_c3b_three_buffers(cuda_device):
    """C3b at full size (two stages: segmented pass, then segment-local tiles) and an
    order-6 permutation with three runs of rearrangement indices (three stages, both
    intermediate buffer sets)."""
    w = workloads.config("C3")
    perm = (0, 3, 1, 4, 2, 5)
    assert lco.plan(w.dims, perm, hierarchical=True).info(w.keys.numel())["path"] == "hier"
    check(w.dims, perm, _np_u64(w.keys), w.vals.numpy(), hierarchical=True)
    rng = np.random.default_rng(66)
    dims = (16, 16, 16, 16, 16, 16)
    keys, vals = _rand_sorted(rng, dims, 2_000_000)
    perm3 = (1, 0, 3, 2, 5, 4)
    p = lco.plan(dims, perm3, hierarchical=True)
    assert len(p.stages()) == 3 and p.info(len(keys))["path"] == "hier"
    check(dims, perm3, keys, vals, hierarchical=True)
    check(dims, perm3, keys, None, return_perm=False, hierarchical=True)
    check(dims, perm3, keys, vals)  # the flat plan of the same handle dims


# ------------------------------------------------------------------ index-matched addition
def _check_add(dims_b, match, ka, va, kb, vb, sign, dev="cuda:0"):
    t = lambda a, dt: torch.as_tensor(np.asarray(a, dtype=dt)).to(dev)
    kc, vc, m = lco.plan(dims_b, match).add(t(np.asarray(ka, np.uint64).view(np.int64), np.int64),
                                            t(va, np.float64),
                                            t(np.asarray(kb, np.uint64).view(np.int64), np.int64),
                                            t(vb, np.float64), sign)
    ek, ev = oracle.add(dims_b, match, ka, va, kb, vb, sign)
    assert m == len(ek), (m, len(ek))
    assert np.array_equal(_np_u64(kc), ek)
    assert np.array_equal(vc.cpu().numpy().view(np.uint64), ev.view(np.uint64))


@pytest.mark.parametrize("order", [3, 4])
def test_add_random_all_matches(order, cuda_device):
    """A + s * permute(B, match) for every match: overlapping supports (collisions summed,
    explicit zeros kept), several merge tiles, duplicates straddling tile boundaries."""
    rng = np.random.default_rng(70 + order)
    dims_b = {3: (40, 33, 50), 4: (12, 17, 10, 14)}[order]
    for match in itertools.permutations(range(order)):
        dims_a = tuple(dims_b[m] for m in match)
        kb, vb = _rand_sorted(rng, dims_b, 20_000)
        kbp = np.sort(oracle.shuffle(dims_b, match, kb))
        ka = np.union1d(kbp[::3], np.sort(rng.choice(int(np.prod(dims_a)), 9_000, replace=False)))
        ka = ka.astype(np.uint64)
        va = rng.standard_normal(len(ka))
        _check_add(dims_b, match, ka, va, kb, vb, 1.0 if sum(match) % 2 else -1.0)


def test_add_edge_cases(cuda_device):
    rng = np.random.default_rng(77)
    dims = (64, 48, 32)
    k, v = _rand_sorted(rng, dims, 30_000)
    _check_add(dims, (0, 1, 2), k, v, k, v, -1.0)          # t - t: explicit zeros
    _check_add(dims, (2, 0, 1), k[:0], v[:0], k, v, 1.0)   # empty A
    dims_a = (32, 64, 48)
    ka, va = _rand_sorted(rng, dims_a, 10_000)
    _check_add(dims, (2, 0, 1), ka, va, k[:0], v[:0], -1.0)  # empty B
    _check_add(dims, (2, 0, 1), ka[:1], va[:1], k[:1], v[:1], 1.0)


def test_add_laplacian_paper_match(cuda_device):
    """The paper's addition: two order-4 operator tensors, one
    re-sorted into the {1,0,3,2} order; the 5-point Laplacian is axis-swap symmetric, so
    A + permute(A) = 2A (closed form) - and vs the oracle at full C2 size."""
    w = workloads.config("C2")
    k, v = _np_u64(w.keys), w.vals.numpy()
    _check_add(w.dims, (1, 0, 3, 2), k, v, k, v, 1.0)
    kc, vc, m = lco.add(w.keys.cuda(), w.vals.cuda(), w.keys.cuda(), w.vals.cuda(), w.dims,
                        (1, 0, 3, 2))
    assert m == len(k) and torch.equal(vc.cpu(), 2.0 * w.vals)


def test_add_eq23_assembly(cuda_device):
    """Eq (2.3) assembled on the GPU: term + permute(term, {1,0,3,2}) = the combinatorial
    Laplacian (closed form), and bit-exact vs the oracle."""
    n = 300
    k, v = workloads.eq23_term(n)
    _check_add((n,) * 4, (1, 0, 3, 2), _np_u64(k), v.numpy(), _np_u64(k), v.numpy(), 1.0)
    kc, vc, m = lco.add(k.cuda(), v.cuda(), k.cuda(), v.cuda(), (n,) * 4, (1, 0, 3, 2))
    ek, ev = workloads.combinatorial_laplacian(n)
    assert torch.equal(kc.cpu(), ek) and torch.equal(vc.cpu(), ev)


# ------------------------------------------------------------------ matrix datatypes
@pytest.mark.parametrize("m,n,nnz", [(3000, 2000, 200_000), (1 << 30, 64, 300_000),
                                     (5, 7, 35), (1000, 1000, 1), (100, 100, 0)])
def test_compress_vs_oracle(m, n, nnz, cuda_device):
    """CSR and DCSR of row-major LCO matrices (tile boundaries, empty majors, a
    row-sparse matrix with 2^30 rows in DCSR form) vs the oracle, bit-exact."""
    rng = np.random.default_rng(m % 97 + nnz)
    if nnz > m * n // 2:
        keys = np.sort(rng.choice(m * n, nnz, replace=False)).astype(np.uint64)
    else:
        keys = np.unique(rng.integers(0, m * n, nnz + nnz // 10 + 2, dtype=np.int64))[:nnz]
        keys = keys.astype(np.uint64)
    k = torch.as_tensor(keys.view(np.int64)).cuda()
    ids, ptr, minor = oracle.compress(keys, m, n, doubly=True)
    d = lco.compress(k, m, n, doubly=True)
    assert d["nz"] == len(ids)
    assert np.array_equal(_np_u64(d["ids"]), ids) and np.array_equal(_np_u64(d["ptr"]), ptr)
    assert np.array_equal(_np_u64(d["minor"]), minor)
    if m <= 1 << 20:
        ptr1, minor1 = oracle.compress(keys, m, n)
        s = lco.compress(k, m, n)
        assert np.array_equal(_np_u64(s["ptr"]), ptr1) and np.array_equal(_np_u64(s["minor"]), minor1)


def test_flatten_to_csc_and_roundtrip(cuda_device):
    """Flatten a 4th-order tensor (rows {2, 0}, cols {3, 1}) column-major on the GPU and
    compress it to CSC / DCSC: equals scipy's CSC of the same matrix; flattening back
    (unflatten = the inverse permutation) returns the tensor."""
    import scipy.sparse as sp
    rng = np.random.default_rng(90)
    dims = (30, 20, 40, 25)
    keys, vals = _rand_sorted(rng, dims, 150_000)
    kt = torch.as_tensor(keys.view(np.int64)).cuda()
    vt = torch.as_tensor(vals).cuda()
    rows, cols = (2, 0), (3, 1)
    km, vm, m, n = lco.flatten(kt, vt, dims, rows, cols, major="col")
    assert (m, n) == (40 * 30, 25 * 20)
    c = np.array(np.unravel_index(keys.astype(np.int64), dims))
    r_idx = c[2] * 30 + c[0]
    c_idx = c[3] * 20 + c[1]
    ref = sp.csc_matrix((vals, (r_idx, c_idx)), shape=(m, n))
    ref.sort_indices()
    s = lco.compress(km, n, m)
    assert np.array_equal(_np_u64(s["ptr"]), ref.indptr)
    assert np.array_equal(_np_u64(s["minor"]), ref.indices)
    assert np.array_equal(vm.cpu().numpy(), ref.data)
    d = lco.compress(km, n, m, doubly=True)
    assert d["nz"] == int((np.diff(ref.indptr) > 0).sum())
    # unflatten: the column-major matrix is the tensor in mode order (3, 1, 2, 0)
    inv = tuple(int(x) for x in np.argsort((3, 1, 2, 0)))
    back, bv, _ = lco.permute(km, vm, (25, 20, 40, 30), inv, return_perm=False)
    assert torch.equal(back, kt) and torch.equal(bv, vt)


# ------------------------------------------------------------------ block transpose
@pytest.mark.parametrize("dims,perm", [((37, 41, 1000), (1, 0, 2)),
                                       ((64, 32, 16, 300), (2, 0, 1, 3)),
                                       ((50, 60, 7, 90), (1, 0, 2, 3)),
                                       ((16, 8, 12, 10, 200), (1, 2, 0, 3, 4)),
                                       ((5, 6, 1 << 20), (1, 0, 2)),
                                       ((3, 700, 9, 400), (0, 2, 1, 3)),
                                       ((20, 30, 40, 500), (2, 1, 0, 3))])
def test_block_path(dims, perm, cuda_device):
    """Permutations whose rearranged modes lie in a small old-order prefix: a transpose of
    runs without sorting (run bounds, block counts in new order, scan, one tiled copy) -
    non-power-of-two dims, empty blocks, ragged tiles at the grid edges, modes between
    and before the tile modes, blocks larger than the on-chip stage ((5, 6, 2^20): ~8K
    nonzeros per block, written straight from registers)."""
    rng = np.random.default_rng(sum(dims))
    keys, vals = _rand_sorted(rng, dims, 250_000)
    info = lco.plan(dims, perm).info(len(keys))
    assert info["path"] == "block", info["path"]
    check(dims, perm, keys, vals)
    check(dims, perm, keys, None, return_perm=False)
    idx = rng.permutation(len(keys)).astype(np.uint32)
    check(dims, perm, keys, vals, idx=idx)
    check(dims, perm, keys, vals, shift=1)  # inputs not 16-byte aligned: no TMA row copies
    w = workloads.config("C4", scale=300)
    assert lco.plan(w.dims, w.perms[0]).info(w.keys.numel())["path"] == "block"
    check(w.dims, w.perms[0], _np_u64(w.keys), w.vals.numpy())


@pytest.mark.parametrize("nnz", [20_479, 20_480, 20_481, 20_543, 20_545])
def test_block_bounds_window_edges(nnz, cuda_device):
    """k_block_bounds' 16-byte path: each warp reads 512 keys as 256 lane pairs, so the
    ragged last warp (nnz = 10 x 2,048 +- 1, odd and even tails) and block boundaries
    between the two keys of a pair or across lanes, chunks and warps must all be found;
    compared with the oracle bit-exactly, aligned (vector) and shifted (scalar path)."""
    dims, perm = (37, 41, 1000), (1, 0, 2)
    rng = np.random.default_rng(nnz)
    keys, vals = _rand_sorted(rng, dims, nnz)
    assert lco.plan(dims, perm).info(len(keys))["path"] == "block"
    check(dims, perm, keys, vals)
    check(dims, perm, keys, vals, shift=1)


# ------------------------------------------------------------------ concurrency (lco.h threading)
def test_one_handle_two_threads_two_streams(cuda_device):
    """include/lco.h: a handle may be used concurrently from several host threads on
    different streams with different workspaces.  Two threads drive one handle on two
    streams (C5-shaped MSD schedule and a C3b-shaped LSD schedule alternate), every
    result bit-exact with the oracle."""
    import threading
    rng = np.random.default_rng(99)
    dims, perm = (4096,) * 5, (4, 3, 2, 1, 0)
    keys = np.unique(rng.integers(0, 2 ** 60, 2_100_000, dtype=np.int64))[:2_000_000].astype(np.uint64)
    vals = rng.standard_normal(len(keys))
    ek, ev, ep = oracle.permute(dims, perm, keys, vals)
    p = lco.Plan(dims, perm)
    k = torch.as_tensor(keys.view(np.int64)).to(cuda_device)
    v = torch.as_tensor(vals).to(cuda_device)
    errors, results = [], {}

    def work(tid):
        try:
            st = torch.cuda.Stream(device=cuda_device)
            ws = torch.empty(p.workspace_size(len(keys)) + 256, dtype=torch.uint8, device=cuda_device)
            outs = []
            for _ in range(4):
                with torch.cuda.stream(st):
                    ko = torch.empty_like(k)
                    vo = torch.empty_like(v)
                    po = torch.empty(len(keys), dtype=torch.int32, device=cuda_device)
                p.permute(k, v, out=(ko, vo, po), workspace=ws, stream=st)
                outs.append((ko, vo, po))
            st.synchronize()
            results[tid] = outs
        except Exception as ex:  # noqa: BLE001
            errors.append(ex)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for outs in results.values():
        for ko, vo, po in outs:
            assert np.array_equal(_np_u64(ko), ek)
            assert np.array_equal(vo.cpu().numpy().view(np.uint64), ev.view(np.uint64))
            assert np.array_equal(po.cpu().numpy().view(np.uint32), ep)


# ------------------------------------------------------------------ MSD level 3 (adaptive re-split)
@pytest.mark.parametrize("perm,sort", [((3, 1, 2, 0), False), ((1, 3, 2, 0), False),
                                       ((2, 0, 3, 1), False), ((0, 2, 1, 3), True),
                                       ((3, 1, 0, 2), True)])
def test_msd_level3_laplacian_skew(perm, sort, cuda_device, monkeypatch):
    """Table 2's cliff: on the Eq (2.3) Laplacian, the level-2 digit of these permutations
    lands on modes that the stencil ties together (l in {j-1, j, j+1}), so a few level-2
    buckets hold thousands of nonzeros.  They are split again on the next 8 bits (level
    3, buffer B -> A) instead of the streaming sort; bit-exact against the oracle."""
    n = 724  # 2.6M nonzeros: two MSD levels (forced: the model picks LSD at this size)
    monkeypatch.setenv("LCO_MSD", "1")
    k, v = workloads.combinatorial_laplacian(n)
    keys, vals = _np_u64(k), v.numpy()
    info = lco.plan((n,) * 4, perm).info(len(keys), sort=sort)
    assert info["path"] == "msd" and info["msd_levels"] == 2, info
    check((n,) * 4, perm, keys, vals, sort=sort)
    check((n,) * 4, perm, keys, None, sort=sort, return_perm=False)


@pytest.mark.parametrize("nnz,one_cta", [(1, False), (100, False), (4095, False), (4097, False),
                                         (5000, False), (8192, False), (5000, True), (8192, True)])
def test_single_tile_path(nnz, one_cta, cuda_device, monkeypatch):
    """Inputs of <= 8,192 nonzeros whose disturbed digits fit 10 bits: one stable counting
    pass (C1's schedule) -- on a cluster of 8 CTAs exchanging digit counts through DSMEM
    (default), or one CTA whose tile order is the output order (LCO_SINGLE_CTA); every
    permutation of an order-3 shape, with / without values, permutation vector, idx_in."""
    if one_cta:
        monkeypatch.setenv("LCO_SINGLE_CTA", "1")
    rng = np.random.default_rng(nnz)
    dims = (16, 12, 5)  # q of every permutation has <= 10 bits
    total = int(np.prod(dims))
    keys = np.sort(rng.choice(total, min(nnz, total), replace=False)).astype(np.uint64)
    if nnz > total:  # larger tensors: (40, 30, 8) has q <= 10 bits for perms moving c2 first
        dims = (40, 30, 8)
        keys = np.sort(rng.choice(40 * 30 * 8, nnz, replace=False)).astype(np.uint64)
    vals = rng.standard_normal(len(keys))
    idx = (rng.permutation(len(keys)) + 17).astype(np.uint32)
    for perm in itertools.permutations(range(3)):
        info = lco.plan(dims, perm).info(len(keys))
        if info["sort_bits"] == 0:
            continue
        if info["sort_bits"] <= 10:
            assert info["path"] == "single", (perm, info["path"])
        check(dims, perm, keys, vals)
        check(dims, perm, keys, None, return_perm=False)
        check(dims, perm, keys, vals, idx=idx)
    w = workloads.config("C1")
    assert lco.plan(w.dims, w.perms[0]).info(w.keys.numel())["path"] == "single"


@pytest.mark.parametrize("stable", [False, True])
def test_msd_level3_crowded_leaves(stable, cuda_device, monkeypatch):
    """C3b's operator under a forced two-level MSD plan: every q value is shared by 128+
    nonzeros (the suffix modes z, z'), so level-2 leaves are oversize, level-3 leaves are
    crowded and go to the deferred list as level-code-4 entries (a regression: the code
    once overflowed the entry's 2-bit level field and those leaves were never written).
    Both the unordered (K' tie-break) and the stable passes, bit-exact."""
    monkeypatch.setenv("LCO_MSD", "1")
    monkeypatch.setenv("LCO_MSD_CTA", "1")
    if stable:
        monkeypatch.setenv("LCO_STABLE_MSD", "1")
    w = workloads.config("C3", scale=96)
    dims, perm = w.dims, w.perms[1]
    info = lco.plan(dims, perm).info(w.keys.numel())
    assert info["path"] == "msd" and info["msd_levels"] == 2
    check(dims, perm, _np_u64(w.keys), w.vals.numpy())


def test_table2_laplacian_level3_full(cuda_device):
    """Table 2's worst permutations at the paper's size (N = 2896, 42M nonzeros), default
    plans (two MSD levels + level 3): permute and sort bit-exact against the oracle (the
    all-cores run of the same definition, oracle.permute_par)."""
    n = 2896
    k, v = workloads.combinatorial_laplacian(n)
    keys, vals = _np_u64(k), v.numpy()
    dk, dv = k.to(cuda_device), v.to(cuda_device)
    for perm, sort in (((3, 1, 2, 0), False), ((0, 2, 1, 3), True)):
        p = lco.plan((n,) * 4, perm)
        ko, vo, po = (p.sort if sort else p.permute)(dk, dv)
        ek, ev, ep = oracle.permute_par((n,) * 4, perm, keys, vals)
        assert np.array_equal(_np_u64(ko), ek), perm
        assert np.array_equal(po.cpu().numpy().view(np.uint32), ep), perm
        assert np.array_equal(vo.cpu().numpy().view(np.uint64), ev.view(np.uint64)), perm


# ------------------------------------------------------------------ prefix plans on the full key
@pytest.mark.parametrize("nnz", [300_000, 2_500_000])
def test_prefix_plan_sorts_full_key_by_msd(nnz, cuda_device):
    """An identity prefix with a shaved key of >= 4 LSD passes runs the MSD schedule of the
    full new key instead (api.cu permute_op; the prefix digits are
    already in order, so both stable sorts give one output), from two MSD levels on;
    bit-exact against the oracle, with and without the permutation vector."""
    rng = np.random.default_rng(77)
    dims, perm = (64,) * 7, (0, 6, 5, 4, 3, 2, 1)
    info = lco.Plan(dims, perm).info(nnz)
    if nnz < 1_000_000:  # below two MSD levels the shaved key stays on LSD passes
        assert (info["path"], info["sort_bits"]) == ("lsd", 36)
    else:
        assert (info["path"], info["sort_bits"], info["msd_levels"]) == ("msd", 42, 2)
    keys, vals = _rand_sorted(rng, dims, nnz)
    check(dims, perm, keys, vals)
    check(dims, perm, keys, vals, return_perm=False)
    # unevenly filled prefix digits: the lowest third of the keys only (level 3 re-splits)
    third = len(keys) // 3
    check(dims, perm, keys[:third], vals[:third])
