"""Host logic of liblco.so (CPU only: no device call is made).

* every symbol declared in include/lco.h is exported;
* the host fast divisor equals plain // (the device kernels use the same arithmetic);
* the plan: rearrangement/resting classification equals the oracle's,
  the Fig 3 plan constants, and — the property the GPU path relies on —
  a stable sort of the sorted input by q = K' div T (T = plan "trailing") reproduces the
  oracle's output for every permutation of orders 1-6 (the suffix modes are free);
* argument errors map to the documented statuses.
"""
import itertools
import os
import re

import numpy as np
import pytest

import oracle
import paper_1802_02619_b200 as lco
from paper_1802_02619_b200 import lco as L
from tests import brute

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "lco.h")).read()
    names = re.findall(r"^LCO_API\s+[\w\s\*]+?\b(lco_\w+)\s*\(", hdr, flags=re.M)
    assert len(names) >= 16
    lib = lco.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert lco.version().startswith("lco-b200")


def test_fastdiv_matches_plain_division():
    rng = np.random.default_rng(0)
    divisors = [1, 2, 3, 5, 6, 7, 10, 30, 48, 641, 1023, 3072, 2 ** 10 - 1, 2 ** 10 + 1,
                2 ** 31 - 1, 2 ** 32 + 1, 2 ** 40 - 3, 2 ** 62 + 1, 2 ** 63 - 1, 6700417]
    divisors += [int(x) for x in rng.integers(1, 2 ** 63 - 1, 30, dtype=np.int64)]
    divisors += [int(x) for x in rng.integers(1, 5000, 30)]
    edge = [0, 1, 2, 2 ** 32 - 1, 2 ** 32, 2 ** 63 - 1, 2 ** 63, 2 ** 64 - 1, 2 ** 64 - 2]
    for d in divisors:
        xs = edge + [d - 1, d, d + 1, 2 * d - 1, 2 * d, (2 ** 64 - 1) // d * d,
                     (2 ** 64 - 1) // d * d - 1]
        xs += [int(x) for x in rng.integers(0, 2 ** 63, 400, dtype=np.int64)]
        xs += [int(x) * 2 + 1 for x in rng.integers(0, 2 ** 62, 100, dtype=np.int64)]
        xs = [x % 2 ** 64 for x in xs]
        assert lco.fastdiv_host(d, xs) == [x // d for x in xs], d
    # exhaustive small range
    for d in range(1, 200):
        xs = list(range(0, 5000))
        assert lco.fastdiv_host(d, xs) == [x // d for x in xs]


def test_fig3_plan_constants():
    """10x3x2 a_ijk, {0,1,2}->{1,0,2}: regions of constant k by dividing
    by n_j n_i = 30; the shaved key (LIV mod 30) div 3 = i; i rearrangement."""
    p = lco.Plan((2, 3, 10), (0, 2, 1))
    info = p.info(60)
    assert info["rearrangement"] == [0, 1, 0]
    assert info["prefix_len"] == 1 and info["num_segments"] == 2
    assert info["segment_divisor"] == 30
    assert info["trailing"] == 3 and info["middle_size"] == 10


def _random_dims(rng, order):
    return tuple(int(x) for x in rng.integers(1, 6 if order <= 4 else 4, order))


@pytest.mark.parametrize("order", [1, 2, 3, 4, 5, 6])
def test_plan_stable_sort_on_shaved_key_equals_oracle(order):
    rng = np.random.default_rng(order)
    perms = list(itertools.permutations(range(order)))
    if len(perms) > 240:
        perms = [perms[i] for i in rng.choice(len(perms), 240, replace=False)]
    for perm in perms:
        dims = _random_dims(rng, order)
        total = int(np.prod(dims))
        nnz = int(rng.integers(0, total + 1))
        keys = np.sort(rng.choice(total, nnz, replace=False)).astype(np.uint64)
        p = lco.Plan(dims, perm)
        info = p.info(nnz)
        assert info["rearrangement"] == oracle.classify(perm)
        new = brute.reencode_np(dims, perm)(keys)
        _, _, ep = oracle.permute(dims, perm, keys)
        if info["path"] == "copy":
            assert np.array_equal(ep, np.arange(nnz))
            continue
        q = new // np.uint64(info["trailing"])
        assert int(q.max(initial=0)) < 2 ** info["sort_bits"]
        assert sum(info["digit_bits"]) + info["leaf_bits"] == info["sort_bits"]
        assert np.array_equal(np.argsort(q, kind="stable"), ep), (dims, perm)
        # the sort plan sorts on every key bit (T = 1)
        si = p.info(nnz, sort=True)
        assert si["trailing"] == 1 and si["sort_bits"] >= info["sort_bits"]


def test_baseline_config_plans():
    """Key bits the passes sort per BASELINE config (SURVEY.md §8(a) sizes table) and the
    schedule chosen at the config's nnz."""
    cases = {
        ("C1", (64, 48, 32), (2, 0, 1), 5000): (5, "single"),
        ("C2a", (512,) * 4, (2, 3, 0, 1), 1308672): (18, "msd"),
        ("C2b", (512,) * 4, (0, 2, 1, 3), 1308672): (18, "tile"),
        ("C3a", (128,) * 6, (3, 4, 5, 0, 1, 2), 14581760): (21, "lsd"),
        ("C3b", (128,) * 6, (0, 3, 1, 4, 2, 5), 14581760): (28, "lsd"),
        ("C4", (2048,) * 4, (1, 0, 2, 3), 54484996): (11, "block"),
        ("C5", (4096,) * 5, (4, 3, 2, 1, 0), 500_000_000): (48, "msd"),
    }
    for (name, dims, perm, nnz), (bits, path) in cases.items():
        info = lco.Plan(dims, perm).info(nnz)
        assert (info["sort_bits"], info["path"]) == (bits, path), (name, info)
        if path not in ("tile", "hier", "block"):  # no radix digits on these paths
            assert sum(info["digit_bits"]) + info["leaf_bits"] == bits
    # C3b: interior resting modes -> two stages: the c3 digit inside
    # the 128 c0 segments (one segmented pass), then c4 inside (c0, c3, c1) regions
    # (segment-local tiles); 14 bits sorted instead of the flat plan's 28
    c3b = lco.Plan((128,) * 6, (0, 3, 1, 4, 2, 5)).info(14581760)
    assert c3b["stage_paths"] == ["seg", "tile"] and c3b["stage_sort_bits"] == [14, 28]
    h = lco.Plan((128,) * 6, (0, 3, 1, 4, 2, 5), hierarchical=True).info(14581760)
    assert h["path"] == "hier" and h["model_bytes"] < h["flat_model_bytes"]
    # measured: the staged plan 0.76 ms vs the flat 3-pass LSD 0.70 ms (the clustered
    # tile sort of stage 2 costs ~2 passes), so the cost model keeps the flat plan
    # C2b: 512 segments of ~2.5K nonzeros (the x rows), sorted in place tile by tile
    c2b = lco.Plan((512,) * 4, (0, 2, 1, 3)).info(1308672)
    assert c2b["num_segments"] == 512 and c2b["leaf_kind"] == "cta" and c2b["launches"] == 3
    c4 = lco.Plan((2048,) * 4, (1, 0, 2, 3)).info(54484996)
    assert c4["norm_dims"] == [2048, 2048, 2 ** 22] and c4["norm_perm"] == [1, 0, 2]
    assert c4["trailing"] == 2048 * 2 ** 22 and c4["path"] == "block" and c4["passes"] == 0


def test_call_schedules():
    """Schedule per nnz: one on-chip leaf when it fits, MSD + leaves for wide keys, LSD
    otherwise (modelled bytes decide; results are identical)."""
    p = lco.Plan((4096,) * 5, (4, 3, 2, 1, 0))
    assert p.info(1000)["path"] == "leaf"
    # one tile of <= 8,192 nonzeros and a digit of <= 10 bits: one stable single-CTA pass
    assert lco.Plan((64, 48, 32), (2, 0, 1)).info(5000)["path"] == "single"
    assert lco.Plan((64, 48, 32), (2, 0, 1)).info(8193)["path"] != "single"
    i = p.info(500_000_000)
    assert i["path"] == "msd" and i["msd_levels"] == 2
    assert sum(i["digit_bits"]) + i["leaf_bits"] == 48
    # 8-bit first MSD digit (runs of ~16 per tile), second digit sized for ~1.9K-nonzero
    # leaves sorted fully staged by one CTA
    assert i["digit_bits"] == [8, 10] and i["leaf_kind"] == "cta"
    assert p.info(8192)["path"] == "leaf" and p.info(8193)["path"] == "msd"
    assert p.info(40_000)["msd_levels"] == 1
    # C4: the rearranged modes (x, y) lie before the free (x', y') modes -> a tiled
    # transpose of the 2048 x 2048 grid of runs; without it, one 11-bit LSD pass
    assert lco.Plan((2048,) * 4, (1, 0, 2, 3)).info(54_484_996)["path"] == "block"


def test_block_schedule_opt_out(monkeypatch):
    monkeypatch.setenv("LCO_NO_BLOCK", "1")
    assert lco.Plan((2048,) * 4, (1, 0, 2, 3)).info(54_484_996)["path"] == "lsd"


def test_identity_and_size1_moves_are_copies():
    assert lco.Plan((4, 5, 6), (0, 1, 2)).info(10)["path"] == "copy"
    assert lco.Plan((4, 1, 6), (1, 0, 2)).info(10)["path"] == "copy"  # only a size-1 mode moves
    assert lco.Plan((7,), (0,)).info(10)["path"] == "copy"


def test_argument_errors():
    with pytest.raises(ValueError, match="PERM"):
        lco.Plan((4, 4), (0, 0))
    with pytest.raises(ValueError, match="OVERFLOW"):
        lco.Plan((2 ** 32, 2 ** 32), (1, 0))
    with pytest.raises(ValueError, match="ORDER"):
        lco.Plan((2,) * 17)
    with pytest.raises(ValueError, match="DIM"):
        lco.Plan((4, 0), (1, 0))
    with pytest.raises(ValueError, match="CAPACITY"):
        lco.Plan((4, 4), (1, 0), max_nnz=2 ** 32)


def test_workspace_sizes():
    p = lco.Plan((4096,) * 5, (4, 3, 2, 1, 0))
    ws = p.workspace_size(500_000_000)
    # two ping-pong (key, value, position) buffers + two look-back status arrays
    assert 2 * 20 * 500_000_000 < ws < 2 * 20 * 500_000_000 + 4 * 10 ** 9
    assert lco.Plan((4, 4), (0, 1)).workspace_size(100) < 1 << 20
    assert p.host_workspace_size(10) > p.workspace_size(10)


def test_no_cpu_fallback():
    import torch
    p = lco.Plan((4, 4), (1, 0))
    with pytest.raises(ValueError, match="CUDA"):
        p.permute(torch.zeros(3, dtype=torch.int64))


@pytest.mark.parametrize("order", [2, 3, 4, 5, 6])
def test_hierarchical_stages_compose_to_oracle(order):
    """Hierarchical plan ("recursively applied to each of these
    sub-regions"): one stage per maximal run of rearrangement indices
    of the normalized permutation.  Applying the stages in order with the oracle's stable
    permute reproduces the oracle's permute of the whole permutation (keys, values and the
    composed permutation vector), and every stage sorts only its own run."""
    rng = np.random.default_rng(100 + order)
    perms = list(itertools.permutations(range(order)))
    if len(perms) > 200:
        perms = [perms[i] for i in rng.choice(len(perms), 200, replace=False)]
    for perm in perms:
        dims = _random_dims(rng, order)
        total = int(np.prod(dims))
        nnz = int(rng.integers(0, min(total, 3000) + 1))
        keys = np.sort(rng.choice(total, nnz, replace=False)).astype(np.uint64)
        vals = rng.standard_normal(nnz)
        p = lco.Plan(dims, perm)
        stages = p.stages()
        norm = p.info(nnz)["norm_perm"]
        flags = oracle.classify(tuple(norm)) if norm else []
        runs = sum(1 for t, f in enumerate(flags) if f and (t == 0 or not flags[t - 1]))
        assert len(stages) == max(1, runs), (dims, perm, stages)
        k, v, pos = keys, vals, np.arange(nnz)
        for sdims, sperm in stages:
            if not sdims:  # every mode has size 1: nothing moves
                continue
            assert int(np.prod(sdims)) == int(np.prod([d for d in dims]))
            k, v, sp = oracle.permute(sdims, sperm, k, v)
            pos = pos[sp]
            if len(stages) > 1:  # a stage's rearrangement indices form one run
                sf = oracle.classify(tuple(sperm))
                assert sum(1 for t, f in enumerate(sf) if f and (t == 0 or not sf[t - 1])) == 1
        ek, ev, ep = oracle.permute(dims, perm, keys, vals)
        assert np.array_equal(k, ek) and np.array_equal(v.view(np.uint64), ev.view(np.uint64))
        assert np.array_equal(pos, ep), (dims, perm)


def test_new_entry_points_reject_bad_arguments_before_any_launch():
    """lco_add / lco_compress / lco_plan_stage: argument errors are detected on the host
    (no device memory touched, no GPU needed) and reported as status codes."""
    import ctypes
    lib = lco.lib()
    h = lco.Plan((4, 5, 6), (2, 0, 1))
    nc = ctypes.c_size_t()
    assert lib.lco_add_workspace_size(h._h, 10, 20, ctypes.byref(nc)) == 0 and nc.value > 0
    # lco_add: NULL count / outputs -> LCO_ERR_NULL (1)
    assert lib.lco_add(h._h, 0, None, None, 0, None, None, 1.0, None, None, None, None, 0, None) == 1
    # lco_add: operand at or above 2^32 nonzeros -> LCO_ERR_CAPACITY (6)
    dummy = ctypes.c_void_p(256)
    assert lib.lco_add(h._h, 2 ** 32, dummy, dummy, 0, None, None, 1.0, dummy, dummy, dummy,
                       None, 0, None) == 6
    # lco_compress: zero dims -> LCO_ERR_DIM (3); missing outputs -> LCO_ERR_NULL (1)
    assert lib.lco_compress(0, None, 0, 5, 0, dummy, None, None, None, None, 0, None) == 3
    assert lib.lco_compress(10, None, 5, 5, 1, dummy, None, None, None, None, 0, None) == 1
    b = ctypes.c_size_t()
    assert lib.lco_compress_workspace_size(1000, 1, ctypes.byref(b)) == 0 and b.value > 0
    assert lib.lco_compress_workspace_size(1000, 0, ctypes.byref(b)) == 0 and b.value == 0
    # lco_plan_stage: out-of-range stage -> LCO_ERR_ARG
    n_st, order = ctypes.c_int(), ctypes.c_int()
    dims = (ctypes.c_uint64 * 16)()
    perm = (ctypes.c_int32 * 16)()
    assert lib.lco_plan_stage(h._h, 5, ctypes.byref(n_st), ctypes.byref(order), dims, perm) != 0
    assert n_st.value == 1
    # the MDT table rejects unknown classes
    assert lib.lco_mdt_choice(4, 0) == -1 and lib.lco_mdt_name(-1) == b"invalid"


def test_block_grid_decomposition():
    """Block transpose (path 7): blocks = runs of constant old modes 0..k (k = last old
    position of a prefix / middle mode) of the NORMALIZED plan; A = old mode k, B = the new
    order's innermost block mode, the tiles span (B, A) with the block modes before B /
    between B and A fixed (hand-derived values; their product is the block count)."""
    cases = {
        ((2048,) * 4, (1, 0, 2, 3), 54_484_996): [2048 * 2048, 2048, 2048, 1, 1],
        # modes 1, 2 fuse: (16, 96, 2000) with perm (1, 0, 2)
        ((16, 8, 12, 10, 200), (1, 2, 0, 3, 4), 250_000): [16 * 96, 96, 16, 1, 1],
        # modes 0, 1 fuse: (2048, 16, 300) with perm (1, 0, 2)
        ((64, 32, 16, 300), (2, 0, 1, 3), 250_000): [2048 * 16, 16, 2048, 1, 1],
        # identity prefix c0 before B
        ((3, 700, 9, 400), (0, 2, 1, 3), 250_000): [3 * 700 * 9, 9, 700, 1, 3],
        # reversal of three modes: c1 sits between B = c0 and A = c2
        ((20, 30, 40, 500), (2, 1, 0, 3), 250_000): [20 * 30 * 40, 40, 20, 30, 1],
    }
    for (dims, perm, nnz), grid in cases.items():
        info = lco.Plan(dims, perm).info(nnz)
        assert info["path"] == "block", (dims, perm, info["path"])
        assert info["block_grid"] == grid, (dims, perm, info["block_grid"])
        nb, da, db, mid, hi = grid
        assert da * db * mid * hi == nb
    # too few nonzeros per block (< 4 on average): sorted instead
    assert lco.Plan((2048,) * 4, (1, 0, 2, 3)).info(4_000_000)["path"] != "block"


def test_partition_world_bound_and_tuning_read_once(monkeypatch):
    """lco_partition_counts / lco_partition take 1..2048 ranks (the widest
    partition digit is 11 bits) and reject 2049 on the host; schedule overrides are read
    once at lco_create, clamped, and never on a call."""
    import ctypes
    lib = lco.lib()
    h = lco.Plan((64, 64, 64), (2, 1, 0))
    dummy = ctypes.c_void_p(256)
    for fn in (lib.lco_partition_counts,):
        assert fn(h._h, 0, None, 2049, dummy, dummy, None, 0, None) == 12  # LCO_ERR_ARG
    assert lib.lco_partition(h._h, 0, None, None, 0, 2049, dummy, None, None, None, dummy, None,
                             0, None) == 12
    # LCO_LSD_MAXBITS=1 on 60 key bits would need 60 passes: clamped to <= 8 passes
    monkeypatch.setenv("LCO_LSD_MAXBITS", "1")
    for dims, perm in (((4096,) * 5, (4, 3, 2, 1, 0)), ((64, 64, 64), (2, 1, 0))):
        info = lco.Plan(dims, perm).info(100_000, sort=True)
        assert 1 <= info["passes"] <= 8
        assert all(1 <= b <= 11 for b in info["digit_bits"])
    monkeypatch.setenv("LCO_LSD_MAXBITS", "0")  # clamped to 1, no division by zero
    assert lco.Plan((64, 64, 64), (2, 1, 0)).info(100_000)["passes"] >= 1
    monkeypatch.delenv("LCO_LSD_MAXBITS")
    # an override set after lco_create does not change the handle's schedule
    q = lco.Plan((512,) * 4, (2, 3, 0, 1), max_nnz=(1 << 32) - 2)
    before = q.info(1_308_672)
    monkeypatch.setenv("LCO_MSD", "1")
    monkeypatch.setenv("LCO_NO_BLOCK", "1")
    assert q.info(1_308_672) == before


def test_prefix_plan_takes_full_key_msd_only_when_modelled_faster():
    """api.cu permute_op: with an identity prefix the flat plan sorts the shaved key q by
    LSD passes; from 4 passes on, the MSD schedule of the full new key K' models below it
    and is taken (same output: the prefix digits are non-decreasing in the input,
    PAPER.md:245-247).  Three-pass plans (C3b, Table 2's 2 % tensor) and segment/tile
    plans stay as they were; the workspace covers either choice."""
    p = lco.Plan((2896,) * 4, (0, 3, 2, 1))
    i = p.info(41_910_912)
    assert (i["path"], i["sort_bits"], i["model_bytes"]) == ("msd", 46, 132.0)
    i = lco.Plan((4096,) * 5, (0, 4, 3, 2, 1)).info(500_000_000)
    assert (i["path"], i["sort_bits"], i["msd_levels"]) == ("msd", 60, 2)
    i = lco.Plan((128,) * 6, (0, 3, 1, 4, 2, 5)).info(14_581_760)  # C3b
    assert (i["path"], i["sort_bits"], i["passes"]) == ("lsd", 28, 3)
    i = lco.Plan((200,) * 4, (0, 3, 2, 1)).info(32_000_000)
    assert (i["path"], i["sort_bits"]) == ("lsd", 23)
    i = lco.Plan((64,) * 7, (0, 6, 5, 4, 3, 2, 1)).info(300_000)
    assert (i["path"], i["sort_bits"]) == ("lsd", 36)  # one-level MSD plans are not taken
    # lco_workspace_size is the maximum over the permute and the sort plan
    q = lco.Plan((2896,) * 4, (3, 2, 1, 0))  # no prefix: MSD on the same 46 bits
    assert p.workspace_size(41_910_912) >= q.workspace_size(41_910_912)
