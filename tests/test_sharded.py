"""Sharded (multi-GPU) orchestration on CPU: world sizes 2 and 3 with the gloo backend.

The device operations are replaced by oracle-backed test doubles (same contracts as
lco_key_histogram / lco_partition / lco_permute); what is tested is the orchestration of
paper_1802_02619_b200.sharded: global index bases, splitter choice from the all-reduced
histogram, count and payload all_to_all, concatenation order, and that the per-rank
outputs concatenate to the single-device oracle result bit for bit (SURVEY.md §8(e),
DESIGN.md "Multi-GPU")."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1802_02619_b200 import sharded


class OracleOps:
    def __init__(self, dims, perm):
        self.dims, self.perm = tuple(dims), tuple(perm)

    def key_histogram(self, keys, bits):
        kb = sharded.key_bits(self.dims)
        new = oracle.shuffle(self.dims, self.perm, keys.numpy().view(np.uint64))
        b = (new >> np.uint64(max(0, kb - bits))).astype(np.int64)
        return torch.from_numpy(np.bincount(b, minlength=1 << bits).astype(np.int64))

    def partition(self, keys, vals, idx_base, splitters):
        spl = np.zeros(0, np.uint64) if splitters is None else splitters.numpy().view(np.uint64)
        sk, sv, si, cnt = oracle.partition(self.dims, self.perm, keys.numpy().view(np.uint64),
                                           vals.numpy(), idx_base, spl)
        return (torch.from_numpy(sk.view(np.int64)), torch.from_numpy(sv),
                torch.from_numpy(si.view(np.int32)), torch.from_numpy(cnt.astype(np.int64)))

    def segment_divisor(self):
        """Identity prefix a (perm[t] = t for t < a) -> segments of constant (c_0..c_{a-1}):
        D = prod(dims[a:]) (0: no prefix), computed here from the definition."""
        a = 0
        while a < len(self.perm) and self.perm[a] == a:
            a += 1
        return int(np.prod(self.dims[a:])) if 0 < a < len(self.perm) else 0

    def permute(self, keys, vals, idx):
        ko, vo, po = oracle.permute(self.dims, self.perm, keys.numpy().view(np.uint64),
                                    vals.numpy(), idx.numpy().view(np.uint32))
        return (torch.from_numpy(ko.view(np.int64)), torch.from_numpy(vo),
                torch.from_numpy(po.view(np.int32)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, perm, keys, vals, cuts, outdir, exchange="auto"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = cuts[rank], cuts[rank + 1]
    k = torch.from_numpy(keys[lo:hi].view(np.int64).copy())
    v = torch.from_numpy(vals[lo:hi].copy())
    ko, vo, po = sharded.permute_sharded(k, v, dims, perm, ops=OracleOps(dims, perm), bits=6,
                                         exchange=exchange)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), k=ko.numpy(), v=vo.numpy(), p=po.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,perm,nnz,uneven,exchange", [
    (2, (64, 48, 32), (2, 0, 1), 5000, False, "auto"),
    (2, (16, 16, 16, 16), (3, 1, 2, 0), 20000, True, "auto"),
    (3, (40, 30, 20), (1, 2, 0), 7000, True, "auto"),
    # identity-prefix segments (C2b / C3b shapes): exchange-free; segments of ~40 nonzeros
    # straddle the cuts, one rank's slice lies inside a single segment
    (3, (64, 8, 8, 16), (0, 2, 1, 3), 6000, True, "auto"),
    (2, (32, 16, 16), (0, 2, 1), 4000, False, "segments"),
    # the same shape through the partition + exchange path
    (3, (64, 8, 8, 16), (0, 2, 1, 3), 6000, True, "nccl"),
])
def test_sharded_matches_single_device(world, dims, perm, nnz, uneven, exchange, tmp_path):
    rng = np.random.default_rng(nnz)
    total = int(np.prod(dims))
    keys = np.sort(rng.choice(total, nnz, replace=False)).astype(np.uint64)
    vals = rng.standard_normal(nnz)
    if uneven:  # one rank gets a small slice, another a large one
        cuts = [0] + sorted(rng.choice(np.arange(1, nnz), world - 1, replace=False).tolist()) + [nnz]
        cuts[1] = min(cuts[1], 17)
        cuts = sorted(cuts)
    else:
        cuts = [nnz * r // world for r in range(world + 1)]
    mp.spawn(_worker, args=(world, _free_port(), dims, perm, keys, vals, cuts, str(tmp_path),
                            exchange), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    ko = np.concatenate([p["k"] for p in parts]).view(np.uint64)
    vo = np.concatenate([p["v"] for p in parts])
    po = np.concatenate([p["p"] for p in parts]).view(np.uint32)
    ek, ev, ep = oracle.permute(dims, perm, keys, vals)
    assert np.array_equal(ko, ek) and np.array_equal(po, ep)
    assert np.array_equal(vo.view(np.uint64), ev.view(np.uint64))
    # every rank owns a contiguous new-key range and the load is spread
    sizes = [len(p["k"]) for p in parts]
    assert sum(sizes) == nnz


def test_choose_splitters_quantiles():
    h = torch.tensor([10, 0, 30, 0, 0, 60, 0, 0], dtype=torch.int64)
    spl = sharded.choose_splitters(h, 2, kbits=6, bits=3)
    below = int(h[: int(spl[0]) >> 3].sum())
    assert below == 40  # 40 / 60 is the split closest to the median
    assert sharded.choose_splitters(h, 1, 6, 3).numel() == 0
    # device-side: ascending, one per rank boundary, every cut at a quantile-closest bin
    rng = np.random.default_rng(3)
    h = torch.from_numpy(rng.integers(0, 50, 256).astype(np.int64))
    for world in (2, 3, 8):
        spl = sharded.choose_splitters(h, world, kbits=16, bits=8)
        assert spl.numel() == world - 1 and bool((spl[1:] >= spl[:-1]).all())
        cum = np.concatenate([[0], np.cumsum(h.numpy())])
        for r, s in enumerate(spl.tolist(), start=1):
            target = (int(cum[-1]) * r + world - 1) // world
            best = min(abs(int(c) - target) for c in cum)
            assert abs(int(cum[s >> 8]) - target) == best


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
def test_virtual_ranks_cuda(world, cuda_device):
    """The CUDA kernels of the sharded path, ranks emulated one after another on one GPU
    (no rank waits on another): key histogram -> splitters -> lco_partition per slice ->
    per-destination concatenation in source order -> lco_permute(idx_in)."""
    import paper_1802_02619_b200 as lco
    import workloads
    w = workloads.config("C5", scale=400_000, device=cuda_device)
    dims, perm = w.dims, w.perms[0]
    p = lco.plan(dims, perm)
    n = w.keys.numel()
    cuts = [n * r // world for r in range(world + 1)]
    kb = sharded.key_bits(dims)
    hist = sum(p.key_histogram(w.keys[cuts[r]:cuts[r + 1]], 12) for r in range(world))
    spl = sharded.choose_splitters(hist, world, kb, 12)
    sends = [p.partition(w.keys[cuts[r]:cuts[r + 1]], w.vals[cuts[r]:cuts[r + 1]], cuts[r], spl)
             for r in range(world)]
    outs = []
    for dst in range(world):
        ks, vs, ix = [], [], []
        for src in range(world):
            sk, sv, si, cnt = sends[src]
            off = int(cnt[:dst].sum())
            c = int(cnt[dst])
            ks.append(sk[off:off + c]); vs.append(sv[off:off + c]); ix.append(si[off:off + c])
        outs.append(p.permute(torch.cat(ks), torch.cat(vs), torch.cat(ix)))
    torch.cuda.synchronize()
    ko = torch.cat([o[0] for o in outs]).cpu().numpy().view(np.uint64)
    vo = torch.cat([o[1] for o in outs]).cpu().numpy()
    po = torch.cat([o[2] for o in outs]).cpu().numpy().view(np.uint32)
    ek, ev, ep = oracle.permute(dims, perm, w.keys.cpu().numpy().view(np.uint64), w.vals.cpu().numpy())
    assert np.array_equal(ko, ek) and np.array_equal(po, ep)
    assert np.array_equal(vo.view(np.uint64), ev.view(np.uint64))
    sizes = [o[0].numel() for o in outs]
    assert max(sizes) < 1.2 * n / world  # splitters balance uniform keys


@pytest.mark.gpu
@pytest.mark.parametrize("world,vals", [(2, True), (4, True), (8, False), (16, True)])
def test_virtual_ranks_direct_exchange(world, vals, cuda_device):
    """The exchange fused into the partition (lco_partition_direct): each (emulated) rank
    counts its records per destination (lco_partition_counts), the counts give every
    source chunk its offset in each receiver (source-rank order), and the partition
    scatter stores the records straight into the receivers' buffers -- which on a
    multi-GPU box are peer-mapped NVLink memory.  The receivers' buffers must equal the
    send chunks of lco_partition concatenated in source order, and the local permutes
    the single-GPU oracle."""
    import paper_1802_02619_b200 as lco
    import workloads
    w = workloads.config("C5", scale=300_000, device=cuda_device)
    dims, perm = w.dims, w.perms[0]
    p = lco.plan(dims, perm)
    n = w.keys.numel()
    cuts = [n * r // world for r in range(world + 1)]
    kb = sharded.key_bits(dims)
    hist = sum(p.key_histogram(w.keys[cuts[r]:cuts[r + 1]], 12) for r in range(world))
    spl = sharded.choose_splitters(hist, world, kb, 12)
    sl = [(w.keys[cuts[r]:cuts[r + 1]], w.vals[cuts[r]:cuts[r + 1]] if vals else None)
          for r in range(world)]
    counts = torch.stack([p.partition_counts(k, spl) for k, _ in sl]).cpu()  # [src][dst]
    total = counts.sum(0)
    rk = [torch.full((int(total[d]),), -1, dtype=torch.int64, device=cuda_device) for d in range(world)]
    rv = [torch.full((int(total[d]),), float("nan"), dtype=torch.float64, device=cuda_device)
          for d in range(world)] if vals else None
    ri = [torch.full((int(total[d]),), -1, dtype=torch.int32, device=cuda_device) for d in range(world)]
    for r, (k, v) in enumerate(sl):
        offs = [int(counts[:r, d].sum()) for d in range(world)]
        cnt = p.partition_direct(k, v, cuts[r], spl, rk, rv, ri, offs)
        assert torch.equal(cnt.cpu(), counts[r])
    torch.cuda.synchronize()
    outs = []
    for d in range(world):
        exp_k, exp_v, exp_i = [], [], []
        for r, (k, v) in enumerate(sl):
            sk, sv, si, cnt = p.partition(k, v if vals else None, cuts[r], spl)
            o, c = int(cnt[:d].sum()), int(cnt[d])
            exp_k.append(sk[o:o + c]); exp_i.append(si[o:o + c])
            if vals:
                exp_v.append(sv[o:o + c])
        assert torch.equal(rk[d], torch.cat(exp_k)) and torch.equal(ri[d], torch.cat(exp_i))
        if vals:
            assert torch.equal(rv[d].view(torch.int64), torch.cat(exp_v).view(torch.int64))
        outs.append(p.permute(rk[d], rv[d] if vals else None, ri[d]))
    torch.cuda.synchronize()
    ko = torch.cat([o[0] for o in outs]).cpu().numpy().view(np.uint64)
    po = torch.cat([o[2] for o in outs]).cpu().numpy().view(np.uint32)
    ek, ev, ep = oracle.permute(dims, perm, w.keys.cpu().numpy().view(np.uint64), w.vals.cpu().numpy())
    assert np.array_equal(ko, ek) and np.array_equal(po, ep)
    if vals:
        vo = torch.cat([o[1] for o in outs]).cpu().numpy()
        assert np.array_equal(vo.view(np.uint64), ev.view(np.uint64))


@pytest.mark.gpu
def test_permute_sharded_world1_nccl(cuda_device, tmp_path):
    """permute_sharded end to end through NCCL with a single rank."""
    import workloads
    w = workloads.config("C5", scale=100_000, device=cuda_device)
    store = dist.FileStore(str(tmp_path / "store"), 1)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=cuda_device)
    try:
        ko, vo, po = sharded.permute_sharded(w.keys, w.vals, w.dims, w.perms[0])
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
    ek, ev, ep = oracle.permute(w.dims, w.perms[0], w.keys.cpu().numpy().view(np.uint64),
                                w.vals.cpu().numpy())
    assert np.array_equal(ko.cpu().numpy().view(np.uint64), ek)
    assert np.array_equal(po.cpu().numpy().view(np.uint32), ep)


@pytest.mark.gpu
def test_permute_sharded_world1_direct(cuda_device, tmp_path):
    """permute_sharded with the fused exchange (symmetric memory + lco_partition_direct)
    end to end with a single rank."""
    import workloads
    w = workloads.config("C5", scale=100_000, device=cuda_device)
    store = dist.FileStore(str(tmp_path / "store"), 1)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=cuda_device)
    try:
        ko, vo, po = sharded.permute_sharded(w.keys, w.vals, w.dims, w.perms[0], exchange="direct")
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
    ek, ev, ep = oracle.permute(w.dims, w.perms[0], w.keys.cpu().numpy().view(np.uint64),
                                w.vals.cpu().numpy())
    assert np.array_equal(ko.cpu().numpy().view(np.uint64), ek)
    assert np.array_equal(po.cpu().numpy().view(np.uint32), ep)
    assert np.array_equal(vo.cpu().numpy().view(np.uint64), ev.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
def test_virtual_ranks_segments_cuda(world, cuda_device):
    """The exchange-free path on the CUDA kernels, ranks emulated one after another on one
    GPU: C3b (identity-prefix segments of ~114K nonzeros at full scale, here scaled) cut
    into equal slices that straddle segments; each rank hands its head to the segment's
    owner (segment_handover), permutes whole segments with global indices, and the
    concatenation equals the single-GPU oracle bit for bit."""
    import paper_1802_02619_b200 as lco
    import workloads
    w = workloads.config("C3", scale=48, device=cuda_device)
    dims, perm = w.dims, w.perms[1]
    p = lco.plan(dims, perm)
    ops = sharded.CudaOps(dims, perm)
    D = ops.segment_divisor()
    assert D > 0
    n = w.keys.numel()
    # cuts a little past the equal split: the symmetric stencil puts equal cuts on segment
    # boundaries, these land inside segments
    cuts = [0] + [n * r // world + 777 for r in range(1, world)] + [n]
    sl = [(w.keys[cuts[r]:cuts[r + 1]], w.vals[cuts[r]:cuts[r + 1]]) for r in range(world)]
    tab = [sharded.segment_row(k, D).tolist() for k, _ in sl]
    give = sharded.segment_handover(tab)
    assert any(c for _, c in give)  # some slice starts inside a segment
    outs = []
    for r in range(world):
        k, v = sl[r]
        c = give[r][1]
        ks, vs = [k[c:]], [v[c:]]
        for s2 in range(r + 1, world):
            if give[s2][0] == r:
                ks.append(sl[s2][0][:give[s2][1]])
                vs.append(sl[s2][1][:give[s2][1]])
        lk, lv = torch.cat(ks), torch.cat(vs)
        idx = torch.arange(cuts[r] + c, cuts[r] + c + lk.numel(), device=cuda_device).to(torch.int32)
        outs.append(p.permute(lk, lv, idx))
    torch.cuda.synchronize()
    ko = torch.cat([o[0] for o in outs]).cpu().numpy().view(np.uint64)
    vo = torch.cat([o[1] for o in outs]).cpu().numpy()
    po = torch.cat([o[2] for o in outs]).cpu().numpy().view(np.uint32)
    ek, ev, ep = oracle.permute(dims, perm, w.keys.cpu().numpy().view(np.uint64), w.vals.cpu().numpy())
    assert np.array_equal(ko, ek) and np.array_equal(po, ep)
    assert np.array_equal(vo.view(np.uint64), ev.view(np.uint64))
