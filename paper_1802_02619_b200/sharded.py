"""Key-range sharded permutation across the GPUs of one box.

Every rank holds a contiguous slice of the sorted input (so slices are increasing old-key
ranges).  Per rank:

1. ``idx_base`` = number of nonzeros on lower ranks (all_gather of the slice sizes);
2. splitters on the NEW key: each rank histograms the top ``bits`` bits of its K'
   (``lco_key_histogram``), the histograms are all-reduced, and rank boundaries are cut
   at the quantiles of the global histogram (identical on every rank);
3. ``lco_partition`` stably routes every nonzero to the rank owning its new-key range:
   send buffers grouped by destination, each group in input order, carrying the OLD key,
   the value and the global source index ``idx_base + i``;
4. an ``all_to_all_single`` of the counts, then ONE grouped batch of NCCL point-to-point
   transfers for the keys, values and indices (over NVLink / NVSwitch);
5. the received records, concatenated in source-rank order, are exactly the global
   input restricted to this rank's new-key range, still sorted by old key (every
   source slice is an increasing key range and the partition is stable), so
   ``lco_permute(..., idx_in=received indices)`` finishes the job.

Rank r's output is the contiguous r-th part of the global output; concatenated over
ranks it equals the single-GPU result bit for bit, including the global permutation
vector.  Permutations with an identity prefix (segments that stay in place, C2b / C3b)
skip steps 2-4: a rank only hands the head of its slice that continues a segment begun
on a lower rank to that rank, then permutes whole segments locally.  The device work is the library's kernels; this module is orchestration only.
It takes an ``ops`` object so the orchestration can be exercised on CPU with the gloo
backend and test doubles (tests/test_sharded.py); the product uses :class:`CudaOps`.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import lco as _lco


class CudaOps:
    """The device operations of the sharded path: liblco.so kernels."""

    def __init__(self, dims, perm):
        self.plan = _lco.plan(dims, perm)
        self._symm = {}  # (group, dtype) -> (capacity, tensor, handle): reused across calls

    def key_histogram(self, keys, bits):
        return self.plan.key_histogram(keys, bits)

    def partition(self, keys, vals, idx_base, splitters):
        return self.plan.partition(keys, vals, idx_base, splitters)

    def permute(self, keys, vals, idx):
        return self.plan.permute(keys, vals, idx)

    def partition_counts(self, keys, splitters):
        return self.plan.partition_counts(keys, splitters)

    def partition_direct(self, keys, vals, idx_base, splitters, rk, rv, ri, offsets):
        return self.plan.partition_direct(keys, vals, idx_base, splitters, rk, rv, ri, offsets)

    def segment_divisor(self):
        """D such that key // D is constant on every region the permutation leaves in place
        (the identity-prefix segments); 0 if there are none."""
        info = self.plan.info(1)
        return int(info["segment_divisor"]) if info["num_segments"] > 1 else 0

    def symmetric(self, group_name, dtype, cap, device):
        """A symmetric-memory buffer of >= cap elements and its rendezvous handle, allocated
        once per (group, dtype) and grown geometrically (never per call)."""
        import torch.distributed._symmetric_memory as symm_mem
        key = (group_name, dtype)
        ent = self._symm.get(key)
        if ent is None or ent[0] < cap:
            c = max(cap, int((ent[0] if ent else 0) * 1.5), 1 << 16)
            t = symm_mem.empty(c, dtype=dtype, device=device)
            ent = (c, t, symm_mem.rendezvous(t, group_name))
            self._symm[key] = ent
        return ent


def key_bits(dims) -> int:
    total = 1
    for d in dims:
        total *= int(d)
    return max(0, (total - 1).bit_length())


def choose_splitters(global_hist: torch.Tensor, world: int, kbits: int, bits: int) -> torch.Tensor:
    """world-1 ascending new-key splitters (int64 tensor on the histogram's device) cutting
    the histogram at its quantiles, with no host round trip.  Rank r receives keys in
    [splitters[r-1], splitters[r])."""
    dev = global_hist.device
    if world <= 1:
        return torch.zeros(0, dtype=torch.int64, device=dev)
    cum = torch.cumsum(global_hist.to(torch.int64), 0)
    total = cum[-1]
    shift = max(0, kbits - bits)
    r = torch.arange(1, world, dtype=torch.int64, device=dev)
    target = (total * r + world - 1) // world
    b = torch.searchsorted(cum, target).clamp_(max=cum.numel() - 1)
    below = torch.where(b > 0, cum[(b - 1).clamp(min=0)], torch.zeros_like(b))
    # cut before bin b or after it, whichever lands closer to the quantile
    cut = torch.where(target - below <= cum[b] - target, b, b + 1)
    cut = torch.cummax(cut, 0).values  # non-decreasing
    return cut << shift


def _exchange(sends, recvs, scnt, rcnt, rank, world, group):
    """Every (send, recv) tensor pair is split by scnt / rcnt (elements per rank) and sent
    to / received from every peer in ONE grouped batch of point-to-point operations (one
    NCCL group launch for keys, values and indices together); the own chunk is a local
    copy."""
    soff = [0] * (world + 1)
    roff = [0] * (world + 1)
    for r in range(world):
        soff[r + 1] = soff[r] + scnt[r]
        roff[r + 1] = roff[r] + rcnt[r]
    ops = []
    for s, rv in zip(sends, recvs):
        if s is None:
            continue
        for peer in range(world):
            if peer == rank:
                rv[roff[peer]:roff[peer + 1]].copy_(s[soff[peer]:soff[peer + 1]])
                continue
            if scnt[peer]:
                ops.append(dist.P2POp(dist.isend, s[soff[peer]:soff[peer + 1]], peer, group))
            if rcnt[peer]:
                ops.append(dist.P2POp(dist.irecv, rv[roff[peer]:roff[peer + 1]], peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def permute_sharded(keys, vals, dims, perm, group=None, ops=None, bits=14, timings=None,
                    exchange="auto"):
    """Permute the globally sorted LCO tensor whose slice this rank holds.

    Returns (keys_out, vals_out, perm_out) of this rank's part of the output; perm_out
    holds GLOBAL source indices.  ``timings`` (dict) receives per-phase seconds measured
    with CUDA events when running on CUDA.  ``exchange``:
      "auto"     "segments" when the permutation keeps identity-prefix segments in place,
                 else "nccl";
      "segments" no key-range exchange: every segment stays at its positions (SURVEY.md
                 §8(e) "exchange-free case"), so each rank only hands the head of its slice
                 that continues a segment begun on a lower rank to that rank, then permutes
                 locally;
      "nccl"     partition into send buffers, then one grouped NCCL exchange;
      "direct"   the partition scatter stores every record into its receiver's
                 symmetric-memory buffer over NVLink (lco_partition_direct; CUDA only)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops = ops or CudaOps(dims, perm)
    dev = keys.device
    cuda = dev.type == "cuda"
    ev = []

    def mark(name):
        if timings is not None and cuda:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            ev.append((name, e))

    mark("start")
    if exchange == "auto":
        exchange = "segments" if ops.segment_divisor() else "nccl"
    if exchange == "segments":
        return _segment_local(keys, vals, ops, rank, world, group, mark, ev, timings, cuda)
    n_local = torch.tensor([keys.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = torch.cat(sizes).tolist()  # one host read for all ranks
    idx_base = sum(sizes[:rank])
    if sum(sizes) >= 2 ** 32:
        raise ValueError("global nnz must be < 2^32 (uint32 permutation vector)")
    kbits = key_bits(dims)
    bits = max(1, min(bits, kbits)) if kbits else 1
    hist = ops.key_histogram(keys, bits)
    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    splitters = choose_splitters(hist, world, kbits, bits) if world > 1 else None
    mark("splitters")
    if exchange == "direct":
        return _direct_exchange(keys, vals, ops, splitters, idx_base, world, rank, group, mark,
                                ev, timings, cuda)
    sk, sv, si, send_counts = ops.partition(keys, vals, idx_base, splitters)
    mark("partition")
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    both = torch.cat([send_counts, recv_counts]).tolist()  # one host read
    scnt, rcnt = both[:world], both[world:]
    nrecv = sum(rcnt)
    rk = torch.empty(nrecv, dtype=sk.dtype, device=dev)
    rv = torch.empty(nrecv, dtype=torch.float64, device=dev) if sv is not None else None
    ri = torch.empty(nrecv, dtype=si.dtype, device=dev)
    _exchange((sk, sv, si), (rk, rv, ri), scnt, rcnt, rank, world, group)
    mark("exchange")
    out = ops.permute(rk, rv, ri)
    mark("local_permute")
    if timings is not None:
        timings["sent_bytes"] = int(sum(c for r, c in enumerate(scnt) if r != rank)) * (
            8 + (8 if sv is not None else 0) + 4)
        timings["recv_nnz"] = nrecv
        _collect(ev, timings, cuda, dev)
    return out


def _collect(ev, timings, cuda, dev):
    if cuda:
        torch.cuda.synchronize(dev)
        for (n0, e0), (n1, e1) in zip(ev[:-1], ev[1:]):
            timings[n1] = e0.elapsed_time(e1) / 1e3


def segment_row(keys, D):
    """This rank's (first segment, last segment, head, n): head = the leading nonzeros of
    its slice that lie in its first segment (device tensor, no host read)."""
    dev = keys.device
    n = keys.numel()
    if not n:
        return torch.tensor([-1, -1, 0, 0], dtype=torch.int64, device=dev)
    ends = torch.stack([keys[0], keys[-1]]) // D
    head = torch.searchsorted(keys, (ends[0] + 1) * D).reshape(1)
    return torch.cat([ends, head, torch.tensor([n], device=dev)]).to(torch.int64)


def segment_handover(tab):
    """tab[r] = segment_row of rank r.  A segment belongs to the lowest rank holding any of
    its nonzeros; returns give[r] = (owner, count): rank r hands its first `count` nonzeros
    to rank `owner` (-1, 0 when its slice starts a segment of its own)."""
    world = len(tab)

    def owner(seg):
        for r in range(world):
            if tab[r][3] and tab[r][0] <= seg <= tab[r][1]:
                return r
        return -1

    give = []
    for r in range(world):
        o = owner(tab[r][0]) if tab[r][3] else r
        give.append((o, tab[r][2]) if o != r else (-1, 0))
    return give


def _segment_local(keys, vals, ops, rank, world, group, mark, ev, timings, cuda):
    """Exchange-free sharding of a permutation that keeps identity-prefix segments in place
    ("regions where k is constant" are sorted independently; SURVEY.md §8(c)
    C18: a segment occupies the same positions in input and output).  A segment belongs
    to the lowest rank holding any of its nonzeros; a rank whose slice starts inside a
    segment begun on a lower rank hands that head to the owner (a point-to-point halo of
    at most one segment per rank boundary), then every rank permutes whole segments
    locally.  Its output is the global output over the same index range."""
    dev = keys.device
    D = ops.segment_divisor()
    row = segment_row(keys, D)
    rows = [torch.zeros(4, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(rows, row, group=group)
    tab = torch.stack(rows).tolist()  # [rank] -> (first seg, last seg, head, n): one host read
    sizes = [t[3] for t in tab]
    if sum(sizes) >= 2 ** 32:
        raise ValueError("global nnz must be < 2^32 (uint32 permutation vector)")
    base = [sum(sizes[:r]) for r in range(world)]

    give = segment_handover(tab)
    my_to, my_cnt = give[rank]
    recv_from = [(r, give[r][1]) for r in range(world) if give[r][0] == rank and give[r][1]]
    nrecv = sum(c for _, c in recv_from)
    rk = torch.empty(nrecv, dtype=keys.dtype, device=dev)
    rv = None if vals is None else torch.empty(nrecv, dtype=vals.dtype, device=dev)
    p2p = []
    if my_cnt:
        p2p.append(dist.P2POp(dist.isend, keys[:my_cnt].contiguous(), my_to, group))
        if vals is not None:
            p2p.append(dist.P2POp(dist.isend, vals[:my_cnt].contiguous(), my_to, group))
    off = 0
    for r, c in recv_from:  # ascending source rank = global order
        p2p.append(dist.P2POp(dist.irecv, rk[off:off + c], r, group))
        if vals is not None:
            p2p.append(dist.P2POp(dist.irecv, rv[off:off + c], r, group))
        off += c
    if p2p:
        for req in dist.batch_isend_irecv(p2p):
            req.wait()
    mark("exchange")
    lk = torch.cat([keys[my_cnt:], rk]) if nrecv else keys[my_cnt:]
    lv = None if vals is None else (torch.cat([vals[my_cnt:], rv]) if nrecv else vals[my_cnt:])
    start = base[rank] + my_cnt  # global index of this rank's first local nonzero
    idx = torch.arange(start, start + lk.numel(), dtype=torch.int64, device=dev).to(torch.int32)
    out = ops.permute(lk.contiguous(), None if lv is None else lv.contiguous(), idx)
    mark("local_permute")
    if timings is not None:
        timings["sent_bytes"] = my_cnt * (8 + (8 if vals is not None else 0))
        timings["recv_nnz"] = lk.numel()
        _collect(ev, timings, cuda, dev)
    return out


def _direct_exchange(keys, vals, ops, splitters, idx_base, world, rank, group, mark, ev, timings,
                     cuda):
    """Partition and exchange in one kernel: counts -> all_gather -> each source's offset
    in every receiver (source-rank order = global input order) -> lco_partition_direct
    into the peers' symmetric-memory buffers -> barrier -> local permute.  The receive
    buffers are allocated and rendezvoused once per (group, dtype) and reused."""
    if not cuda:
        raise ValueError("exchange='direct' needs CUDA tensors (peer-mapped device memory)")
    dev = keys.device
    counts = ops.partition_counts(keys, splitters)  # [world] to each destination
    allc = torch.empty(world * world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allc, counts, group=group)
    allc = allc.view(world, world).cpu()  # [src][dst]
    offs = [int(allc[:rank, d].sum()) for d in range(world)]
    nrecv = int(allc[:, rank].sum())
    cap = max(1, int(allc.sum(0).max()))  # symmetric buffers: the same size on every rank
    group_name = (group or dist.group.WORLD).group_name
    bufs = []
    for dt in (torch.int64, torch.float64 if vals is not None else None, torch.int32):
        if dt is None:
            bufs.append(None)
            continue
        c, t, h = ops.symmetric(group_name, dt, cap, dev)
        bufs.append((t, h, c))
    peers = [None if b is None else [b[1].get_buffer(d, (b[2],), b[0].dtype) for d in range(world)]
             for b in bufs]
    ops.partition_direct(keys, vals, idx_base, splitters, peers[0], peers[1], peers[2], offs)
    bufs[0][1].barrier(channel=0)  # every rank's stores have landed
    mark("exchange")
    rk = bufs[0][0][:nrecv]
    rv = None if bufs[1] is None else bufs[1][0][:nrecv]
    ri = bufs[2][0][:nrecv]
    out = ops.permute(rk, rv, ri)
    mark("local_permute")
    if timings is not None:
        timings["sent_bytes"] = int(sum(int(allc[rank, d]) for d in range(world) if d != rank)) * (
            8 + (8 if vals is not None else 0) + 4)
        timings["recv_nnz"] = nrecv
        _collect(ev, timings, cuda, dev)
    return out


def _mode(args, ops):
    m = getattr(args, "exchange", "auto")
    if m == "auto":
        m = "segments" if ops.segment_divisor() else "nccl"
    return m


def bench_main(args):
    """bench.py --gpus N under torchrun: C5 sharded by key range across the ranks.
    One JSON line on rank 0 with the contract's keys; times are CUDA events on each rank,
    max over ranks; the end-to-end number copies every rank's slice from pinned host
    memory and its part of the output back inside the timed region."""
    import json
    import os
    import sys

    import numpy as np

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench as _bench
    import workloads

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world, rank = dist.get_world_size(), dist.get_rank()
    cfg = args.config
    name = cfg[:2]
    w = workloads.config(name, device=dev, scale=args.scale)
    perm = w.perms[1 if cfg.endswith("b") else 0]
    dims = tuple(int(d) for d in w.dims)
    recipe = w.recipe
    n = w.keys.numel()
    lo, hi = n * rank // world, n * (rank + 1) // world
    keys = w.keys[lo:hi].contiguous()
    vals = w.vals[lo:hi].contiguous()
    wname = w.name
    del w
    torch.cuda.empty_cache()
    ops = CudaOps(dims, perm)
    for _ in range(args.warmup):
        permute_sharded(keys, vals, dims, perm, ops=ops, exchange=getattr(args, 'exchange', 'auto'))
    torch.cuda.synchronize()
    clocks = _bench.ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    tms, exch, launches = [], [], 0
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        t = {}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        permute_sharded(keys, vals, dims, perm, ops=ops, timings=t,
                        exchange=getattr(args, 'exchange', 'auto'))
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
        tms.append(e0.elapsed_time(e1) / 1e3)
        exch.append((t.get("exchange", 0.0), t.get("sent_bytes", 0)))
        # this library's kernels per step: (key histogram, partition pass of 4,) local permute
        seg = getattr(args, "exchange", "auto") in ("auto", "segments") and ops.segment_divisor()
        launches += (0 if seg else 1 + 4) + ops.plan.info(t.get("recv_nnz", 0))["launches"]
    clk = clocks.stop() if clocks else None
    mine = torch.tensor([float(np.mean(tms)), float(np.mean([x[0] for x in exch])),
                         float(np.mean([x[1] for x in exch]))], dtype=torch.float64, device=dev)
    mx = mine.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)

    # ---- end to end: pinned host slice in, this rank's output back, every step ----
    e2e = None
    if not getattr(args, "no_e2e", False):
        hk, hv = keys.cpu().pin_memory(), vals.cpu().pin_memory()
        del keys, vals
        torch.cuda.empty_cache()
        e2e_steps = max(1, min(args.steps, 3))
        ems, hbytes, dbytes = [], 0, 0
        dk, dv = torch.empty_like(hk, device=dev), torch.empty_like(hv, device=dev)
        outs = None
        for _ in range(e2e_steps + 1):  # the first round sizes the pinned outputs
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dk.copy_(hk, non_blocking=True)
            dv.copy_(hv, non_blocking=True)
            ko, vo, po = permute_sharded(dk, dv, dims, perm, ops=ops,
                                         exchange=getattr(args, 'exchange', 'auto'))
            if outs is None:
                outs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (ko, vo, po)]
            for h, d in zip(outs, (ko, vo, po)):
                h.copy_(d, non_blocking=True)
            b.record()
            torch.cuda.synchronize()
            dist.barrier()
            ems.append(a.elapsed_time(b) / 1e3)
            hbytes, dbytes = 16 * hk.numel(), 20 * ko.numel()
        ems = ems[1:]
        em = torch.tensor([float(np.mean(ems)), float(hbytes), float(dbytes)], dtype=torch.float64,
                          device=dev)
        dist.all_reduce(em, op=dist.ReduceOp.MAX)
        e2e = {"value": n / float(em[0]), "unit": "nonzeros/s",
               "h2d_bytes_per_step": int(float(em[1])) * world,
               "d2h_bytes_per_step": int(float(em[2])) * world,
               "ms_per_step": float(em[0]) * 1e3,
               "api": "permute_sharded on pinned host slices (H2D, sharded permute, D2H)"}
    cpu = None
    if rank == 0 and not getattr(args, "no_cpu", False):
        # the CPU oracle (1 core and all cores) on a strided sample of rank 0's slice,
        # itself a sorted LCO tensor of the same workload
        import types
        sl = types.SimpleNamespace(keys=hk if e2e is not None else keys.cpu(),
                                   vals=hv if e2e is not None else vals.cpu(), dims=dims,
                                   name=f"{wname} (rank 0 slice)")
        cpu = _bench.oracle_baseline(sl, perm, max_nnz=getattr(args, "cpu_nnz", 40_000_000))
    if rank == 0:
        sec = float(mx[0])
        t_ex, sent = float(mx[1]), float(mx[2])
        nvlink = (sent / t_ex / 900e9) if t_ex > 0 else None
        peak, peak_src = _bench.peaks()
        # 32 B per nonzero (read K + V, write K' + V) of each GPU's share
        # over the step time (the exchange crosses NVLink, reported separately)
        achieved = 32.0 * n / world / sec / 1e9
        line = {
            "metric": "nonzeros permuted/sec and achieved HBM GB/s fraction at 1/2/4/8 B200",
            "value": n / sec, "unit": "nonzeros/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "u64 keys / f64 values (moved, bit-exact)", "data": "synthetic",
            "config": {"workload": f"{cfg}: {recipe}; perm {tuple(perm)}; sharded by key range "
                                   f"over {world} GPUs", "nnz": n,
                       "parallelism": f"key-range sharding x{world} ("
                                      + {"direct": "partition stores into peer symmetric memory",
                                         "nccl": "partition + grouped NCCL send/recv",
                                         "segments": "exchange-free: identity-prefix segments "
                                                     "stay in place, boundary halo only"}[
                                          _mode(args, ops)] + ")",
                       "l2": "inputs >> L2"},
            "exchange": {"seconds": t_ex, "sent_bytes_per_gpu": sent,
                         "nvlink_frac_of_900GBps": nvlink},
            "hbm_frac": achieved / peak,
            "roofline": {"bound": "hbm", "kernel": "sharded step (per GPU: partition, exchange, "
                                                   "local permute)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "alg_bytes_per_nnz": 32,
                         "frac_36B": 36.0 * n / world / sec / 1e9 / peak,
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
