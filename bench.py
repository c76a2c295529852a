#!/usr/bin/env python
"""Benchmark of the LCO permutation hot path (BASELINE.json metric: nonzeros permuted/s
and achieved HBM fraction).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]

Default workload: BASELINE config C5 (the config the metric is quoted on at 1/2/4/8
GPUs): order-5 4096^5 tensor, 500M unique uniform keys, N(0,1) values, permutation
(4,3,2,1,0).  One step = one lco_permute of the whole tensor (all §8(a) rows: decode,
re-encode, digit histograms, stable radix passes, value gather), inputs resident in
HBM.  Prints ONE JSON line on rank 0.  N > 1 (torchrun) runs the key-range sharded
path (paper_1802_02619_b200.sharded).

--impl reference times the CPU oracle (oracle/, single core, as it stands) on a bounded
sample of the same workload; this repo has no runnable upstream implementation.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "nonzeros permuted/sec and achieved HBM GB/s fraction at 1/2/4/8 B200"
UNIT = "nonzeros/s"

# Algorithmic bytes per nonzero of each kernel: the bytes the
# kernel must move at minimum for the work it does (reads + writes, perm included).
KERNEL_BYTES = {
    "k_count_first": 8,       # read K (LIV shuffle + digit histogram)
    "k_count": 8,             # read K'
    "k_count_seg": 8,         # read K'
    "k_scatter_first": 36,    # read K, V; write K', V, position
    "k_scatter_single": 36,   # read K, V; write K', V, perm
    "k_scatter_mid": 40,      # read K', V, position; write them
    "k_scatter_seg": 40,
    "k_scatter_last": 40,
    "k_leafw": 40,            # read K', V, position; write K', V, perm (final)
    "k_leafw_l1": 40,
    "k_leafr": 40,            # CTA leaves, 32-bit sort keys (read K', V, pos; write)
    "k_leafs": 40,            # CTA leaves, fully staged
    "k_leafc": 40,            # CTA leaves, 64-bit sort keys
    "k_leaf_l1": 40,
    "k_leafc_tiles": 36,      # segment-local tiles: read K, V; write K', V, perm
    "k_leaf": 36,
    "k_leaf_deferred": 40,
    "k_copy": 36,             # read K, V; write K, V, perm
    "k_block_bounds": 8,      # read K (run bounds of the blocks)
    "k_block_tiles": 36,      # read K, V; write K', V, perm (tiled transpose of runs)
    "k_partition": 36,
}
STEP_BYTES = 36  # read K+V, write K'+V (32) + the uint32 perm (4)

CONFIGS = {
    # name: (workloads config, perm index)
    "C1": ("C1", 0), "C2a": ("C2", 0), "C2b": ("C2", 1), "C3a": ("C3", 0), "C3b": ("C3", 1),
    "C4": ("C4", 0), "C5": ("C5", 0),
}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        self.thread.join(1)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def oracle_baseline(w, perm, target_s=15.0, max_nnz=40_000_000):
    """Time the CPU oracle (1 core, as it stands) on a strided sample of the workload."""
    import oracle
    n = w.keys.numel()
    stride = max(1, -(-n // max_nnz))
    ks = w.keys[::stride].cpu().numpy().view(np.uint64).copy()
    vs = w.vals[::stride].cpu().numpy().copy()
    oracle.permute(w.dims, perm, ks[:1000], vs[:1000])  # load / warm
    t0 = time.perf_counter()
    oracle.permute(w.dims, perm, ks, vs)
    dt = time.perf_counter() - t0
    return {"value": len(ks) / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"every {stride}th nonzero of the sorted {w.name} input "
                      f"({len(ks)} nnz, itself a sorted LCO tensor), one oracle.permute call "
                      f"(decode / re-encode / std::stable_sort / gather), {dt:.2f} s"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle  # noqa: F401
    import workloads
    cfg, pi = CONFIGS[args.config]
    w = workloads.config(cfg, device="cuda" if torch.cuda.is_available() else "cpu")
    perm = w.perms[pi]
    n = w.keys.numel()
    sample = min(n, args.ref_nnz)
    stride = max(1, n // sample)
    ks = w.keys[::stride][:sample].cpu().numpy().view(np.uint64).copy()
    vs = w.vals[::stride][:sample].cpu().numpy().copy()
    import oracle as orc
    for _ in range(args.warmup):
        orc.permute(w.dims, perm, ks[:100_000], vs[:100_000])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        orc.permute(w.dims, perm, ks, vs)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    value = len(ks) / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 keys / f64 values (moved)",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {w.recipe}; perm {perm}",
                   "nnz": n, "sample_nnz": len(ks)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"every {stride}th nonzero of the sorted input "
                                   f"({len(ks)} nnz) per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def run_single(args):
    import paper_1802_02619_b200 as lco
    import workloads
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    cfg, pi = CONFIGS[args.config]
    t0 = time.time()
    w = workloads.config(cfg, device=dev, scale=args.scale)
    gen_s = time.time() - t0
    perm = w.perms[pi]
    n = w.keys.numel()
    p = lco.plan(w.dims, perm)
    info = p.info(n)
    ws = torch.empty(p.workspace_size(n) + 256, dtype=torch.uint8, device=dev)
    ko = torch.empty_like(w.keys)
    vo = torch.empty_like(w.vals)
    po = torch.empty(n, dtype=torch.int32, device=dev)
    out = (ko, vo, po)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    in_bytes = n * 16
    flush = in_bytes < 4 * l2_bytes
    fbuf = torch.empty(2 * l2_bytes // 4 + 1, dtype=torch.float32, device=dev) if flush else None
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        p.permute(w.keys, w.vals, out=out, workspace=ws)
    torch.cuda.synchronize()
    p.profile_enable(args.steps)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for s in range(args.steps):
        if flush:
            fbuf.fill_(float(s))
        ev[s][0].record(stream)
        p.permute(w.keys, w.vals, out=out, workspace=ws)
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(step_ms))
    names, rows = p.profile_read()
    p.profile_enable(0)
    counts = {}
    for nm in names:
        counts[nm] = counts.get(nm, 0) + 1
    per_call = {}
    for c in rows:
        acc = {}
        for nm, t in zip(names, c):
            acc[nm] = acc.get(nm, 0.0) + t
        for nm, t in acc.items():
            per_call.setdefault(nm, []).append(t)
    tot = {nm: float(np.mean(v)) for nm, v in per_call.items()}
    kernels_only = {k: v for k, v in tot.items() if k.startswith("k_")}
    dom = max(kernels_only, key=kernels_only.get)
    dom_launch_ms = tot[dom] / counts[dom]
    peak, peak_src = peaks()
    alg = KERNEL_BYTES.get(dom, STEP_BYTES) * n
    achieved = alg / (dom_launch_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config, {}).get(dom)
        except Exception:
            traffic = None
    step_achieved = STEP_BYTES * n / (ms / 1e3) / 1e9
    value = n / (ms / 1e3)

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        try:
            kh = w.keys.cpu().pin_memory()
            vh = w.vals.cpu().pin_memory()
            hko = torch.empty_like(kh).pin_memory()
            hvo = torch.empty_like(vh).pin_memory()
            hpo = torch.empty(n, dtype=torch.int32).pin_memory()
            del ws
            hws = torch.empty(p.host_workspace_size(n) + 256, dtype=torch.uint8, device=dev)
            p.permute_host(kh, vh, out=(hko, hvo, hpo), workspace=hws, device=dev)
            torch.cuda.synchronize()
            e2e_steps = max(1, min(args.steps, 3))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(e2e_steps):
                p.permute_host(kh, vh, out=(hko, hvo, hpo), workspace=hws, device=dev)
            e1.record(stream)
            torch.cuda.synchronize()
            ems = e0.elapsed_time(e1) / e2e_steps
            ok = bool(torch.equal(hko, ko.cpu()) and torch.equal(hpo, po.cpu()))
            e2e = {"value": n / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": 16 * n,
                   "d2h_bytes_per_step": 20 * n, "ms_per_step": ems, "matches_device": ok,
                   "api": "lco_permute_host (pinned host buffers, H2D+permute+D2H per step)"}
            # Pipelined: consecutive (independent) steps on two streams with their own
            # workspaces and host outputs (the ABI allows a handle on several streams), so
            # one step's D2H overlaps the next one's H2D on the full-duplex host link.
            if not args.e2e_sequential:
                try:
                    hws2 = torch.empty(p.host_workspace_size(n) + 256, dtype=torch.uint8, device=dev)
                    outs = [(hko, hvo, hpo), (torch.empty_like(hko).pin_memory(),
                                              torch.empty_like(hvo).pin_memory(),
                                              torch.empty_like(hpo).pin_memory())]
                    wss = [hws, hws2]
                    sts = [stream, torch.cuda.Stream(device=dev)]
                    torch.cuda.synchronize()
                    p.permute_host(kh, vh, out=outs[1], workspace=wss[1], device=dev, stream=sts[1])
                    torch.cuda.synchronize()
                    psteps = max(2, min(args.steps, 8))
                    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    f0.record(sts[0])
                    sts[1].wait_event(f0)
                    for i in range(psteps):
                        j = i % 2
                        p.permute_host(kh, vh, out=outs[j], workspace=wss[j], device=dev, stream=sts[j])
                    done1 = torch.cuda.Event()
                    done1.record(sts[1])
                    sts[0].wait_event(done1)
                    f1.record(sts[0])
                    torch.cuda.synchronize()
                    pms = f0.elapsed_time(f1) / psteps
                    ok2 = all(bool(torch.equal(o[0], ko.cpu()) and torch.equal(o[2], po.cpu()))
                              for o in outs)
                    e2e.update({"value": n / (pms / 1e3), "ms_per_step": pms,
                                "matches_device": ok and ok2, "pipeline_streams": 2,
                                "sequential_value": n / (ems / 1e3), "sequential_ms_per_step": ems,
                                "api": "lco_permute_host (pinned host buffers, H2D+permute+D2H "
                                       "per step; consecutive steps alternate two streams)"})
                    del hws2, outs
                except Exception as ex:  # noqa: BLE001
                    e2e["pipeline_error"] = repr(ex)[:200]
            del hws
        except Exception as ex:  # noqa: BLE001
            e2e = {"value": None, "unit": UNIT, "error": repr(ex)[:200]}

    cpu = None
    if not args.no_cpu:
        cpu = oracle_baseline(w, perm, max_nnz=args.cpu_nnz)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64 keys / f64 values (moved, bit-exact)",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {w.recipe}; perm {perm}", "nnz": n,
                   "dims": list(w.dims), "perm": list(perm), "parallelism": "single GPU",
                   "l2": ("L2 flushed between steps" if flush else
                          f"inputs {in_bytes / 1e9:.1f} GB >> L2 {l2_bytes / 1e6:.0f} MB"),
                   "plan": {k: info[k] for k in ("sort_bits", "passes", "digit_bits",
                                                  "radix_bits", "path", "tile")}},
        "hbm_frac": step_achieved / peak,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "alg_bytes_per_nnz": KERNEL_BYTES.get(dom), "launch_ms": dom_launch_ms,
                     "peak_source": peak_src},
        "step_roofline": {"alg_bytes_per_nnz": STEP_BYTES, "achieved": step_achieved,
                          "peak": peak, "unit": "GB/s", "frac": step_achieved / peak},
        "kernels_ms": {k: round(v, 4) for k, v in tot.items()},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": info["launches"] * args.steps,
        "clocks": clk,
        "wall_s_timed": wall,
        "gen_s": gen_s,
        "gpu": torch.cuda.get_device_name(dev),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-sequential", action="store_true",
                    help="e2e: one stream only (no overlap of consecutive steps)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "direct"],
                    help="N > 1: NCCL all_to_all after the partition, or the partition storing "
                         "straight into the peers' symmetric memory (lco_partition_direct)")
    ap.add_argument("--cpu-nnz", type=int, default=40_000_000)
    ap.add_argument("--ref-nnz", type=int, default=20_000_000)
    ap.add_argument("--scale", type=int, default=None,
                    help="shrink the workload (grid size / nnz) for profiling runs")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    world, rank, local = dist_env()
    if world > 1:
        from paper_1802_02619_b200 import sharded
        sharded.bench_main(args)
        return
    run_single(args)


if __name__ == "__main__":
    main()
