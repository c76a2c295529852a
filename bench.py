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

# Algorithmic bytes: read key + value, write key + value = 32 B per
# nonzero, 36 B with the uint32 permutation vector.  Every roofline fraction below is
# (these bytes x the nonzeros one launch / one step processes) / time / measured peak --
# the same figure for the dominant kernel and for the step, so that a kernel's own extra
# traffic (carried positions, re-reads) lowers its fraction instead of inflating it.
ALG_BYTES = 32
ALG_BYTES_PERM = 36
# The bytes each kernel itself must move at minimum, reported beside the
# fraction for context only.
KERNEL_MODEL_BYTES = {
    "k_count_first": 8, "k_count": 8, "k_count_seg": 8,
    "k_scatter_first": 36, "k_scatter_single": 36, "k_scatter_mid": 40, "k_scatter_seg": 40,
    "k_scatter_last": 40, "k_leafw": 40, "k_leafw_l1": 40, "k_leafr": 40, "k_leafs": 40,
    "k_leafc": 40, "k_leafs_l1": 40, "k_leafr_l1": 40, "k_leafc_l1": 40, "k_leafc_tiles": 36,
    "k_leaf_deferred": 40, "k_copy": 36, "k_block_bounds": 8, "k_block_tiles": 36,
    "k_partition": 36,
}

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


def traffic_of(config, marker):
    """DRAM bytes (read + write) per launch of the kernel behind `marker`, from one ncu
    capture (profiles/traffic.json, written by scripts/save_profiles.py, which matches
    every bench marker to the launch of the same kernel name in ncu's launch list)."""
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        e = json.load(open(tpath)).get(config, {}).get(marker)
    except Exception:  # noqa: BLE001
        return None
    if isinstance(e, dict):
        return e.get("bytes")
    return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_baseline(w, perm, max_nnz=40_000_000):
    """Time the CPU oracle as it stands on a strided sample of the workload (itself a
    sorted LCO tensor): the single-core definition and the same
    definition on every core of the process affinity mask (§8(d)(ii): OpenMP decode /
    gather, __gnu_parallel::stable_sort)."""
    import oracle
    n = w.keys.numel()
    stride = max(1, -(-n // max_nnz))
    ks = w.keys[::stride].cpu().numpy().view(np.uint64).copy()
    vs = w.vals[::stride].cpu().numpy().copy()
    oracle.permute(w.dims, perm, ks[:1000], vs[:1000])  # load / warm
    t0 = time.perf_counter()
    oracle.permute(w.dims, perm, ks, vs)
    dt = time.perf_counter() - t0
    sample = (f"every {stride}th nonzero of the sorted {w.name} input ({len(ks)} nnz, itself a "
              f"sorted LCO tensor), one oracle permute call (decode / re-encode / stable sort / "
              f"gather)")
    out = {"value": len(ks) / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"{sample}, {dt:.2f} s", "cpu_model": cpu_model()}
    try:
        threads = oracle.par_threads()
        oracle.permute_par(w.dims, perm, ks[:100_000], vs[:100_000])  # load / warm
        t0 = time.perf_counter()
        oracle.permute_par(w.dims, perm, ks, vs)
        dp = time.perf_counter() - t0
        out["all_cores"] = {"value": len(ks) / dp, "unit": UNIT, "cores": threads,
                            "affinity_cpus": len(os.sched_getaffinity(0)),
                            "kind": "oracle (OpenMP + __gnu_parallel::stable_sort)",
                            "sample": f"{sample}, {dp:.2f} s"}
    except Exception as ex:  # noqa: BLE001
        out["all_cores"] = {"error": repr(ex)[:200]}
    return out


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

    # The timed step replays one CUDA graph of the lco_permute call (every kernel of the
    # call, same buffers: launch latency and host overhead removed); the
    # per-kernel times come from the same call launched directly (graphs hide them).
    graph = None
    if not args.no_graph:
        graph = p.graph(w.keys, w.vals, out=out, workspace=ws)
        torch.cuda.synchronize()

    def timed(steps, outs, do_flush, profile=False, sample_clocks=False, use_graph=False):
        """CUDA events on the launching stream around each step; L2 flushed before each
        step when do_flush (inputs smaller than 4x L2)."""
        if profile:
            p.profile_enable(steps)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        clocks = ClockSampler(0) if sample_clocks else None
        if clocks:
            clocks.start()
            time.sleep(0.3)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for st in range(steps):
            if do_flush:
                fbuf.fill_(float(st))
            ev[st][0].record(stream)
            if use_graph:
                graph.replay()
            else:
                p.permute(w.keys, w.vals, out=outs, workspace=ws)
            ev[st][1].record(stream)
        torch.cuda.synchronize()
        wall_s = time.perf_counter() - w0
        clk_ = clocks.stop() if clocks else None
        return [x.elapsed_time(y) for x, y in ev], wall_s, clk_

    direct_ms, _, _ = timed(args.steps, out, flush, profile=True)
    names, rows = p.profile_read()
    p.profile_enable(0)
    step_ms, wall, clk = timed(args.steps, out, flush, sample_clocks=True,
                               use_graph=graph is not None)
    ms = float(np.mean(step_ms))
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
    # 32 B x the nonzeros one launch processes (every launch of the
    # dominant kernel here processes all n), over that kernel's CUDA-event launch time
    achieved = ALG_BYTES * n / (dom_launch_ms / 1e3) / 1e9
    traffic = traffic_of(args.config, dom)
    step_achieved = ALG_BYTES * n / (ms / 1e3) / 1e9
    value = n / (ms / 1e3)
    # secondary figures: without the permutation vector (40 B/nnz schedule
    # row), and for sub-L2 inputs the L2-warm time beside the flushed (cold) one
    extra = {"direct_launch": {"ms_per_step": float(np.mean(direct_ms)),
                               "value": n / (float(np.mean(direct_ms)) / 1e3),
                               "note": "the same call launched kernel by kernel (no graph)"}}
    np_ms, _, _ = timed(max(3, args.steps // 2), (ko, vo, None), flush)
    extra["no_perm"] = {"ms_per_step": float(np.mean(np_ms)),
                        "value": n / (float(np.mean(np_ms)) / 1e3),
                        "step_frac_32B": ALG_BYTES * n / (float(np.mean(np_ms)) / 1e3) / 1e9 / peak}
    if flush:
        wm, _, _ = timed(args.steps, out, False, use_graph=graph is not None)
        extra["l2_warm"] = {"ms_per_step": float(np.mean(wm)), "value": n / (float(np.mean(wm)) / 1e3),
                            "note": "inputs left in L2 between steps (no flush)"}
        extra["l2_cold"] = {"ms_per_step": ms, "value": value,
                            "note": "L2 flushed before every step (the headline)"}

    used_graph = graph is not None
    graph = None  # releases the captured buffers' references
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
                   "step": ("one CUDA-graph replay of the lco_permute call" if used_graph
                            else "one lco_permute call"),
                   "plan": {k: info[k] for k in ("sort_bits", "passes", "digit_bits",
                                                  "radix_bits", "path", "tile")}},
        "hbm_frac": step_achieved / peak,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "alg_bytes_per_nnz": ALG_BYTES, "alg_bytes_per_launch": ALG_BYTES * n,
                     "frac_36B": ALG_BYTES_PERM * n / (dom_launch_ms / 1e3) / 1e9 / peak,
                     "launch_ms": dom_launch_ms, "launch_share_of_step": tot[dom] / ms,
                     "kernel_model_bytes_per_nnz": KERNEL_MODEL_BYTES.get(dom),
                     "peak_source": peak_src},
        "step_roofline": {"alg_bytes_per_nnz": ALG_BYTES, "achieved": step_achieved,
                          "peak": peak, "unit": "GB/s", "frac": step_achieved / peak,
                          "frac_36B": ALG_BYTES_PERM * n / (ms / 1e3) / 1e9 / peak},
        **extra,
        "kernels_ms": {k: round(v, 4) for k, v in tot.items()},
        "markers": names,
        "cpu_baseline": cpu,
        "e2e": e2e,
        # one profiling marker per kernel launch of the call (lco_profile), times steps
        "gpu_launches": (len(names) if names else info["launches"]) * args.steps,
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
    ap.add_argument("--no-graph", action="store_true",
                    help="time the call launched kernel by kernel instead of a CUDA-graph replay")
    ap.add_argument("--exchange", default="auto", choices=["auto", "segments", "nccl", "direct"],
                    help="N > 1: auto (segments when identity-prefix segments stay in place, "
                         "else nccl), the exchange-free segment path, partition + one grouped "
                         "NCCL exchange, or the partition storing straight into the peers' "
                         "symmetric memory (lco_partition_direct)")
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
