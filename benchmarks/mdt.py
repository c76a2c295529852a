#!/usr/bin/env python
"""Steps 1-2 of a sparse tensor product (§5.2, :325-331) on B200: flatten a
tensor into an LCO matrix (the permutation hot path) and compress it into CSR / DCSR
(lco_compress).  Workloads: C4 (2048^4 biharmonic operator, 54.5M nonzeros) flattened
rows {y, x} x cols {x', y'} (= BASELINE C4's permutation), and a hyper-sparse random
order-5 tensor flattened with 3 modes to rows (row-sparse: DCSR).  Reports times, the
compress kernels' achieved HBM bandwidth (algorithmic bytes: read the keys, write minor
indices + pointers) against MEASURED_PEAKS.json, and the hyper-sparsity class.

    python benchmarks/mdt.py [--reps 10] [--out profiles/...json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1802_02619_b200 as lco  # noqa: E402
import workloads  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = []
    cases = []
    w = workloads.config("C4", device=dev)
    cases.append(("C4 biharmonic 2048^4, rows (y, x) x cols (x', y')", w.keys, w.vals, w.dims,
                  (1, 0), (2, 3)))
    k, v = workloads.random_tensor((1024,) * 5, 20_000_000, seed=11, device=dev)
    cases.append(("random 1024^5, 20M nnz, rows (0, 1, 2) x cols (3, 4)", k, v, (1024,) * 5,
                  (0, 1, 2), (3, 4)))
    for name, keys, vals, dims, r, c in cases:
        nnz = keys.numel()
        km, vm, m, n = lco.flatten(keys, vals, dims, r, c)
        t_flat = timed(lambda: lco.flatten(keys, vals, dims, r, c), args.reps)
        cls = lco.sparsity_class(m, n, nnz)
        row = {"case": name, "nnz": nnz, "m": m, "n": n, "class": cls, "flatten_ms": t_flat}
        t_d = timed(lambda: lco.compress(km, m, n, doubly=True), args.reps)
        d = lco.compress(km, m, n, doubly=True)
        row.update({"dcsr_ms": t_d, "nonempty_rows": d["nz"],
                    "dcsr_gbs": (16 * nnz + 16 * d["nz"]) / (t_d / 1e3) / 1e9})
        if m <= nnz * 4:
            t_s = timed(lambda: lco.compress(km, m, n), args.reps)
            row.update({"csr_ms": t_s, "csr_gbs": (16 * nnz + 8 * (m + 1)) / (t_s / 1e3) / 1e9})
        row["peak_gbs"] = peak
        print(json.dumps(row), flush=True)
        rows.append(row)
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
