#!/usr/bin/env python
"""GPU analogue of the paper's addition experiment (Fig 2(c)): the two
order-4 terms of Eq (2.3) on an N x N image, the second re-sorted into the {1,0,3,2}
order and added (lco_add = lco_permute + merge of two sorted LIV streams).  Reports the
permutation and merge times, the share the permutation takes of the whole operation
(the paper: 65 % for LCO on the CPU), nonzeros/s and the merge kernel's achieved HBM
bandwidth (algorithmic bytes: read A and B' keys+values, write C keys+values) against
MEASURED_PEAKS.json.  Inputs resident in HBM; CUDA events.  The result is checked
against the closed form (the combinatorial Laplacian).

    python benchmarks/addition.py [--n 2896 1024 ...] [--reps 10] [--out profiles/...json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1802_02619_b200 as lco  # noqa: E402
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[1024, 2048, 2896])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--hierarchical", action="store_true",
                    help="permute B with the staged plan (LCO_FLAG_HIERARCHICAL)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = []
    for n in args.n:
        k, v = workloads.eq23_term(n, device=dev)
        p = lco.plan((n,) * 4, (1, 0, 3, 2), hierarchical=args.hierarchical)
        na = nb = k.numel()
        ws = torch.empty(p.add_workspace_size(na, nb) + 256, dtype=torch.uint8, device=dev)
        kc = torch.empty(na + nb, dtype=torch.int64, device=dev)
        vc = torch.empty(na + nb, dtype=torch.float64, device=dev)
        nc = torch.zeros(1, dtype=torch.int64, device=dev)
        out = (kc, vc, nc)
        for _ in range(3):
            p.add(k, v, k, v, 1.0, out=out, workspace=ws, trim=False)
        torch.cuda.synchronize()
        p.profile_enable(args.reps * 2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            p.add(k, v, k, v, 1.0, out=out, workspace=ws, trim=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        names, calls = p.profile_read()
        p.profile_enable(0)
        # calls alternate: permute (B -> A's order), then the merge
        t_perm = float(np.mean([sum(c) for c in calls[0::2]]))
        t_merge = float(np.mean([sum(c) for c in calls[1::2]]))
        m = int(nc.item())
        ek, ev = workloads.combinatorial_laplacian(n, device=dev)
        ok = m == ek.numel() and torch.equal(kc[:m], ek) and torch.equal(vc[:m], ev)
        merge_bytes = 16 * (na + nb) + 16 * m
        row = {"n": n, "hierarchical": args.hierarchical, "permute_path": p.info(nb)["path"],
               "nnz_a": na, "nnz_b": nb, "nnz_c": m, "ms": ms, "permute_ms": t_perm,
               "merge_ms": t_merge, "permute_share": t_perm / (t_perm + t_merge),
               "nnz_per_s": (na + nb) / (ms / 1e3),
               "merge_gbs": merge_bytes / (t_merge / 1e3) / 1e9,
               "merge_frac": merge_bytes / (t_merge / 1e3) / 1e9 / peak,
               "permute_gbs": 36 * nb / (t_perm / 1e3) / 1e9,
               "closed_form_ok": bool(ok), "peak_gbs": peak}
        print(json.dumps(row), flush=True)
        rows.append(row)
        del ws, kc, vc, k, v
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
