#!/usr/bin/env python
"""GPU analogue of the paper's permutation experiment (§4.2, Fig 4, Table 2;
SURVEY §8(f) NEXT 1): every one of the 23 non-identity permutations of a 4th-order
tensor, permuted with RP (lco_permute: stable radix over only the disturbed digits of
the shaved key) versus a full stable radix sort of the shuffled keys (lco_sort: all key
digits), on (a) the combinatorial Laplacian of Eq (2.3) at N = 2^11.5 ~ 2896 (Table 2's
size, ~42M nonzeros) and (b) a 2%-fill tensor.  Both produce identical outputs, and the
RP output passes the output certificate (perm bijection, key = re-encode of its source,
value bits, strictly increasing keys) -- both checked on every permutation.  Times are
CUDA-event medians with inputs resident in HBM.

    python benchmarks/table2.py [--n 2896] [--fill-n 200] [--reps 5] [--out profiles/...]
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1802_02619_b200 as lco  # noqa: E402
import workloads  # noqa: E402

# Table 2, paper lex orders (least significant first)
TABLE2 = {(3, 1, 2, 0): ("Max", 3.50, 3.54), (2, 1, 3, 0): ("Median", 3.54, 3.45),
          (1, 0, 2, 3): ("Min", 2.71, 1.38)}


def lex_to_perm(lex):
    n = len(lex)
    return tuple(n - 1 - lex[n - 1 - t] for t in range(n))


def perm_to_lex(perm):
    n = len(perm)
    return tuple(n - 1 - perm[n - 1 - t] for t in range(n))


def timed(fn, reps):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    fn()
    torch.cuda.synchronize()
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


def _reencode(keys, dims, perm):
    """K' of every key by torch integer ops (decode from the last mode, Horner under the
    new order): an independent check of the library's LIV shuffle."""
    c = [None] * len(dims)
    k = keys.clone()
    for m in range(len(dims) - 1, -1, -1):
        c[m] = k % dims[m]
        k = k // dims[m]
    out = torch.zeros_like(keys)
    for p in perm:
        out = out * dims[p] + c[p]
    return out


def certified(keys, vals, dims, perm, out):
    """The output certificate (with unique input keys it implies equality with the
    definition): perm a bijection, key = re-encode(source key), value bits of the source,
    keys strictly increasing."""
    ko, vo, po = out
    n = keys.numel()
    src = po.long()
    return bool(torch.equal(torch.sort(src).values, torch.arange(n, device=keys.device))
                and torch.equal(ko, _reencode(keys[src], dims, perm))
                and torch.equal(vo.view(torch.int64), vals[src].view(torch.int64))
                and bool((ko[1:] > ko[:-1]).all()))


def run(name, keys, vals, dims, reps):
    n = keys.numel()
    rows = []
    for perm in itertools.permutations(range(4)):
        if perm == (0, 1, 2, 3):
            continue
        p = lco.Plan(dims, perm)
        ws = torch.empty(p.workspace_size(n) + 256, dtype=torch.uint8, device=keys.device)
        out_p = (torch.empty_like(keys), torch.empty_like(vals),
                 torch.empty(n, dtype=torch.int32, device=keys.device))
        out_s = (torch.empty_like(keys), torch.empty_like(vals),
                 torch.empty(n, dtype=torch.int32, device=keys.device))
        t_rp = timed(lambda: p.permute(keys, vals, out=out_p, workspace=ws), reps)
        t_sort = timed(lambda: p.sort(keys, vals, out=out_s, workspace=ws), reps)
        same = all(torch.equal(x, y) for x, y in zip(out_p, out_s)) and \
            certified(keys, vals, dims, perm, out_p)
        ip, isr = p.info(n), p.info(n, sort=True)
        # the hierarchical plan (LCO_FLAG_HIERARCHICAL): one stable sort per run of
        # rearrangement indices, where the permutation has >= 2 runs
        t_h, h_paths = None, None
        if ip["stages"] >= 2:
            ph = lco.Plan(dims, perm, hierarchical=True)
            wsh = torch.empty(ph.workspace_size(n) + 256, dtype=torch.uint8, device=keys.device)
            out_h = (torch.empty_like(keys), torch.empty_like(vals),
                     torch.empty(n, dtype=torch.int32, device=keys.device))
            t_h = timed(lambda: ph.permute(keys, vals, out=out_h, workspace=wsh), reps)
            same = same and all(torch.equal(x, y) for x, y in zip(out_p, out_h))
            h_paths = ph.info(n)["stage_paths"]
            del wsh, out_h
        lex = perm_to_lex(perm)
        rows.append({"tensor": name, "perm": perm, "paper_lex": lex,
                     "rearrangement_indices": sum(ip["rearrangement"]),
                     "rp_ms": t_rp, "sort_ms": t_sort, "speedup": t_sort / t_rp,
                     "rp_bits": ip["sort_bits"], "sort_bits": isr["sort_bits"],
                     "rp_path": ip["path"], "sort_path": isr["path"], "identical": same,
                     "hier_ms": t_h, "hier_stage_paths": h_paths,
                     "paper": TABLE2.get(lex)})
        del ws, out_p, out_s
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2896)
    ap.add_argument("--fill-n", type=int, default=200)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    k, v = workloads.combinatorial_laplacian(args.n, device=dev)
    rows = run(f"laplacian N={args.n} ({k.numel()} nnz)", k, v, (args.n,) * 4, args.reps)
    del k, v
    k, v = workloads.fill_tensor(args.fill_n, 0.02, seed=3, device=dev)
    rows += run(f"2% fill N={args.fill_n} ({k.numel()} nnz)", k, v, (args.fill_n,) * 4, args.reps)
    lines = ["| tensor | perm (row-major) | paper lex | R idx | RP bits | sort bits | RP path | "
             "RP ms | sort ms | sort/RP | staged RP ms (stage paths) | identical | "
             "paper (MSD s / RP s) |", "|" + "---|" * 13]
    for r in rows:
        pap = "" if not r["paper"] else f"{r['paper'][0]}: {r['paper'][1]} / {r['paper'][2]}"
        hier = "" if r["hier_ms"] is None else f"{r['hier_ms']:.3f} ({'+'.join(r['hier_stage_paths'])})"
        lines.append(f"| {r['tensor']} | {r['perm']} | {r['paper_lex']} | "
                     f"{r['rearrangement_indices']} | {r['rp_bits']} | {r['sort_bits']} | "
                     f"{r['rp_path']} | {r['rp_ms']:.3f} | {r['sort_ms']:.3f} | "
                     f"{r['speedup']:.2f} | {hier} | {r['identical']} | {pap} |")
    text = "\n".join(lines)
    print(text)
    for name in {r["tensor"] for r in rows}:
        sp = sorted(r["speedup"] for r in rows if r["tensor"] == name)
        print(f"{name}: sort/RP min {sp[0]:.2f} median {sp[len(sp) // 2]:.2f} max {sp[-1]:.2f}")
    if args.out:
        with open(args.out, "w") as f:
            f.write(text + "\n")
        with open(args.out.replace(".md", ".json"), "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
