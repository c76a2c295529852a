"""Per-kernel CUDA-event times of one permutation: python scripts/kprof.py laplacian 2896 3,1,2,0 [sort]"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1802_02619_b200 as lco
import workloads

kind, n, perm = sys.argv[1], int(sys.argv[2]), tuple(int(x) for x in sys.argv[3].split(","))
sort = len(sys.argv) > 4 and sys.argv[4] == "sort"
if kind == "laplacian":
    k, v = workloads.combinatorial_laplacian(n, device="cuda")
    dims = (n,) * 4
else:
    w = workloads.config(kind, device="cuda", scale=None if n == 0 else n)
    k, v, dims = w.keys, w.vals, w.dims
p = lco.plan(dims, perm)
fn = p.sort if sort else p.permute
print(p.info(k.numel(), sort=sort))
for _ in range(3):
    fn(k, v)
torch.cuda.synchronize()
p.profile_enable(5)
for _ in range(5):
    fn(k, v)
torch.cuda.synchronize()
names, rows = p.profile_read()
p.profile_enable(0)
acc = {}
for r in rows:
    for nm, t in zip(names, r):
        acc[nm] = acc.get(nm, 0.0) + t / len(rows)
print({k2: round(x, 4) for k2, x in acc.items()}, "total", round(sum(acc.values()), 4))
