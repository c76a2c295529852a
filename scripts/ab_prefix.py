"""A/B of permute_op (api.cu): identity-prefix plans with >= 4 LSD passes on the shaved key
vs the MSD schedule of the full new key.  Run twice: default and LCO_NO_PREFIX_MSD=1.
usage: python scripts/ab_prefix.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_1802_02619_b200 import lco  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


dev = "cuda:0"
cases = []
k, v = workloads.random_tensor((4096,) * 5, 200_000_000, seed=5, values="normal", device=dev)
cases += [("random 4096^5 200M", (4096,) * 5, p, k, v) for p in ((0, 4, 3, 2, 1), (0, 1, 4, 3, 2))]
k2, v2 = workloads.combinatorial_laplacian(2896, dev)
cases += [("laplacian 2896", (2896,) * 4, p, k2, v2) for p in ((0, 3, 2, 1), (0, 2, 3, 1))]
k3, v3 = workloads.random_tensor((64,) * 7, 3_000_000, seed=9, values="normal", device=dev)
cases += [("random 64^7 3M", (64,) * 7, (0, 6, 5, 4, 3, 2, 1), k3, v3)]
k4 = k3[:300_000].contiguous()
cases += [("random 64^7 300K (low keys)", (64,) * 7, (0, 6, 5, 4, 3, 2, 1), k4, v3[:300_000].contiguous())]
k5 = k[:6_000_000].contiguous()  # the lowest 3 % of the keys: 8 of 256 first digits used
cases += [("random 4096^5, lowest 6M of 200M keys", (4096,) * 5, (0, 4, 3, 2, 1), k5, v[:6_000_000].contiguous())]
k6 = k[:40_000_000].contiguous()
cases += [("random 4096^5, lowest 40M of 200M keys", (4096,) * 5, (0, 4, 3, 2, 1), k6, v[:40_000_000].contiguous())]
out = []
for name, dims, perm, kk, vv in cases:
    p = lco.Plan(dims, perm)
    n = kk.numel()
    ws = torch.empty(p.workspace_size(n), dtype=torch.uint8, device=dev)
    o = (torch.empty_like(kk), torch.empty_like(vv), torch.empty(n, dtype=torch.int32, device=dev))
    ms = timed(lambda: p.permute(kk, vv, out=o, workspace=ws))
    i = p.info(n)
    out.append({"case": name, "perm": perm, "nnz": n, "path": i["path"], "sort_bits": i["sort_bits"],
                "ms": round(ms, 4)})
    print(json.dumps(out[-1]), flush=True)
