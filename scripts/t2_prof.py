"""Per-kernel times (lco_profile) of chosen Table 2 permutations of the Laplacian tensor:
python scripts/t2_prof.py "1,3,2,0" "2,0,3,1" ...   (env overrides apply per plan)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1802_02619_b200 as lco  # noqa: E402
import workloads  # noqa: E402

dev = torch.device("cuda:0")
n = 2896
k, v = workloads.combinatorial_laplacian(n, device=dev)
for arg in sys.argv[1:]:
    sort = arg.startswith("s:")
    perm = tuple(int(x) for x in arg.split(":")[-1].split(","))
    p = lco.Plan((n,) * 4, perm)
    ws = torch.empty(p.workspace_size(k.numel()) + 256, dtype=torch.uint8, device=dev)
    out = (torch.empty_like(k), torch.empty_like(v), torch.empty(k.numel(), dtype=torch.int32, device=dev))
    fn = (lambda: p.sort(k, v, out=out, workspace=ws)) if sort else (lambda: p.permute(k, v, out=out, workspace=ws))
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    p.profile_enable(5)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    names, rows = p.profile_read()
    p.profile_enable(0)
    med = np.median(np.array(rows), axis=0)
    print(arg, p.info(k.numel(), sort=sort)["path"], f"total {med.sum():.3f} ms")
    print("   ", ", ".join(f"{a} {b:.3f}" for a, b in zip(names, med) if b > 0.004))
