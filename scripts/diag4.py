import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1802_02619_b200 as lco, workloads, oracle
def run(name, keys, vals, dims, perm):
    p = lco.plan(dims, perm)
    n = keys.numel()
    ko, vo, po = p.permute(keys, vals)
    torch.cuda.synchronize()
    ek, ev, ep = oracle.permute(dims, perm, keys.cpu().numpy().view(np.uint64), vals.cpu().numpy())
    bad = int((ko.cpu().numpy().view(np.uint64) != ek).sum())
    i = p.info(n)
    print(name, n, i["path"], i["msd_levels"], i["digit_bits"], i["leaf_bits"], "bad", bad, flush=True)
for sc in (48, 64, 96):
    w = workloads.config("C3", device="cuda", scale=sc)
    run(f"C3b s{sc}", w.keys, w.vals, w.dims, w.perms[1])
k, v = workloads.combinatorial_laplacian(1448, device="cuda")
run("lap1448 (3,1,2,0)", k, v, (1448,) * 4, (3, 1, 2, 0))
k, v = workloads.combinatorial_laplacian(2896, device="cuda")
run("lap2896 (3,1,2,0)", k, v, (2896,) * 4, (3, 1, 2, 0))
