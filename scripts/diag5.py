import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1802_02619_b200 as lco, workloads, oracle
w = workloads.config("C3", device="cuda", scale=96)
dims, perm = w.dims, w.perms[1]
p = lco.plan(dims, perm)
ko, vo, po = p.permute(w.keys, w.vals)
torch.cuda.synchronize()
ek, ev, ep = oracle.permute(dims, perm, w.keys.cpu().numpy().view(np.uint64), w.vals.cpu().numpy())
print(os.environ.get("LCO_L3_FLAT"), "bad", int((ko.cpu().numpy().view(np.uint64) != ek).sum()))
