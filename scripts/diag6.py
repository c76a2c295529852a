import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1802_02619_b200 as lco, workloads, oracle
w = workloads.config("C3", device="cuda", scale=96)
dims, perm = w.dims, w.perms[1]
p = lco.plan(dims, perm)
ko = torch.full_like(w.keys, -7)
vo = torch.empty_like(w.vals)
po = torch.full((w.keys.numel(),), -7, dtype=torch.int32, device="cuda")
p.permute(w.keys, w.vals, out=(ko, vo, po))
torch.cuda.synchronize()
ek, ev, ep = oracle.permute(dims, perm, w.keys.cpu().numpy().view(np.uint64), w.vals.cpu().numpy())
k = ko.cpu().numpy()
print("unwritten", int((k == -7).sum()), "of", len(k))
seg = slice(0, 10420)
kk = k[seg].view(np.uint64); ee = ek[seg]
print("seg0 bad", int((kk != ee).sum()), "unwritten", int((k[seg] == -7).sum()))
print("got", kk[:12]); print("exp", ee[:12])
print("sorted(got)==sorted(exp) in seg0:", np.array_equal(np.sort(kk), np.sort(ee)))
T = 96 * 96
print("q got", (kk[:12] // T), "q exp", (ee[:12] // T))
