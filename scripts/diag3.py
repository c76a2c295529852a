import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1802_02619_b200 as lco, workloads, oracle
scale = int(sys.argv[1]) if len(sys.argv) > 1 else None
w = workloads.config("C3", device="cuda", scale=scale)
perm = w.perms[1]
p = lco.plan(w.dims, perm)
n = w.keys.numel()
print("n", n, p.info(n))
ko, vo, po = p.permute(w.keys, w.vals)
torch.cuda.synchronize()
ek, ev, ep = oracle.permute(w.dims, perm, w.keys.cpu().numpy().view(np.uint64), w.vals.cpu().numpy())
k = ko.cpu().numpy().view(np.uint64)
bad = np.nonzero(k != ek)[0]
print("bad", len(bad))
if len(bad):
    print("first", bad[:10], "last", bad[-5:])
    T = 128 * 128
    q_e = ek[bad] // T
    print("q of bad (expected)", np.unique(q_e >> 4)[:20], "count uniq", len(np.unique(q_e)))
    # runs of bad positions
    runs = np.split(bad, np.nonzero(np.diff(bad) != 1)[0] + 1)
    print("runs", len(runs), [ (r[0], len(r)) for r in runs[:10]])
    # is output a permutation of expected within the run?
    r = runs[0]
    print("sorted equal within first run:", np.array_equal(np.sort(k[r]), np.sort(ek[r])))
    print("got", k[r[0]:r[0]+8], "exp", ek[r[0]:r[0]+8])
