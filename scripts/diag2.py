import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1802_02619_b200 as lco, workloads, oracle
w = workloads.config("C3", device="cuda")
perm = w.perms[1]
p = lco.plan(w.dims, perm)
n = w.keys.numel()
ws = torch.empty(p.workspace_size(n) + 256, dtype=torch.uint8, device="cuda")
out = (torch.empty_like(w.keys), torch.empty_like(w.vals), torch.empty(n, dtype=torch.int32, device="cuda"))
ek, ev, ep = oracle.permute(w.dims, perm, w.keys.cpu().numpy().view(np.uint64), w.vals.cpu().numpy())
mode = sys.argv[1] if len(sys.argv) > 1 else "direct"
g = p.graph(w.keys, w.vals, out=out, workspace=ws) if mode == "graph" else None
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if g is not None and it % 2: g.replay()
    else: p.permute(w.keys, w.vals, out=out, workspace=ws)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    ok = np.array_equal(out[0].cpu().numpy().view(np.uint64), ek) and np.array_equal(out[2].cpu().numpy().view(np.uint32), ep)
    print(mode, it, "graph" if (g is not None and it % 2) else "direct", round(dt * 1e3, 3), "ms ok", ok, flush=True)
