"""Phase timing of sc_cluster's steps on a workload (GPU box): lambda_max, lambda_k,
filter, k-means -- each through its own C-ABI call, CUDA-event timed."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_08863_b200 as sc
from scinputs import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c3_sbm1m"
w = configs.WORKLOADS[wl]
g = configs.build_graph(wl, cache=True)
G = sc.Graph.from_csr(g)
n, R, p = g.n, w.R, w.order
out = {"workload": wl}
def timed(name, fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    out[name + "_s"] = round(time.perf_counter() - t0, 4); return r
lmax = timed("lambda_max", lambda: sc.sc_lambda_max(G.handle, 60, 0.01, 1))
lk, ck = timed("lambda_k", lambda: sc.sc_estimate_lambda_k(G.handle, w.k, lmax, p, True, 32, 2, 40, 1e-4))
Y = torch.empty((n, R), dtype=torch.float32, device="cuda")
timed("filter", lambda: sc.sc_filter_lowpass_f32(G.handle, lk, lmax, p, w.jackson, R, 3, None, Y))
lab = torch.empty(n, dtype=torch.int32, device="cuda")
res = timed("kmeans", lambda: sc.sc_kmeans(Y, n, R, w.k, w.kmeans_restarts, 100, 4, None, lab))
out.update(inertia=res[0], iters=res[1], best=res[2], count_k=ck)
if g.labels is not None:
    out["ari"] = sc.sc_ari(lab, torch.from_numpy(g.labels).cuda(), n)
print(json.dumps(out))
