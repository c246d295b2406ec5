"""k-means alone on sc_cluster's own features (GPU box; tooling): lambda_k estimated as in
sc_cluster (probes seed ^ 0x5e5e5e5e, Jackson, 32 probes), features filtered with the
workload's order and seed, then one sc_kmeans call (argv: workload, restarts, max_iter)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1509_08863_b200 as sc
from scinputs import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c3_sbm1m"
restarts = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 100
w = configs.WORKLOADS[wl]
g = configs.build_graph(wl, cache=True)
G = sc.Graph.from_csr(g)
seed = 1
lmax = sc.sc_lambda_max(G.handle, 60, 0.01, seed ^ 0x1a2b3c4d)
lk, _ = sc.sc_estimate_lambda_k(G.handle, w.k, lmax, w.order, True, 32, seed ^ 0x5e5e5e5e, 40, 1e-4)
Y = torch.empty((g.n, w.R), dtype=torch.float32, device="cuda")
sc.sc_filter_lowpass_f32(G.handle, lk, lmax, w.order, w.jackson, w.R, seed, None, Y)
lab = torch.empty(g.n, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
res = sc.sc_kmeans(Y, g.n, w.R, w.k, restarts, iters, seed, None, lab)
torch.cuda.synchronize()
print(json.dumps({"workload": wl, "restarts": restarts, "max_iter": iters, "seconds": time.perf_counter() - t0,
                  "inertia": res[0], "iters": res[1]}))
