"""k-means only (GPU box): features = filtered block of a workload, one sc_kmeans call."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1509_08863_b200 as sc
from scinputs import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c3_sbm1m"
restarts = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
w = configs.WORKLOADS[wl]
g = configs.build_graph(wl, cache=True)
G = sc.Graph.from_csr(g)
n, R = g.n, w.R
lmax = 2.0 * G.info()[3]
Y = torch.empty((n, R), dtype=torch.float32, device="cuda")
sc.sc_filter_lowpass_f32(G.handle, 0.005 * lmax, lmax, w.order, w.jackson, R, 3, None, Y)
lab = torch.empty(n, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
res = sc.sc_kmeans(Y, n, R, w.k, restarts, iters, 4, None, lab)
torch.cuda.synchronize()
print(json.dumps({"workload": wl, "restarts": restarts, "max_iter": iters, "seconds": time.perf_counter() - t0,
                  "inertia": res[0], "iters": res[1]}))
