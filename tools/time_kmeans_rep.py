"""k-means call timed repeatedly in one process (GPU box): first call (module loading,
pool growth) vs steady state.  argv: workload restarts max_iter reps"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1509_08863_b200 as sc
from scinputs import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c3_sbm1m"
restarts = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 100
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
w = configs.WORKLOADS[wl]
g = configs.build_graph(wl, cache=True)
G = sc.Graph.from_csr(g)
n, R = g.n, w.R
lmax = 2.0 * G.info()[3]
Y = torch.empty((n, R), dtype=torch.float32, device="cuda")
sc.sc_filter_lowpass_f32(G.handle, 0.005 * lmax, lmax, w.order, w.jackson, R, 3, None, Y)
lab = torch.empty(n, dtype=torch.int32, device="cuda")
out = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = sc.sc_kmeans(Y, n, R, w.k, restarts, iters, 4, None, lab)
    torch.cuda.synchronize()
    out.append(round(time.perf_counter() - t0, 4))
print(json.dumps({"workload": wl, "restarts": restarts, "seconds": out, "iters": res[1], "inertia": res[0]}))
