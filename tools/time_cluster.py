"""sc_cluster phases on one workload (GPU box; tooling): SC_CLUSTER_TRACE per-phase times."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SC_CLUSTER_TRACE", "1")
import torch
import paper_1509_08863_b200 as sc
from scinputs import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c3_sbm1m"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = configs.WORKLOADS[wl]
g = configs.build_graph(wl, cache=True)
G = sc.Graph.from_csr(g)
lab = torch.empty(g.n, dtype=torch.int32, device="cuda")
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    info = sc.sc_cluster(G.handle, w.k, w.R, w.order, w.jackson, 32, 1, w.kmeans_restarts, 100, False, lab)
    torch.cuda.synchronize()
    print(json.dumps({"workload": wl, "seconds": time.perf_counter() - t0, "info": list(info)}), flush=True)
