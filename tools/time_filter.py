"""Filter pass time on a workload (GPU box): sc_filter_lowpass_f32 with device buffers, median of reps."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1509_08863_b200 as sc
from scinputs import configs
wl = sys.argv[1] if len(sys.argv) > 1 else "c2_sbm100k"
w = configs.WORKLOADS[wl]
g = configs.build_graph(wl, cache=True)
G = sc.Graph.from_csr(g)
lmax = 2.0 * G.info()[3]
Y = torch.empty((g.n, w.R), device="cuda")
X = torch.randn((g.n, w.R), device="cuda")
ts = []
for i in range(7):
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sc.sc_filter_lowpass_f32(G.handle, 0.1 * lmax, lmax, w.order, w.jackson, w.R, 3, X, Y); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(json.dumps({"workload": wl, "ms": sorted(ts)[3]}))
