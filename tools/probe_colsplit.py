"""Gather-locality probe for the column-block idea (DESIGN.md §0(f) item 1), GPU box.

Times the streaming fused step (sc_cheb_step_f32, R = 32 columns, y_mode 0) on random
graphs with N = 10^6 rows and 20 nonzeros per row whose column indices are uniform in
[0, f N): the gathered T_s table is f * 128 MB.  Everything else the launch moves is
unchanged, so the ratio of the times is what a column split of the CSR would buy on the
gather side."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_08863_b200 as sc

N, DEG, R = 1_000_000, 20, 32
rng = np.random.default_rng(7)
out = {}
for f in (1.0, 0.5, 0.25):
    span = int(N * f)
    col = np.sort(rng.integers(0, span, size=(N, DEG), dtype=np.int32), axis=1).reshape(-1)
    rp = np.arange(0, N * DEG + 1, DEG, dtype=np.int64)
    h = sc.sc_graph_load(N, N, N * DEG, rp, col, None)
    T0 = torch.randn(N, R, device="cuda")
    T1 = torch.randn(N, R, device="cuda")
    T2 = torch.empty(N, R, device="cuda")
    st = torch.cuda.current_stream()
    def step():
        sc.sc_cheb_step_f32(h, 0, N, R, T0, R, T1, R, T2, R, None, R, 0.1, -2.0, -1.0, 0, 0, 0, 0)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(50):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / 50
    out[f"table_MB_{int(128 * f)}"] = {"us_per_step": round(us, 1),
                                        "gather_TBps": round(N * DEG * R * 4 / us / 1e6, 2)}
    sc.sc_graph_free(h)
    del T0, T1, T2
print(json.dumps(out))
