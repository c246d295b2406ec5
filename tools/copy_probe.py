"""Host<->device copy bandwidth from pinned memory (GPU box), contiguous and 2-D strided."""
import json, torch
n, R = 1_000_000, 64
h = torch.empty((n, R), dtype=torch.float32, pin_memory=True)
d = torch.empty((n, R), dtype=torch.float32, device="cuda")
out = {}
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = t(lambda: d.copy_(h, non_blocking=True)); out["h2d_GBps"] = round(n * R * 4 / ms / 1e6, 1)
ms = t(lambda: h.copy_(d, non_blocking=True)); out["d2h_GBps"] = round(n * R * 4 / ms / 1e6, 1)
ms = t(lambda: d[:, :32].copy_(h[:, :32], non_blocking=True)); out["h2d_2d_half_GBps"] = round(n * 32 * 4 / ms / 1e6, 1)
ms = t(lambda: h[:, :32].copy_(d[:, :32], non_blocking=True)); out["d2h_2d_half_GBps"] = round(n * 32 * 4 / ms / 1e6, 1)
print(json.dumps(out))
