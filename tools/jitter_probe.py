import torch, time, json
a = torch.randn(8192, 8192, device="cuda")
res = []
for i in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); c0 = time.process_time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        b = a @ a
    e1.record(); torch.cuda.synchronize()
    res.append((round(time.perf_counter() - t0, 4), round(e0.elapsed_time(e1) / 1e3, 4)))
print(json.dumps(res))
