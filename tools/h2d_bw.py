import torch, time
n = 38928384 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
o = torch.empty(13 * 1024 * 1024 // 2, dtype=torch.bfloat16, device="cuda")
ho = torch.empty_like(o, device="cpu").pin_memory()
for _ in range(5): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): d.copy_(h, non_blocking=True)
b.record(); torch.cuda.synchronize()
print("H2D 39MB GB/s", 50 * n * 2 / (a.elapsed_time(b) / 1e3) / 1e9)
# chunked into 3 copies like q,k,v
hs = [h[i * n // 3:(i + 1) * n // 3] for i in range(3)]
ds = [d[i * n // 3:(i + 1) * n // 3] for i in range(3)]
a.record()
for _ in range(50):
    for x, y in zip(ds, hs): x.copy_(y, non_blocking=True)
b.record(); torch.cuda.synchronize()
print("H2D 3x13MB GB/s", 50 * n * 2 / (a.elapsed_time(b) / 1e3) / 1e9)
s2 = torch.cuda.Stream()
a.record()
for _ in range(50):
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(o, non_blocking=True)
b.record(); torch.cuda.synchronize()
print("H2D+D2H concurrent, H2D GB/s", 50 * n * 2 / (a.elapsed_time(b) / 1e3) / 1e9)
