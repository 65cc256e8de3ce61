import torch, time
n = 14 * 1024 * 1024 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory(); d = torch.empty(n, device="cuda")
h2 = torch.empty(n, dtype=torch.float32).pin_memory(); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3): d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(f, k=20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(k)]; b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / k
h2d = t(lambda: d.copy_(h, non_blocking=True)); d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
bb = t(both)
mb = n * 4 / 1e6
print(f"H2D {mb/h2d:.1f} GB/s ({h2d*1e3:.0f} us), D2H {mb/d2h:.1f} GB/s ({d2h*1e3:.0f} us), both concurrent {bb*1e3:.0f} us")
