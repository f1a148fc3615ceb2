import torch, time
d = torch.empty(133_000_000 // 4, device="cuda")
h = torch.empty_like(d, device="cpu").pin_memory()
for _ in range(3): h.copy_(d, non_blocking=True); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10): h.copy_(d, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"D2H 133 MB pinned: {ms:.3f} ms = {133e6/ms/1e6:.1f} GB/s")
hh = torch.empty_like(d, device="cpu")
t=time.perf_counter(); hh.copy_(d); torch.cuda.synchronize(); print("pageable", (time.perf_counter()-t)*1e3, "ms")
