"""PCIe bandwidth from pinned host memory (H2D, D2H, both at once) at C4's e2e size."""
import torch
n = 1 << 31   # 8 GiB per direction (keys + values of 2^30 pairs)
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); fn(); torch.cuda.synchronize(); b.record(); b.synchronize(); return a.elapsed_time(b)
for rep in range(2):
    th = t(lambda: d.copy_(h, non_blocking=True))
    td = t(lambda: h.copy_(d, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    tb = t(both)
    print(f"H2D {n/th/1e6:.1f} GB/s ({th:.1f} ms)  D2H {n/td/1e6:.1f} GB/s ({td:.1f} ms)  both {tb:.1f} ms")
