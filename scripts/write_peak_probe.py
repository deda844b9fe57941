"""Pure-write HBM ceiling on this B200: cudaMemset / torch fill of a 3.2 GB
buffer (the K1 tree's per-step output size), CUDA events, best of 10."""
import torch

n = 3_200_000_000 // 4
buf = torch.empty(n, dtype=torch.int32, device="cuda")
for name, fn in (("fill_", lambda i: buf.fill_(i)), ("zero_", lambda i: buf.zero_())):
    fn(0)
    torch.cuda.synchronize()
    best = 1e9
    for i in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(i)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{name}: {best:.3f} ms for 3.2 GB -> {3.2e9 / (best * 1e-3) / 1e9:.0f} GB/s")
src = torch.empty(n // 2, dtype=torch.int32, device="cuda")
dst = torch.empty(n // 2, dtype=torch.int32, device="cuda")
best = 1e9
for i in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dst.copy_(src)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
print(f"copy 1.6 GB: {best:.3f} ms -> {3.2e9 / (best * 1e-3) / 1e9:.0f} GB/s (read+write)")
