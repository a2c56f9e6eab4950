"""Pinned host -> device copy bandwidth (the e2e path's bound): one 4-GB copy and 128-MB chunks."""
import torch
n = 1 << 30
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
for chunk in (n, 1 << 25, 1 << 26, 1 << 27):
    for _ in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for off in range(0, n, chunk):
            d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"chunk {chunk * 4 >> 20} MB: {4 * n / ms / 1e6:.1f} GB/s")
