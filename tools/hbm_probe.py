"""Calibrate achievable HBM read bandwidth with simple torch reductions (context for the
rank-r kernels' roofline).  Prints GB/s for a few sizes."""
import torch

for mib in (64, 128, 512, 2048):
    x = torch.randn(mib * 1024 * 1024 // 2, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(1, device="cuda", dtype=torch.float32)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(12):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        y = x.sum(dtype=torch.float32)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"sum {mib} MiB: {ms*1e3:.1f} us  {mib*2**20/ms/1e6:.0f} GB/s")
    x2 = torch.empty_like(x)
    ts = []
    for i in range(12):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x2.copy_(x)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"copy {mib} MiB: {ms*1e3:.1f} us  {2*mib*2**20/ms/1e6:.0f} GB/s (read+write)")
