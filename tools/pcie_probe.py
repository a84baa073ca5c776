"""PCIe copy rates on this box: H2D, D2H alone and concurrently (pinned host memory), the
bound of bench.py's e2e leg (256 MiB of copies per C2 step)."""
import json
import torch

N = 128 << 20
dev = torch.device("cuda", 0)
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N, dtype=torch.uint8, device=dev)
d_out = torch.empty(N, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
t_both = timed(both)
print(json.dumps({"bytes": N, "h2d_GBps": N / t_h2d / 1e6, "d2h_GBps": N / t_d2h / 1e6,
                  "concurrent_ms": t_both, "concurrent_GBps_each": N / t_both / 1e6,
                  "h2d_ms": t_h2d, "d2h_ms": t_d2h}))
