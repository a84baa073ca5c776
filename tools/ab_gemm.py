"""Same-process A/B of one tcgen05 GEMM launch (runlora_debug_gemm) in two builds, on the
SAME device buffers: isolates kernel-code effects from workspace-placement effects.

    python tools/ab_gemm.py OLD.so NEW.so --M 8192 --N 4096 --K 4096 [--K2 64] [--b-mn] [--bn 256]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ab_lib import load  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs=2)
    ap.add_argument("--M", type=int, default=8192)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--K2", type=int, default=0)
    ap.add_argument("--bn", type=int, default=256)
    ap.add_argument("--b-mn", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--blocks", type=int, default=15)
    a = ap.parse_args()
    M, N, K, K2 = a.M, a.N, a.K, a.K2
    g = torch.Generator(device="cuda").manual_seed(1)
    A1 = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B1 = (torch.randn(K, N, device="cuda", generator=g) if a.b_mn else torch.randn(N, K, device="cuda", generator=g)).to(torch.bfloat16)
    A2 = torch.randn(M, max(K2, 8), device="cuda", generator=g).to(torch.bfloat16)
    B2 = (torch.randn(max(K2, 8), N, device="cuda", generator=g) if a.b_mn else torch.randn(N, max(K2, 8), device="cuda", generator=g)).to(torch.bfloat16)
    D = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    fns = []
    for i, path in enumerate(a.libs):
        rl = load(path, f"rl_g{i}")
        h = rl.Handle(0)
        f = rl._lib.runlora_debug_gemm
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int,
                      C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]

        def run(f=f, h=h, d=D[i]):
            st = f(h._h, M, N, K, A1.data_ptr(), 0, B1.data_ptr(), int(a.b_mn), K2, A2.data_ptr(), B2.data_ptr(), 0,
                   d.data_ptr(), None, a.bn, 1, 2, torch.cuda.current_stream().cuda_stream)
            assert st == 0, st
        fns.append((run, h))
    for run, _ in fns:
        for _ in range(5):
            run()
    torch.cuda.synchronize()
    t = [[], []]
    for _ in range(a.blocks):
        for i, (run, _) in enumerate(fns):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            t[i].append(e0.elapsed_time(e1) * 1e3 / a.reps)
    print(json.dumps({"shape": [M, N, K, K2], "b_mn": a.b_mn, "bn": a.bn, "a_us": float(np.median(t[0])),
                      "b_us": float(np.median(t[1])), "b_over_a": float(np.median(np.array(t[1]) / np.array(t[0]))),
                      "same": bool(torch.equal(D[0], D[1]))}))


if __name__ == "__main__":
    main()
