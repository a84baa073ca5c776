"""Microbenchmark of one tcgen05 GEMM launch (runlora_debug_gemm) vs cuBLAS (torch.matmul).

    python tools/gemm_bench.py --M 8192 --N 4096 --K 4096 --cg 2 --bn 256 [--b-mn] [--reps 50]
Prints one JSON line per configuration.  Used for roofline work on the main GEMM.
"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03415_b200 import runlora as rl  # noqa: E402


def sustain(fn, seconds):
    import subprocess
    import time
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                          "--format=csv,noheader,nounits", "-lms", "100", "-i", "0"], stdout=subprocess.PIPE, text=True)
    torch.cuda.synchronize()
    t0 = time.time()
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    p.terminate()
    out = p.communicate()[0].strip().splitlines()
    clk = sorted(float(l.split(",")[0]) for l in out if l.strip())
    pw = sorted(float(l.split(",")[1]) for l in out if l.strip())
    cap = sum(1 for l in out if "Active" in l and "Not" not in l)
    return {"sustain_us": e0.elapsed_time(e1) * 1e3 / n, "sm_mhz_median": clk[len(clk) // 2] if clk else None,
            "power_w_median": pw[len(pw) // 2] if pw else None, "power_cap_samples": cap, "samples": len(out)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=8192)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--K2", type=int, default=0)
    ap.add_argument("--cg", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--bn", type=int, default=256)
    ap.add_argument("--a-mn", action="store_true")
    ap.add_argument("--b-mn", action="store_true")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--splits", type=int, default=1)
    ap.add_argument("--cublas", action="store_true")
    ap.add_argument("--check", action="store_true", help="compare D with an fp32 torch product (K2 = 0, K-major)")
    ap.add_argument("--sustain", type=float, default=0.0, help="also run back-to-back for this many seconds, "
                    "sampling SM clock and power")
    a = ap.parse_args()
    f = rl._lib.runlora_debug_gemm
    P, I = C.c_void_p, C.c_int
    f.restype = I
    f.argtypes = [P, I, I, I, P, I, P, I, I, P, P, I, P, P, I, I, I, P]
    h = rl.handle(0)
    bf = torch.bfloat16
    M, N, K = a.M, a.N, a.K
    A = torch.randn(K, M, device="cuda", dtype=bf) if a.a_mn else torch.randn(M, K, device="cuda", dtype=bf)
    B = torch.randn(K, N, device="cuda", dtype=bf) if a.b_mn else torch.randn(N, K, device="cuda", dtype=bf)
    A2 = torch.randn(M, max(a.K2, 8), device="cuda", dtype=bf)
    B2 = torch.randn(max(a.K2, 8), N, device="cuda", dtype=bf) if a.b_mn else \
        torch.randn(N, max(a.K2, 8), device="cuda", dtype=bf)
    D = torch.empty(M, N, device="cuda", dtype=bf) if a.splits == 1 else \
        torch.empty(a.splits, M, N, device="cuda", dtype=torch.float32)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    flops = 2.0 * M * N * (K + a.K2)
    for cg in a.cg:
        def run():
            st = f(h._h, M, N, K, A.data_ptr(), int(a.a_mn), B.data_ptr(), int(a.b_mn), a.K2, A2.data_ptr(),
                   B2.data_ptr(), 0 if a.splits == 1 else 2, D.data_ptr(), None, a.bn, a.splits, cg, s)
            assert st == 0, rl._lib.runlora_last_error()
        for _ in range(5):
            run()
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        med = ts[len(ts) // 2]
        if a.check:
            ref = A.float() @ B.float().t()
            err = ((D.float() - ref).norm() / ref.norm()).item()
            print(json.dumps({"check": "tc_gemm", "cg": cg, "bn": a.bn, "rel_fro": err}), flush=True)
            assert err < 1e-2, err
        rec = {"kernel": "tc_gemm", "cg": cg, "bn": a.bn, "M": M, "N": N, "K": K, "K2": a.K2, "splits": a.splits,
               "GBps_A": (M * K * 2) / (med * 1e-3) / 1e9,
               "a_mn": a.a_mn, "b_mn": a.b_mn, "median_us": med * 1e3, "min_us": ts[0] * 1e3,
               "tflops_median": flops / (med * 1e-3) / 1e12}
        if a.sustain:
            rec.update(sustain(run, a.sustain))
        print(json.dumps(rec), flush=True)
    if a.cublas:
        At = A.t() if a.a_mn else A
        Bt = B if a.b_mn else B.t()
        for _ in range(5):
            torch.matmul(At, Bt, out=D)
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(At, Bt, out=D)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        med = ts[len(ts) // 2]
        rec = {"kernel": "cublas", "M": M, "N": N, "K": K, "median_us": med * 1e3, "min_us": ts[0] * 1e3,
               "tflops_median": 2.0 * M * N * K / (med * 1e-3) / 1e12}
        if a.sustain:
            rec.update(sustain(lambda: torch.matmul(At, Bt, out=D), a.sustain))
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
