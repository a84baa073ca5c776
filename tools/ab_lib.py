"""Same-process A/B of two builds of librunlora.so: alternating blocks of forward+backward
steps of one plan, CUDA-event timed, medians (the clocks and power state drift across a run;
interleaving hits both builds alike).

    python tools/ab_lib.py OLD.so NEW.so [--plan 2,1] [--r 16] [--steps 50] [--blocks 20]
Both libraries are loaded with RTLD_LOCAL (ctypes default), each behind its own copy of the
binding module.
"""
import argparse
import importlib.util
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def load(path, name):
    os.environ["RUNLORA_LIB"] = os.path.abspath(path)
    spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, "paper_2312_03415_b200", "runlora.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs=2)
    ap.add_argument("--plan", default="2,1")
    ap.add_argument("--r", type=int, default=16)
    ap.add_argument("--shape", default=None, help="n,k,m")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--blocks", type=int, default=20)
    ap.add_argument("--warm", type=int, default=100)
    a = ap.parse_args()
    c = synth.C2[a.r]
    if a.shape:
        n, k, m = (int(x) for x in a.shape.split(","))
        c = synth.case(f"ab_{n}_{k}_{m}_{a.r}", 0, 78, n, k, m, a.r, "bf16")
    d = {kk: v.cuda() for kk, v in synth.operands(c).items()}
    f, b = (int(x) for x in a.plan.split(","))
    arms, mods = [], []
    for i, path in enumerate(a.libs):
        rl = load(path, f"rl_ab{i}")
        h = rl.Handle(0)
        mods.append((rl, h))
        shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
        out = {"Y": torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda"),
               "dX": torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda"),
               "dA": torch.empty(c.k, c.r, device="cuda"), "dB": torch.empty(c.r, c.m, device="cuda")}
        ws = torch.empty(rl.workspace_size(shape), dtype=torch.uint8, device="cuda")

        def step(h=h, shape=shape, out=out, ws=ws):
            h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], out["Y"], ws)
            h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], out["dX"], out["dA"], out["dB"], ws=ws)
        arms.append((path, step, out))
    for _, step, _ in arms:
        for _ in range(a.warm):
            step()
    torch.cuda.synchronize()
    import time
    t = [[], []]
    host = [[], []]
    for _ in range(a.blocks):
        for i, (_, step, _) in enumerate(arms):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            h0 = time.perf_counter()
            for _ in range(a.steps):
                step()
            host[i].append((time.perf_counter() - h0) * 1e6 / a.steps)  # enqueue time per step
            e1.record()
            torch.cuda.synchronize()
            t[i].append(e0.elapsed_time(e1) * 1e3 / a.steps)
    same = all(torch.equal(arms[0][2][k], arms[1][2][k]) for k in ("Y", "dX", "dA", "dB"))
    work = []
    if os.environ.get("RUNLORA_LTRACE"):  # per-kernel in-step work (first ready -> last exit)
        import ctypes as C
        for i, (_, step, _) in enumerate(arms):
            mod, h = mods[i]
            lib = mod._lib
            lib.runlora_debug_ltrace.restype = C.c_int
            lib.runlora_debug_kernel_name.restype = C.c_char_p
            buf = np.zeros(8 * 4096, dtype=np.uint64)
            kids = np.zeros(4096, dtype=np.int32)
            args = (h._h, buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), kids.ctypes.data_as(C.POINTER(C.c_int)), 4096)
            lib.runlora_debug_ltrace(*args)
            for _ in range(a.steps):
                step()
            nrec = lib.runlora_debug_ltrace(*args)
            rec = buf[: 8 * nrec].reshape(nrec, 8).astype(np.int64)
            per_step = nrec // a.steps
            rows = []
            for pos in range(per_step):  # launch position within the step: name, work, gap
                idx = [s_ * per_step + pos for s_ in range(a.steps)]
                nm = lib.runlora_debug_kernel_name(int(kids[idx[0]])).decode()
                wk = np.median([(rec[j, 4] - rec[j, 1]) / 1e3 for j in idx])
                gp = np.median([(rec[j, 1] - rec[j - 1, 4]) / 1e3 for j in idx if j > 0])
                rows.append(f"{nm}:{wk:.1f}+{gp:.1f}")
            work.append(rows)
    print(json.dumps({"workload": c.name, "plan": f"F{f}+B{b}", "a": a.libs[0], "b": a.libs[1],
                      "a_us": float(np.median(t[0])), "b_us": float(np.median(t[1])),
                      "b_over_a": float(np.median(np.array(t[1]) / np.array(t[0]))), "outputs_bit_identical": same,
                      "host_enqueue_us": [float(np.median(host[0])), float(np.median(host[1]))], "work_us": work}))


if __name__ == "__main__":
    main()
