#!/usr/bin/env python
"""Benchmark of the RunLoRA hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--r 16] [--impl reference]

A step is one pass of the whole hot path over one batch: the plan
chosen by the selector (cached, chosen before warm-up), forward, backward (adapter
grads then dX) and — for N > 1 — the token-sharded DP exchange (allreduce of the
packed fp32 [dA | dB], overlapped with dX).  Workload at N=1: BASELINE.json
configs[1] (Llama-7B attention projection, n = 8192 tokens, k = m = 4096), rank
r = 16; under torchrun every rank runs that workload on its own 8192 tokens
(weak scaling) and value = all ranks' tokens / max-over-ranks step time.

`--impl reference` times the CPU fp64 oracle (the only reference this tier has;
oracle/) on the host cores on a bounded token sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "LoRA-linear fwd+bwd tokens/s, tensor-pipe util, speedup vs default XW+(XA)B"
UNIT = "tokens/s"
CAPTION = "synthetic: seeded i.i.d. Gaussian operands with BASELINE.json's laws (no dataset/weights)"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def _case(r):
    return synth.C2[r]


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"rl_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.index)], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        busy = [s for s in sm if smax is None or s > 0.5 * smax] or sm
        return {"sm_mhz": float(np.median(busy)) if busy else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- reference arm
def run_reference(args):
    """CPU fp64 oracle, as it stands, on a bounded token sample of the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    c = _case(args.r)
    f, b = O.select_by_flops(c.n, c.k, c.m, c.r)
    ns = args.ref_tokens
    ops = synth.operands(synth.case(c.name, c.cfg, c.sub, ns, c.k, c.m, c.r, c.dtype))
    X, W, A, B, dY = (ops[k].double().numpy() for k in ("X", "W", "A", "B", "dY"))

    def step():
        O.forward(f, X, W, A, B)
        O.backward(b, X, W, A, B, dY)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    cores = len(os.sched_getaffinity(0))
    val = ns / dt
    sample = (f"{ns}-token contiguous slice of {c.name} (n={c.n}, k={c.k}, m={c.m}, r={c.r}); "
              f"oracle forward{f}+backward{b} in fp64 numpy")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": CAPTION,
            "config": {"workload": c.name, "n": c.n, "k": c.k, "m": c.m, "r": c.r, "sample_tokens": ns,
                       "plan": f"F{f}+B{b}", "criterion": "flops"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _launch_work(h, rl, step, steps):
    """Median in-step work time (µs) per library kernel name over `steps` steps, from the
    library's launch records (RUNLORA_LTRACE): last CTA exit - first CTA ready."""
    import ctypes as C
    lib = rl._lib
    if not hasattr(lib, "runlora_debug_ltrace"):
        return {}
    lib.runlora_debug_ltrace.restype = C.c_int
    lib.runlora_debug_kernel_name.restype = C.c_char_p
    buf = np.zeros(8 * 4096, dtype=np.uint64)
    kids = np.zeros(4096, dtype=np.int32)
    args = (h._h, buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), kids.ctypes.data_as(C.POINTER(C.c_int)), 4096)
    lib.runlora_debug_ltrace(*args)  # reset
    for _ in range(steps):
        step()
    n = lib.runlora_debug_ltrace(*args)
    rec = buf[: 8 * n].reshape(n, 8).astype(np.int64)
    out = {}
    for i in range(n):
        if rec[i, 4] > 0 and rec[i, 1] > 0:
            out.setdefault(lib.runlora_debug_kernel_name(int(kids[i])).decode(), []).append((rec[i, 4] - rec[i, 1]) / 1e3)
    return {k: float(np.median(v)) for k, v in out.items()}


def cpu_baseline(c, fwd, bwd, target_s=12.0, slice_tokens=1024):
    """The oracle timed on the host cores on a bounded sample (rank 0, N=1 only): the
    selected pair on consecutive 1024-token slices of the workload (cycling), until
    ~target_s seconds of CPU work have been timed."""
    import oracle as O
    ns = min(slice_tokens, c.n)
    nslices = max(1, min(c.n, 4 * ns) // ns)
    ops = synth.operands(synth.case(c.name, c.cfg, c.sub, nslices * ns, c.k, c.m, c.r, c.dtype))
    W, A, B = (ops[k].double().numpy() for k in ("W", "A", "B"))
    Xa, dYa = ops["X"].double().numpy(), ops["dY"].double().numpy()
    t_total, tok_total, i = 0.0, 0, 0
    while t_total < target_s:
        s0 = (i % nslices) * ns
        X, dY = Xa[s0:s0 + ns], dYa[s0:s0 + ns]
        t0 = time.perf_counter()
        O.forward(fwd, X, W, A, B)
        O.backward(bwd, X, W, A, B, dY)
        t_total += time.perf_counter() - t0
        tok_total += ns
        i += 1
    return {"value": tok_total / t_total, "unit": UNIT, "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
            "sample": f"{i} contiguous {ns}-token slices of {c.name} ({tok_total} tokens, {t_total:.1f} s of CPU "
                      f"work); oracle forward{fwd}+backward{bwd}, fp64 numpy/BLAS on all host cores, each slice "
                      "including the n-independent W+AB term"}


# ------------------------------------------------------------------ main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--r", type=int, default=16, choices=sorted(synth.C2))
    ap.add_argument("--impl", default="runlora", choices=["runlora", "reference"])
    ap.add_argument("--criterion", default="time", choices=["flops", "time", "hybrid"])
    ap.add_argument("--ref-tokens", type=int, default=512)
    ap.add_argument("--plan", default=None, help="force a variant pair, e.g. 1,1 (skips selection)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-default-chain", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the multi-rank code path on one GPU (not a performance mode)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch.distributed as dist
    # per-launch records (first/last CTA ready and exit): the in-step work time of each
    # kernel, reported beside the CUDA-event durations (read over a window of steps below)
    os.environ.setdefault("RUNLORA_LTRACE", "1")
    from paper_2312_03415_b200 import runlora as rl
    from paper_2312_03415_b200 import dp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        # 6 main-GEMM stages leave shared memory for NCCL's kernels, which then co-reside
        # with the dX GEMM that the adapter-gradient allreduce overlaps
        os.environ.setdefault("RUNLORA_MAIN_STAGES", "6")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    c = _case(args.r)
    n, k, m, r = c.n, c.k, c.m, c.r
    ops = synth.operands(c)
    d = {kk: v.to(dev) for kk, v in ops.items()}
    shape = rl.make_shape(n, k, m, r, rl.BF16)
    h = rl.handle(local)
    ws = h.workspace(shape)
    Y = torch.empty(n, m, dtype=torch.bfloat16, device=dev)
    dX = torch.empty(n, k, dtype=torch.bfloat16, device=dev)
    # DP exchange: NCCL allreduce (default) or the one-shot symmetric-memory kernel (opt-in)
    sym = None
    if world > 1 and args.backend == "nccl" and os.environ.get("RUNLORA_DP_TRANSPORT") == "symm":
        sym = dp.SymmetricAllreduce(k, r, m, dev, h)
    g = sym.grads if sym is not None else dp.PackedAdapterGrads.create(k, r, m, dev)
    crit = {"flops": rl.BY_FLOPS, "time": rl.BY_TIME, "hybrid": rl.HYBRID}[args.criterion]
    if args.plan:
        crit = rl.BY_FLOPS
        args.criterion = "forced"
    plan = h.select(shape, crit, ops={"X": d["X"], "W": d["W"], "A": d["A"], "B": d["B"], "dY": d["dY"], "Y": Y,
                                      "dX": dX, "dA": g.dA, "dB": g.dB}, grad_dtype=rl.F32)
    fwd, bwd = plan.fwd, plan.bwd
    if args.plan:
        fwd, bwd = (int(x) for x in args.plan.split(","))
    if world > 1:
        fwd, bwd = dp.broadcast_plan(fwd, bwd, device=dev)
    comm = torch.cuda.Stream(dev) if world > 1 else None

    def step():
        h.forward(fwd, shape, d["X"], d["W"], d["A"], d["B"], Y, ws)
        if world > 1:
            work = dp.overlapped_backward(
                lambda: h.backward_params(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], g.dA, g.dB, ws=ws),
                lambda: h.backward_input(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, ws=ws),
                g, comm_stream=comm, exchange=sym)
            work.wait()
        else:
            h.backward(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, g.dA, g.dB, ws=ws)

    def timed(fn, K):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / K
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # ---------------- device-resident timing (value)
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    l0 = h.launch_count()
    ms = timed(step, args.steps)
    launches = (h.launch_count() - l0) // args.steps
    clk = clocks.stop()
    value = world * n / (ms * 1e-3)
    flops_step = plan.flops_fwd[fwd] + plan.flops_bwd[bwd]

    # ---------------- per-kernel profile (same steps, library CUDA events on the launch stream)
    h.profile_enable(True)
    h.profile_read(reset=True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize(dev)
    prof = h.profile_read(reset=True)
    h.profile_enable(False)
    peaks, peak_src = _peaks()
    main_ms = prof.get("gemm_main", (0, 0.0))
    main_launches = main_ms[0]
    # algorithmic FLOPs of the main GEMM launches of one step: forward
    # Y GEMM (+ concat tail for F1) and dX GEMM (+ concat tail for B1..B3).
    f_main = 2 * n * m * (k + (r if fwd == 1 else 0)) + 2 * n * k * (m + (r if bwd <= 3 else 0))
    per_launch_s = (main_ms[1] / max(main_launches, 1)) * 1e-3
    main_per_step = main_launches / args.steps
    flops_per_launch = f_main / main_per_step if main_launches else None
    achieved = flops_per_launch / per_launch_s / 1e12 if main_launches else None
    step_prof_ms = sum(v[1] for v in prof.values()) / args.steps
    kernels = {nm: {"launches_per_step": v[0] / args.steps, "ms_per_step": v[1] / args.steps,
                    "share": (v[1] / args.steps) / step_prof_ms if step_prof_ms else None}
               for nm, v in prof.items()}
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            traffic = json.load(f).get("gemm_main", {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    # the main GEMMs are timed inside a long back-to-back loop (power-capped clocks), so the
    # denominator is the SUSTAINED cuBLAS bf16 figure; the burst fraction is reported beside it
    p_sus = peaks.get("bf16_tflops_sustained") or peaks["bf16_tflops"]
    roof = {"bound": "tensor", "achieved": achieved, "peak": p_sus, "unit": "TFLOP/s",
            "frac": achieved / p_sus if achieved else None, "traffic": traffic,
            "kernel": "gemm_main (tcgen05 Y / dX GEMM, 256x512 + 256x256 pair tiles)",
            "peak_source": f"of {peak_src}: bf16 sustained (cuBLAS, seconds-long loop under the power cap)",
            "peak_burst": peaks["bf16_tflops"], "frac_of_burst": achieved / peaks["bf16_tflops"] if achieved else None,
            "flops_per_launch": flops_per_launch}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            nl = json.load(f).get("gemm_main", {}).get("launches", [])
        if nl:
            roof["tensor_pipe_pct_ncu"] = sum(x.get("tensor_pipe_pct", 0) for x in nl) / len(nl)
    except Exception:
        pass
    # HBM-bound rank-r kernels: algorithmic bytes per launch / live duration vs measured HBM
    # copy bandwidth (SURVEY §8(d) "Algorithmic HBM bytes for the rank-r kernels").
    hbm = peaks["hbm_gbs"]
    alg = {
        "gemm_proj": (2 * n * (k if fwd == 1 else 0) + 2 * n * r + 2 * k * r,  # forward1: Z2 = X·A
                      2 * n * (k + m) + 4 * n * r + 2 * r * (k + m)),          # backward: Z1, Z2
        "gemm_tokred": (2 * n * (k + m) + 4 * n * r,),                          # dA, dBᵀ partials
        "gemm_wprime": (4 * k * m + 2 * r * (k + m),) * 2,
    }
    hbm_roof = {}
    for nm, (cnt, ms_tot) in prof.items():
        if nm not in alg or not cnt:
            continue
        per_step = cnt / args.steps
        bytes_step = sum(alg[nm][: int(round(per_step))]) if nm == "gemm_proj" and fwd == 1 else \
            alg[nm][-1] * per_step
        gbs = bytes_step / (ms_tot / args.steps * 1e-3) / 1e9
        hbm_roof[nm] = {"bound": "hbm", "bytes_per_step": bytes_step, "achieved": gbs, "peak": hbm,
                        "unit": "GB/s", "frac": gbs / hbm, "peak_source": f"of {peak_src}: HBM copy bandwidth"}
    # in-step work time per launch (first CTA ready after the PDL wait -> last CTA exit)
    work = _launch_work(h, rl, step, min(args.steps, 40))
    for nm, r_ in hbm_roof.items():
        if nm in work:
            per_launch = r_["bytes_per_step"] / max(1.0, round(prof[nm][0] / args.steps))
            r_["work_us_per_launch"] = work[nm]
            r_["achieved_work"] = per_launch / (work[nm] * 1e-6) / 1e9
            r_["frac_work"] = r_["achieved_work"] / hbm
    if "gemm_main" in work:
        roof["work_us_per_launch"] = work["gemm_main"]
    roof["hbm_kernels"] = hbm_roof

    # ---------------- end to end through the C ABI with host buffers
    # Every step: H2D of its X, dY from pinned host memory, forward + backward, D2H of dA, dB
    # (runlora_step_host).  Two steps are in flight on two streams with their own device
    # buffers and workspaces, so one step's PCIe copies overlap the other's kernels.
    hx = ops["X"].pin_memory()
    hdy = ops["dY"].pin_memory()
    sets = []
    for j in range(2):
        gj = dp.PackedAdapterGrads.create(k, r, m, dev)
        devj = {"W": d["W"], "A": d["A"], "B": d["B"],
                "X": torch.empty_like(d["X"]), "dY": torch.empty_like(d["dY"]),
                "Y": torch.empty_like(Y), "dX": torch.empty_like(dX), "dA": gj.dA, "dB": gj.dB}
        hostj = {"X": hx, "dY": hdy, "dA": torch.empty(k, r, dtype=torch.float32).pin_memory(),
                 "dB": torch.empty(r, m, dtype=torch.float32).pin_memory()}
        sets.append((torch.cuda.Stream(dev), devj, hostj, gj, torch.empty_like(ws)))

    def e2e_run(K):
        cur = torch.cuda.current_stream(dev)
        for st_j, *_ in sets:
            st_j.wait_stream(cur)
        for i in range(K):
            st_j, devj, hostj, gj, wsj = sets[i % 2]
            with torch.cuda.stream(st_j):
                h.step_host(shape, fwd, bwd, hostj, devj, rl.F32, ws=wsj)
                if world > 1:
                    dp.allreduce_adapter_grads(gj)
        for st_j, *_ in sets:
            cur.wait_stream(st_j)

    e2e_run(max(4, args.warmup // 4))
    e2e_steps = max(4, args.steps // 8)
    e2e_ms = timed(lambda: e2e_run(e2e_steps), 1) / e2e_steps
    e2e = {"value": world * n / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": hx.numel() * 2 + hdy.numel() * 2,
           "d2h_bytes_per_step": k * r * 4 + r * m * 4,
           "note": "runlora_step_host: H2D X, dY from pinned host, forward, backward, D2H dA, dB (fp32) every step; "
                   "2 steps in flight on 2 streams (copies of one overlap the other's kernels); Y, dX stay resident"}

    # ---------------- default XW + (XA)B autograd chain on the same box (comparator)
    default = None
    if not args.no_default_chain:
        Xg = d["X"].clone().requires_grad_(True)
        Ag = d["A"].clone().requires_grad_(True)
        Bg = d["B"].clone().requires_grad_(True)
        Wf = d["W"]

        def default_step():
            Xg.grad = Ag.grad = Bg.grad = None
            Yd = Xg @ Wf + (Xg @ Ag) @ Bg
            Yd.backward(d["dY"])
            if world > 1:
                dist.all_reduce(Ag.grad)
                dist.all_reduce(Bg.grad)

        for _ in range(args.warmup):
            default_step()
        dms = timed(default_step, args.steps)
        default = {"ms_per_step": dms, "tokens_per_s": world * n / (dms * 1e-3),
                   "impl": "torch eager bf16 autograd (cuBLAS), XA cached by autograd"}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "bf16", "data": CAPTION,
               "config": {"workload": c.name, "n_per_rank": n, "k": k, "m": m, "r": r,
                          "global_tokens": world * n, "plan": f"F{fwd}+B{bwd}", "criterion": args.criterion,
                          "plan_times_us": plan.as_dict()["time_fwd_us"] | {f"B{v}": t for v, t in
                                                                           plan.as_dict()["time_bwd_us"].items()},
                          "flops_pick": f"F{plan.flops_fwd_pick}+B{plan.flops_bwd_pick}",
                          "parallelism": f"dp{world} token-sharded, " + ("one-shot symmetric-memory allreduce" if sym is not None else "NCCL allreduce") + " of fp32 [dA|dB]",
                          "l2": "inputs larger than L2: per-step working set X, dY, Y, dX 64 MiB each + W 32 MiB "
                                "(288 MiB) > 126 MB L2"},
               "tflops": flops_step / (ms * 1e-3) / 1e12,
               "speedup_vs_default": (default["ms_per_step"] / ms) if default else None,
               "default_chain": default,
               "roofline": roof, "kernels": kernels, "gpu_launches": launches * args.steps,
               "gpu_launches_per_step": launches, "clocks": clk, "e2e": e2e}
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(c, fwd, bwd)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
