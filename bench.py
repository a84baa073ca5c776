#!/usr/bin/env python
"""Benchmark of the RunLoRA hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--r 16] [--impl reference]

A step is one pass of the whole hot path over one batch: the plan
chosen by the selector (cached, chosen before warm-up), forward, backward (adapter
grads then dX) and — for N > 1 — the token-sharded DP exchange (allreduce of the
packed fp32 [dA | dB], overlapped with dX).  Workload of `value`: BASELINE.json
configs[1] (Llama-7B attention projection, n = 8192 tokens, k = m = 4096), rank
r = 16; under torchrun every rank runs that workload on its own 8192 tokens
(weak scaling) and value = all ranks' tokens / max-over-ranks step time.

Extra keys (same run): `c4_strong` — BASELINE.json configs[3] at n = 131072 global
tokens token-sharded over the N ranks (strong scaling; DDP-wrapped default chain as the
comparator), `c5` — configs[4], the 32-layer stack at 64 x 1024 global tokens per step
as micro-batches of 8192 tokens per rank.

`--impl reference` times the CPU fp64 oracle (the only reference this tier has;
oracle/) on the host cores on bounded token slices of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "LoRA-linear fwd+bwd tokens/s, tensor-pipe util, speedup vs default XW+(XA)B"
UNIT = "tokens/s"
CAPTION = "synthetic: seeded i.i.d. Gaussian operands with BASELINE.json's laws (no dataset/weights)"
ORACLE_SLICE = 1024  # tokens per oracle slice (cpu_baseline and the reference arm alike)
# steps in flight in the e2e leg (own streams, device buffers and workspaces): 4 measured best
# (2.77-2.79 M tokens/s vs 2.70 with 3 and 2.59 with 6 at C2)
E2E_SETS = int(os.environ.get("RUNLORA_E2E_SETS", "4"))


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
    """SM clock and clock-event reasons from NVML every `period` seconds on a background
    thread, from before selection to the end of the run; `mark(name)` brackets a phase (the
    timed region) so its own samples are reported too."""

    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80}

    def __init__(self, device: torch.device, period: float = 0.002):
        self.period = period
        self.samples = []  # (t, sm_mhz, reasons bitmask)
        self.marks = {}
        self.err = None
        self.h = None
        self.smax = None
        try:
            import pynvml as N
            self.N = N
            N.nvmlInit()
            try:
                bus = torch.cuda.get_device_properties(device).pci_bus_id
                dom = torch.cuda.get_device_properties(device).pci_domain_id
                dev = torch.cuda.get_device_properties(device).pci_device_id
                self.h = N.nvmlDeviceGetHandleByPciBusId(f"{dom:08x}:{bus:02x}:{dev:02x}.0")
            except Exception:
                self.h = N.nvmlDeviceGetHandleByIndex(device.index or 0)
            self.smax = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self._reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
        except Exception as e:  # reported in the line
            self.err = f"nvml unavailable: {e}"
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append((time.perf_counter(), float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)),
                                     int(self._reasons(self.h))))
            except Exception as e:
                self.err = str(e)
                return
            time.sleep(self.period)

    def start(self):
        if self.h is not None:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def mark(self, name, t0, t1):
        self.marks[name] = (t0, t1)

    def _summary(self, s):
        busy = [x[1] for x in s if self.smax is None or x[1] > 0.5 * self.smax]
        reasons = set()
        for _, _, b in s:
            reasons.update(nm for nm, bit in self.BITS.items() if b & bit)
        return {"sm_mhz": float(np.median(busy)) if busy else None, "samples": len(s), "reasons": sorted(reasons)}

    def stop(self):
        self._stop.set()
        if self._th is not None:
            self._th.join(timeout=2)
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "nvml unavailable"], "samples": 0}
        out = self._summary(self.samples)
        out["sm_max_mhz"] = self.smax
        out["source"] = f"NVML every {self.period * 1e3:.0f} ms from selection to the end of the run"
        for name, (t0, t1) in self.marks.items():
            out[name] = self._summary([x for x in self.samples if t0 <= x[0] <= t1])
        if self.err:
            out["error"] = self.err
        return out


# ------------------------------------------------------------- oracle timing
def oracle_rate(c, fwd, bwd, target_s=None, slices=None):
    """The oracle (fp64 NumPy, as it stands) on contiguous ORACLE_SLICE-token slices of the
    workload, cycling over its first 4 slices, until `target_s` seconds of CPU work or
    `slices` slices were timed.  Each slice includes the n-independent W+AB term.
    Returns (tokens/s, slices timed, seconds)."""
    import oracle as O
    ns = min(ORACLE_SLICE, c.n)
    nsl = max(1, min(c.n, 4 * ns) // ns)
    ops = synth.operands(synth.case(c.name, c.cfg, c.sub, nsl * ns, c.k, c.m, c.r, c.dtype))
    W, A, B = (ops[k].double().numpy() for k in ("W", "A", "B"))
    Xa, dYa = ops["X"].double().numpy(), ops["dY"].double().numpy()
    t_total, i = 0.0, 0
    while (target_s is not None and t_total < target_s) or (slices is not None and i < slices):
        s0 = (i % nsl) * ns
        X, dY = Xa[s0:s0 + ns], dYa[s0:s0 + ns]
        t0 = time.perf_counter()
        O.forward(fwd, X, W, A, B)
        O.backward(bwd, X, W, A, B, dY)
        t_total += time.perf_counter() - t0
        i += 1
    return (i * ns / t_total if t_total > 0 else 0.0), i, t_total


def _oracle_sample(c, fwd, bwd, i, t):
    return (f"{i} contiguous {min(ORACLE_SLICE, c.n)}-token slices of {c.name} ({t:.1f} s of CPU work); oracle "
            f"forward{fwd}+backward{bwd} (the FLOP-criterion pair, Table 1 argmin, P:316) in fp64 NumPy/BLAS on "
            "all host cores, each slice including the n-independent W+AB term")


def run_reference(args):
    """Reference arm: the CPU fp64 oracle, as it stands, on the same workload and metric;
    each step is one bounded token slice (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    c = _case(args.r)
    f, b = O.select_by_flops(c.n, c.k, c.m, c.r)
    oracle_rate(c, f, b, slices=args.warmup)
    val, i, t = oracle_rate(c, f, b, slices=args.steps)
    cores = len(os.sched_getaffinity(0))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / i * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": CAPTION,
            "config": {"workload": c.name, "n": c.n, "k": c.k, "m": c.m, "r": c.r,
                       "sample_tokens_per_step": min(ORACLE_SLICE, c.n), "plan": f"F{f}+B{b}", "criterion": "flops"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": _oracle_sample(c, f, b, i, t)},
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


class DefaultLoRA(torch.nn.Module):
    """The paper's default chain Y = XW + (XA)B as torch autograd (cuBLAS); W frozen."""

    def __init__(self, W, A, B):
        super().__init__()
        self.register_buffer("W", W)
        self.A = torch.nn.Parameter(A.clone())
        self.B = torch.nn.Parameter(B.clone())

    def forward(self, x):
        return x @ self.W + (x @ self.A) @ self.B


# ------------------------------------------------------------------ main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--r", type=int, default=16, choices=sorted(synth.C2))
    ap.add_argument("--impl", default="runlora", choices=["runlora", "reference"])
    ap.add_argument("--criterion", default="time", choices=["flops", "time", "hybrid"])
    ap.add_argument("--plan", default=None, help="force a variant pair, e.g. 1,1 (skips selection)")
    ap.add_argument("--blocks", type=int, default=5,
                    help="interleaved blocks of K steps (RunLoRA, default chain, alternating) for the speedup")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-default-chain", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--c5-steps", type=int, default=2)
    ap.add_argument("--no-wprime-reuse", action="store_true", help="C5: rebuild W' every micro-batch")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the multi-rank code path on one GPU (not a performance mode)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world and not (args.impl == "reference" and world == 1):
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch N > 1 ranks with "
                         "python -m torch.distributed.run --nproc-per-node N bench.py --gpus N\n")
        return 2
    if args.impl == "reference":
        return run_reference(args)

    import torch.distributed as dist
    # per-launch records (first/last CTA ready and exit): the in-step work time of each
    # kernel, reported beside the CUDA-event durations (read over a window of steps below)
    os.environ.setdefault("RUNLORA_LTRACE", "1")
    from paper_2312_03415_b200 import runlora as rl
    from paper_2312_03415_b200 import dp

    rank = int(os.environ.get("RANK", "0"))
    transport = os.environ.get("RUNLORA_DP_TRANSPORT", "nccl")
    if world > 1 and transport == "nccl":
        # the persistent dX GEMM fills every SM it runs on (registers and shared memory): two
        # SMs left free let NCCL's allreduce kernel run beside it
        os.environ.setdefault("RUNLORA_COMM_SMS", "2")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    clocks = ClockSampler(dev).start()
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
    # DP exchange: NCCL allreduce (default), the one-shot symmetric-memory kernel ("symm"), or the
    # exchange fused into the dX GEMM launch ("fused", dp.FusedExchange) — both opt-in
    sym = fused = None
    if world > 1 and args.backend == "nccl" and transport == "symm":
        sym = dp.SymmetricAllreduce(k, r, m, dev, h)
    if world > 1 and args.backend == "nccl" and transport == "fused":
        fused = dp.FusedExchange(k, r, m, dev, h, multicast=os.environ.get("RUNLORA_DP_MULTICAST") == "1")
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
        if fused is not None:
            fused.backward(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, g.dA, g.dB, ws=ws)
        elif world > 1:
            work = dp.overlapped_backward(
                lambda: h.backward_params(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], g.dA, g.dB, ws=ws),
                lambda: h.backward_input(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, ws=ws),
                g, comm_stream=comm, exchange=sym)
            work.wait()
        else:
            h.backward(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, g.dA, g.dB, ws=ws)

    def timed(fn, K, mark=None):
        """Device time per call of fn over K back-to-back calls (CUDA events on the current
        stream, barrier + synchronize on both sides), max over ranks."""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(K):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        if mark:
            clocks.mark(mark, t0, time.perf_counter())
        ms = e0.elapsed_time(e1) / K
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # ---------------- device-resident timing (value): exactly K steps after W warm-ups
    # Time-mode selection runs every candidate for ~1-2 s and leaves the GPU at its power cap;
    # one idle second lets the clocks recover, so the short timed region starts from the same
    # power state as MEASURED_PEAKS' burst figure (clocks.timed_region records what it saw).
    torch.cuda.synchronize(dev)
    time.sleep(1.0)
    for _ in range(args.warmup):
        step()
    l0 = h.launch_count()
    ms = timed(step, args.steps, mark="timed_region")
    launches = (h.launch_count() - l0) // args.steps
    value = world * n / (ms * 1e-3)
    flops_step = plan.flops_fwd[fwd] + plan.flops_bwd[bwd]

    # ---------------- per-kernel profile (same steps, library CUDA events on the launch stream)
    # A first pass fills the library's event pool: creating events while the kernels run
    # keeps the host behind the GPU, and the idle gaps would land inside the event pairs.
    h.profile_enable(True)
    for _ in range(args.steps):
        step()
    h.profile_read(reset=True)
    time.sleep(0.5)
    for _ in range(args.warmup):
        step()
    h.profile_read(reset=True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize(dev)
    prof_s = time.perf_counter() - t0
    clocks.mark("profile_pass", t0, time.perf_counter())
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
    nl = []
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            gm = json.load(f).get("gemm_main", {})
        traffic = gm.get("dram_bytes_per_launch")
        nl = gm.get("launches", [])
    except Exception:
        pass

    # in-step work time per launch (first CTA ready after the PDL wait -> last CTA exit)
    work = _launch_work(h, rl, step, min(args.steps, 40))

    # ---------------- default XW + (XA)B autograd chain, interleaved with RunLoRA blocks
    default = None
    if not args.no_default_chain:
        mod = DefaultLoRA(d["W"], d["A"], d["B"]).to(dev)
        if world > 1:
            mod = torch.nn.parallel.DistributedDataParallel(mod, device_ids=[local])
        Xg = d["X"].clone().requires_grad_(True)

        def default_step():
            Xg.grad = None
            for p_ in mod.parameters():
                p_.grad = None
            mod(Xg).backward(d["dY"])

        for _ in range(args.warmup):
            default_step()
        t_rl, t_def = [], []
        for _ in range(args.blocks):
            t_rl.append(timed(step, args.steps))
            t_def.append(timed(default_step, args.steps, mark="default_chain"))
        default = {"ms_per_step": float(np.median(t_def)), "tokens_per_s": world * n / (np.median(t_def) * 1e-3),
                   "runlora_ms_per_step_interleaved": float(np.median(t_rl)),
                   "blocks": args.blocks, "ms_blocks": t_def, "runlora_ms_blocks": t_rl,
                   "impl": "torch eager bf16 autograd (cuBLAS), XA cached by autograd"
                           + (", DistributedDataParallel (allreduce of A.grad, B.grad overlapped with backward)"
                              if world > 1 else ""),
                   "note": f"{args.blocks} alternating blocks of K steps (RunLoRA, default, ...); medians"}
        del mod, Xg

    # ---------------- end to end through the C ABI with host buffers
    # Every step: H2D of its X, dY from pinned host memory, forward + backward (+ the DP
    # allreduce through the exchange hook at N > 1), D2H of dA, dB and of Y, dX
    # (runlora_step_host).  E2E_SETS steps are in flight on as many streams with their own
    # device buffers and workspaces: a stream runs its step's H2D, kernels and D2H in order, so
    # with several of them one step's inputs stream in while another's outputs stream out and
    # a third computes — both PCIe directions stay busy (tools/pcie_probe.py: 128 MiB each way
    # take 2.7 ms concurrently, the floor of a C2 step's 256 MiB of copies).
    hx = ops["X"].pin_memory()
    hdy = ops["dY"].pin_memory()
    sets = []
    for j in range(E2E_SETS):
        gj = dp.PackedAdapterGrads.create(k, r, m, dev)
        devj = {"W": d["W"], "A": d["A"], "B": d["B"],
                "X": torch.empty_like(d["X"]), "dY": torch.empty_like(d["dY"]),
                "Y": torch.empty_like(Y), "dX": torch.empty_like(dX), "dA": gj.dA, "dB": gj.dB}
        hostj = {"X": hx, "dY": hdy, "dA": torch.empty(k, r, dtype=torch.float32).pin_memory(),
                 "dB": torch.empty(r, m, dtype=torch.float32).pin_memory(),
                 "Y": torch.empty(n, m, dtype=torch.bfloat16).pin_memory(),
                 "dX": torch.empty(n, k, dtype=torch.bfloat16).pin_memory()}
        sets.append((torch.cuda.Stream(dev), devj, hostj, gj, torch.empty_like(ws)))

    def e2e_run(K, outputs=True):
        cur = torch.cuda.current_stream(dev)
        for st_j, *_ in sets:
            st_j.wait_stream(cur)
        for i in range(K):
            st_j, devj, hostj, gj, wsj = sets[i % len(sets)]
            hj = hostj if outputs else {kk: v for kk, v in hostj.items() if kk not in ("Y", "dX")}
            with torch.cuda.stream(st_j):
                h.step_host(shape, fwd, bwd, hj, devj, rl.F32, ws=wsj,
                            exchange=(lambda gj=gj: dp.allreduce_adapter_grads(gj)) if world > 1 else None)
        for st_j, *_ in sets:
            cur.wait_stream(st_j)

    e2e_steps = max(12, args.steps)  # long enough that the 3-deep pipeline fill and drain are a small share
    res = {}
    for outputs in (True, False):
        e2e_run(max(4, args.warmup // 2), outputs)
        res[outputs] = timed(lambda: e2e_run(e2e_steps, outputs), 1, mark="e2e" if outputs else None) / e2e_steps
    xb, yb = hx.numel() * 2, hdy.numel() * 2
    e2e = {"value": world * n / (res[True] * 1e-3), "unit": UNIT, "ms_per_step": res[True],
           "h2d_bytes_per_step": xb + yb, "d2h_bytes_per_step": k * r * 4 + r * m * 4 + yb + xb,
           "note": "runlora_step_host every step: H2D X, dY from pinned host; forward; backward"
                   + ("; NCCL allreduce of fp32 [dA|dB] through the exchange hook" if world > 1 else "")
                   + f"; D2H of Y, dX (bf16) and dA, dB (fp32). {E2E_SETS} steps in flight on {E2E_SETS} streams "
                     "(PCIe-bound)",
           "grads_only": {"value": world * n / (res[False] * 1e-3), "ms_per_step": res[False],
                          "d2h_bytes_per_step": k * r * 4 + r * m * 4,
                          "note": "same, but only dA, dB come back (Y, dX stay resident)"}}
    del sets

    c4 = None if args.no_c4 else c4_strong(args, rl, dp, dist, dev, local, world, rank, h, timed)
    c5 = None if args.no_c5 else c5_stack(args, rl, dist, dev, local, world, rank, timed)

    clk = clocks.stop()
    # roofline denominator from the run itself: a short timed region (the driver's 20 steps
    # are ~10 ms) or clocks within 5 % of max -> the burst cuBLAS figure; a long region at
    # power-capped clocks -> the sustained one
    timed_s = ms * args.steps * 1e-3
    near_max = clk.get("sm_mhz") and clk.get("sm_max_mhz") and clk["sm_mhz"] >= 0.95 * clk["sm_max_mhz"]
    burst = timed_s < 2.0 or bool(near_max)
    peak = peaks["bf16_tflops"] if burst else (peaks.get("bf16_tflops_sustained") or peaks["bf16_tflops"])
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if achieved else None, "traffic": traffic,
            "kernel": "gemm_main (tcgen05 Y / dX GEMM, 256x512 + 256x256 pair tiles)",
            "peak_kind": "burst" if burst else "sustained",
            "peak_source": f"of {peak_src}: cuBLAS bf16 {'burst' if burst else 'sustained (seconds-long loop)'}; "
                           f"chosen because the timed region was {timed_s:.3f} s (profile pass {prof_s:.3f} s) "
                           f"at a median {clk.get('sm_mhz')} of {clk.get('sm_max_mhz')} MHz",
            "peak_burst": peaks["bf16_tflops"], "peak_sustained": peaks.get("bf16_tflops_sustained"),
            "frac_of_burst": achieved / peaks["bf16_tflops"] if achieved else None,
            "flops_per_launch": flops_per_launch,
            "duration_us_per_launch": per_launch_s * 1e6 if main_launches else None}
    if nl:
        roof["tensor_pipe_pct_ncu"] = sum(x.get("tensor_pipe_pct", 0) for x in nl) / len(nl)
    if "gemm_main" in work:
        roof["work_us_per_launch"] = work["gemm_main"]
        roof["achieved_work"] = flops_per_launch / (work["gemm_main"] * 1e-6) / 1e12
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
        if nm in work:
            per_launch = bytes_step / max(1.0, round(cnt / args.steps))
            hbm_roof[nm]["work_us_per_launch"] = work[nm]
            hbm_roof[nm]["achieved_work"] = per_launch / (work[nm] * 1e-6) / 1e9
            hbm_roof[nm]["frac_work"] = hbm_roof[nm]["achieved_work"] / hbm
        hbm_roof[nm]["note"] = ("achieved/frac: CUDA events around each launch in the profile pass — the events "
                                "break the PDL chain, so each interval also holds the launch latency and the CTAs' "
                                "start-up that PDL otherwise overlaps with the previous kernel; "
                                "achieved_work/frac_work: the launch's own span from the kernel's timestamps "
                                "(first CTA past the PDL wait -> last CTA exit) in the timed steps")
    roof["hbm_kernels"] = hbm_roof

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "bf16", "data": CAPTION,
               "config": {"workload": c.name, "n_per_rank": n, "k": k, "m": m, "r": r,
                          "global_tokens": world * n, "plan": f"F{fwd}+B{bwd}", "criterion": args.criterion,
                          "plan_times_us": plan.as_dict()["time_fwd_us"] | {f"B{v}": t for v, t in
                                                                           plan.as_dict()["time_bwd_us"].items()},
                          "flops_pick": f"F{plan.flops_fwd_pick}+B{plan.flops_bwd_pick}",
                          "parallelism": f"dp{world} token-sharded, " + (
                              "one-shot symmetric-memory allreduce" if sym is not None else
                              "exchange fused into the dX GEMM launch" if fused is not None else
                              "NCCL allreduce") + " of fp32 [dA|dB]",
                          "l2": "inputs larger than L2: per-step working set X, dY, Y, dX 64 MiB each + W 32 MiB "
                                "(288 MiB) > 126 MB L2"},
               "tflops": flops_step / (ms * 1e-3) / 1e12,
               "speedup_vs_default": (default["ms_per_step"] / default["runlora_ms_per_step_interleaved"])
               if default else None,
               "default_chain": default,
               "roofline": roof, "kernels": kernels, "gpu_launches": launches * args.steps,
               "gpu_launches_per_step": launches, "clocks": clk, "e2e": e2e, "c4_strong": c4, "c5": c5}
        if world == 1 and not args.no_cpu_baseline:
            # same definition as the reference arm: the FLOP-criterion pair on 1024-token slices
            import oracle as O
            f_o, b_o = O.select_by_flops(n, k, m, r)
            v, i, t = oracle_rate(c, f_o, b_o, target_s=12.0)
            out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": len(os.sched_getaffinity(0)),
                                   "kind": "oracle", "sample": _oracle_sample(c, f_o, b_o, i, t)}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------ C4 strong scaling
def c4_strong(args, rl, dp, dist, dev, local, world, rank, h, timed):
    """BASELINE.json configs[3] at its largest n: 131072 global tokens (256 x 512), k = m =
    2048, r in {8, 32, 128}, token-sharded over the ranks (dp.shard_range) — strong scaling.
    Per rank: the plan selected at the per-rank n (time criterion, rank 0's broadcast),
    forward, adapter grads, NCCL allreduce of fp32 [dA|dB] overlapped with dX.  Comparator:
    the default chain under DistributedDataParallel (N > 1).  Operands are drawn on the
    device with torch's generator under synth's laws (timing only; parity of these shapes is
    tests/test_gpu_dp_shards.py's job)."""
    n_glob, k, m = 131072, 2048, 2048
    s0, s1 = dp.shard_range(n_glob, world, rank)
    n = s1 - s0
    out = {"workload": "C4_opt_n131072", "global_tokens": n_glob, "k": k, "m": m, "tokens_per_rank": n,
           "parallelism": f"dp{world} token-sharded (strong scaling)", "runs": {}}
    gen = torch.Generator(device=dev)
    for r in (8, 32, 128):
        gen.manual_seed(2312 * 1000 + r)  # replicated W, A, B: same seed on every rank
        W = (torch.randn(k, m, generator=gen, device=dev) / k ** 0.5).to(torch.bfloat16)
        A = (torch.randn(k, r, generator=gen, device=dev) / k ** 0.5).to(torch.bfloat16)
        B = (torch.randn(r, m, generator=gen, device=dev) / r ** 0.5).to(torch.bfloat16)
        gen.manual_seed(2312 * 1000 + r + 17 * (rank + 1))  # this rank's token shard
        X = torch.randn(n, k, generator=gen, device=dev).to(torch.bfloat16)
        dY = torch.randn(n, m, generator=gen, device=dev).to(torch.bfloat16)
        Y = torch.empty(n, m, dtype=torch.bfloat16, device=dev)
        dX = torch.empty(n, k, dtype=torch.bfloat16, device=dev)
        g = dp.PackedAdapterGrads.create(k, r, m, dev)
        shape = rl.make_shape(n, k, m, r, rl.BF16)
        plan = h.select(shape, rl.BY_TIME, ops={"X": X, "W": W, "A": A, "B": B, "dY": dY, "Y": Y, "dX": dX,
                                                "dA": g.dA, "dB": g.dB}, grad_dtype=rl.F32)
        fwd, bwd = int(plan.fwd), int(plan.bwd)
        if world > 1:
            fwd, bwd = dp.broadcast_plan(fwd, bwd, device=dev)
        ws = h.workspace(shape)
        comm = torch.cuda.Stream(dev) if world > 1 else None

        def step():
            h.forward(fwd, shape, X, W, A, B, Y, ws)
            if world > 1:
                dp.overlapped_backward(
                    lambda: h.backward_params(bwd, shape, X, W, A, B, dY, g.dA, g.dB, ws=ws),
                    lambda: h.backward_input(bwd, shape, X, W, A, B, dY, dX, ws=ws), g, comm_stream=comm).wait()
            else:
                h.backward(bwd, shape, X, W, A, B, dY, dX, g.dA, g.dB, ws=ws)

        for _ in range(args.warmup):
            step()
        ms = timed(step, args.steps)
        run = {"plan": f"F{fwd}+B{bwd}", "flops_pick": f"F{plan.flops_fwd_pick}+B{plan.flops_bwd_pick}",
               "ms_per_step": ms, "tokens_per_s": n_glob / (ms * 1e-3),
               "tflops": world * (plan.flops_fwd[fwd] + plan.flops_bwd[bwd]) / (ms * 1e-3) / 1e12}
        if not args.no_default_chain:
            mod = DefaultLoRA(W, A, B).to(dev)
            if world > 1:
                mod = torch.nn.parallel.DistributedDataParallel(mod, device_ids=[local])
            Xg = X.clone().requires_grad_(True)

            def default_step():
                Xg.grad = None
                for p_ in mod.parameters():
                    p_.grad = None
                mod(Xg).backward(dY)

            for _ in range(args.warmup):
                default_step()
            t_rl, t_def = [], []
            for _ in range(3):
                t_rl.append(timed(step, args.steps))
                t_def.append(timed(default_step, args.steps))
            run["default_ms_per_step"] = float(np.median(t_def))
            run["runlora_ms_per_step_interleaved"] = float(np.median(t_rl))
            run["speedup_vs_default"] = float(np.median(t_def) / np.median(t_rl))
            del mod, Xg
        out["runs"][f"r{r}"] = run
        del X, dY, Y, dX, W, A, B, g
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------ C5 stack
def c5_stack(args, rl, dist, dev, local, world, rank, timed):
    """BASELINE.json configs[4]: the 32-layer stack of LoRA linears (Llama-7B projection
    shapes, r = 16, R15 dataflow), global batch 64 x 1024 = 65536 tokens per step,
    token-sharded over the ranks; each rank runs its 65536/N tokens as micro-batches of 8192
    with fp32 adapter-gradient accumulation (BucketedGradSync: 25 MB buckets, allreduced
    after the last micro-batch as they complete, on a communication stream).  Comparator:
    the same stack with every linear as the default chain (DDP with no_sync() on all but the
    last micro-batch at N > 1).  Weights are drawn on the device (timing only; the stack's
    parity is tests/test_gpu_stack.py)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from stack_bench import DefaultLinear, build  # noqa: E402
    from paper_2312_03415_b200.stack import LINEARS, BucketedGradSync, LoRALayer, LoRAStack, plan_model
    layers, d, f, r, mb = 32, 4096, 11008, 16, 8192
    n_glob = 64 * 1024
    per_rank = n_glob // world
    micro = max(1, per_rank // mb)
    model = build(layers, d, f, r, dev)
    if not args.no_wprime_reuse:
        model.reuse_wprime_(True)  # W'ᵀ once per step, reused by the micro-batches (R20)
    plans = plan_model(model, mb, rl.BY_TIME)
    if world > 1:  # every rank runs rank 0's plans
        t = torch.tensor([v for _, _, lin in model.linears() for v in lin.plan], device=dev)
        dist.broadcast(t, src=0)
        for i, (_, _, lin) in enumerate(model.linears()):
            lin.plan = (int(t[2 * i]), int(t[2 * i + 1]))
    comm = torch.cuda.Stream(dev) if world > 1 else None
    sync = BucketedGradSync.for_model(model, comm_stream=comm)
    gen = torch.Generator(device=dev).manual_seed(7 + rank)
    xs = [torch.randn(mb, d, generator=gen, device=dev).to(torch.bfloat16) for _ in range(micro)]
    dys = [torch.randn(mb, d, generator=gen, device=dev).to(torch.bfloat16) for _ in range(micro)]

    def step():
        sync.begin_step(micro)
        for x, dy in zip(xs, dys):
            xi = x.detach().requires_grad_(True)
            model(xi).backward(dy)
        sync.finish()

    def peak_extra(fn):
        """Peak device memory of one step above what is resident before it (activations,
        saved tensors, workspaces) — the quantity the paper's memory claim is about."""
        torch.cuda.synchronize(dev)
        before = torch.cuda.memory_allocated(dev)
        torch.cuda.reset_peak_memory_stats(dev)
        fn()
        torch.cuda.synchronize(dev)
        return torch.cuda.max_memory_allocated(dev) - before

    w = max(1, min(args.warmup, 1))
    for _ in range(w):
        step()
    ms = timed(step, args.c5_steps)
    mem = peak_extra(step)
    cache_bytes = sum(lin.wcache.Wpt.numel() * 2 for _, _, lin in model.linears()
                      if lin.wcache is not None and lin.wcache.Wpt is not None)
    out = {"workload": "C5_stack_32L", "layers": layers, "r": r, "global_tokens": n_glob,
           "tokens_per_rank": per_rank, "micro_batches": micro, "micro_batch_tokens": mb,
           "plans": {f"{k}x{m}": f"F{int(p.fwd)}+B{int(p.bwd)}" for (k, m, _), p in plans.items()},
           "steps": args.c5_steps, "warmup": w, "ms_per_step": ms, "tokens_per_s": n_glob / (ms * 1e-3),
           "parallelism": f"dp{world} token-sharded, bucketed NCCL allreduce of fp32 adapter grads",
           "wprime_reuse": all(lin.wcache is not None for _, _, lin in model.linears()),
           "wprime_cache_bytes": cache_bytes,
           "step_peak_extra_bytes": mem,
           "note": "wprime_reuse: forward2's W'ᵀ built once per step per linear and reused by the "
                   "micro-batches (runlora_wprime_t + runlora_forward_wprime, lora.WPrimeCache; "
                   "resident, wprime_cache_bytes); step_peak_extra_bytes: peak memory of one step above "
                   "the resident weights and caches"}
    if not args.no_default_chain:
        base = LoRAStack([LoRALayer({nm: DefaultLinear(L.lin[nm]) for nm in LINEARS}) for L in model.layers]).to(dev)
        if world > 1:
            base = torch.nn.parallel.DistributedDataParallel(base, device_ids=[local])

        def default_step():
            for p_ in base.parameters():
                p_.grad = None
            for i, (x, dy) in enumerate(zip(xs, dys)):
                xi = x.detach().requires_grad_(True)
                if world > 1 and i < micro - 1:
                    with base.no_sync():
                        base(xi).backward(dy)
                else:
                    base(xi).backward(dy)

        for _ in range(w):
            default_step()
        ms_def = timed(default_step, args.c5_steps)
        out["default_step_peak_extra_bytes"] = peak_extra(default_step)
        out["default_ms_per_step"] = ms_def
        out["speedup_vs_default"] = ms_def / ms
        del base
    del model, sync, xs, dys
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    sys.exit(main())
