"""a8: token-sharded data parallelism through the CUDA kernels, checked
against the FULL-n fp64 oracle.

dA = Xᵀ·dY·Bᵀ and dB = Aᵀ·Xᵀ·dY are sums over tokens (Eq. 3), so the sum
of the P ranks' fp32 [dA | dB] must equal the full-batch gradients; Y and dX are row-wise
(Eq. 1, Eq. 3 third line), so each rank's rows must equal the full evaluation's rows.

1. P in {2, 4, 8} ranks emulated on one GPU (the profiling guide: never run ranks whose
   kernels wait on one another as separate launches on one GPU): shard p's rows
   dp.shard_range(n, P, p) run through forward + backward with rank 0's per-rank plan (both
   the FLOP pick and the measured-time pick at n/P tokens), and the P fp32 buffers are summed
   by ONE runlora_allreduce_sum_f32 launch over the P buffers (the exchange kernel, rank
   order).  C4 shapes (k = m = 2048, r in {8, 32, 128}, n in {4096, 32768}).
2. Two real ranks (torchrun, gloo exchange — a host-side collective, so no GPU kernel waits
   on another) on this GPU: dp.overlapped_backward with the C-ABI kernels per shard, the
   allreduced [dA | dB] against the full-n oracle.
"""
import json
import os
import subprocess
import sys

import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu
TOL = 2e-2
HEALTHY = 5e-3
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    return runlora


def _np(t):
    return t.detach().to(torch.float64).cpu().numpy()


CASES = [synth.C4[(r, n)] for r in (8, 32, 128) for n in (4096, 32768)]


@pytest.mark.parametrize("c", CASES, ids=lambda c: c.name)
def test_emulated_ranks_match_full_n_oracle(rl, c):
    from paper_2312_03415_b200 import dp
    ops = synth.operands(c)
    d = {k: v.cuda() for k, v in ops.items()}
    W, A, B = (_np(ops[k]) for k in ("W", "A", "B"))
    wA, wB = O.adapter_grads(ops["X"].float().numpy(), A, B, ops["dY"].float().numpy())  # full n
    h = rl.handle(0)
    k, m, r = c.k, c.m, c.r
    errs = {}
    for P in (2, 4, 8):
        shards = [dp.shard_range(c.n, P, p) for p in range(P)]
        n0 = shards[0][1] - shards[0][0]
        s0 = rl.make_shape(n0, k, m, r, rl.BF16)
        # rank 0's per-rank plans: Table 1 at n/P, and the measured-time pick on its own shard
        Yt = torch.empty(n0, m, dtype=torch.bfloat16, device="cuda")
        dXt = torch.empty(n0, k, dtype=torch.bfloat16, device="cuda")
        gt = dp.PackedAdapterGrads.create(k, r, m, "cuda")
        pf = rl.select_by_flops(s0)
        pt = h.select(s0, rl.BY_TIME, ops={"X": d["X"][:n0], "W": d["W"], "A": d["A"], "B": d["B"],
                                           "dY": d["dY"][:n0], "Y": Yt, "dX": dXt, "dA": gt.dA, "dB": gt.dB},
                      grad_dtype=rl.F32)
        assert (pf.fwd, pf.bwd) == O.select_by_flops(n0, k, m, r)
        rows = synth.sample_rows(c.n, P=P, seed_cfg=c.cfg * 100 + c.sub)
        ridx = torch.as_tensor(rows, device="cuda")
        wY = O.forward_rows(_np(ops["X"][rows]), W, A, B)
        wX = O.dX_rows(_np(ops["dY"][rows]), W, A, B)
        for fwd, bwd in sorted({(int(pf.fwd), int(pf.bwd)), (int(pt.fwd), int(pt.bwd))}):
            Y = torch.full((c.n, m), float("nan"), dtype=torch.bfloat16, device="cuda")
            dX = torch.full((c.n, k), float("nan"), dtype=torch.bfloat16, device="cuda")
            bufs = [dp.PackedAdapterGrads.create(k, r, m, "cuda") for _ in range(P)]
            for b in bufs:
                b.flat.fill_(float("nan"))
            for p, (lo, hi) in enumerate(shards):
                sp = rl.make_shape(hi - lo, k, m, r, rl.BF16)
                h.forward(fwd, sp, d["X"][lo:hi], d["W"], d["A"], d["B"], Y[lo:hi])
                h.backward(bwd, sp, d["X"][lo:hi], d["W"], d["A"], d["B"], d["dY"][lo:hi], dX[lo:hi], bufs[p].dA,
                           bufs[p].dB)
            out = torch.full((k * r + r * m,), float("nan"), device="cuda")
            h.allreduce_sum_f32([b.flat.data_ptr() for b in bufs], out)  # the a8 exchange, rank order
            torch.cuda.synchronize()
            # the exchange sums in rank order: bit-identical to the same fp32 sum on the host side
            ref = bufs[0].flat.clone()
            for b in bufs[1:]:
                ref += b.flat
            assert torch.equal(out, ref)
            e = {"dA": O.rel_fro(_np(out[:k * r].view(k, r)), wA), "dB": O.rel_fro(_np(out[k * r:].view(r, m)), wB),
                 "Y": O.rel_fro(_np(Y[ridx]), wY), "dX": O.rel_fro(_np(dX[ridx]), wX)}
            errs[(P, f"F{fwd}+B{bwd}")] = e
    bad = {key: e for key, e in errs.items() if max(e.values()) > TOL}
    assert not bad, bad
    assert max(max(e.values()) for e in errs.values()) < HEALTHY, errs


_CHILD = r"""
import json, os, sys, torch
import torch.distributed as dist
sys.path.insert(0, {root!r})
import synth
from paper_2312_03415_b200 import dp
from paper_2312_03415_b200 import runlora as rl
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
c = synth.C4[(32, 4096)]
ops = synth.operands(c)
lo, hi = dp.shard_range(c.n, world, rank)
d = {{k: (v[lo:hi] if k in ("X", "dY") else v).cuda() for k, v in ops.items()}}
h = rl.handle(0)
shape = rl.make_shape(hi - lo, c.k, c.m, c.r, rl.BF16)
p = rl.select_by_flops(shape)
fwd, bwd = dp.broadcast_plan(int(p.fwd), int(p.bwd))
g = dp.PackedAdapterGrads.create(c.k, c.r, c.m, "cuda")
Y = torch.empty(hi - lo, c.m, dtype=torch.bfloat16, device="cuda")
dX = torch.empty(hi - lo, c.k, dtype=torch.bfloat16, device="cuda")
h.forward(fwd, shape, d["X"], d["W"], d["A"], d["B"], Y)
work = dp.overlapped_backward(
    lambda: h.backward_params(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], g.dA, g.dB),
    lambda: h.backward_input(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX), g,
    comm_stream=torch.cuda.Stream())
work.wait()
torch.cuda.synchronize()
if rank == 0:
    torch.save({{"dA": g.dA.cpu(), "dB": g.dB.cpu(), "plan": (fwd, bwd)}}, sys.argv[1])
dist.barrier()
dist.destroy_process_group()
"""


def test_two_ranks_gloo_allreduce_matches_full_n_oracle(tmp_path):
    script = tmp_path / "child.py"
    script.write_text(_CHILD.format(root=ROOT))
    f = tmp_path / "out.pt"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29581", str(script), str(f)]
    p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    got = torch.load(f)
    c = synth.C4[(32, 4096)]
    ops = synth.operands(c)
    wA, wB = O.adapter_grads(ops["X"].float().numpy(), _np(ops["A"]), _np(ops["B"]), ops["dY"].float().numpy())
    eA, eB = O.rel_fro(got["dA"].double().numpy(), wA), O.rel_fro(got["dB"].double().numpy(), wB)
    assert eA < HEALTHY and eB < HEALTHY, json.dumps({"dA": eA, "dB": eB, "plan": got["plan"]})
