"""The data-parallel code paths on the GPU with a real NCCL process group of one rank
(this round has one GPU; the multi-rank host logic is tests/test_dp_gloo.py and
tests/test_dp_stack_gloo.py): adapter-gradient allreduce on a communication stream
overlapped with the dX GEMM (dp.overlapped_backward), and the stack's bucketed sync with
its collectives issued from the backward.  A one-rank SUM is the identity, so the results
must equal the non-distributed ones bit for bit.
"""
import socket

import pytest
import torch
import torch.distributed as dist

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_overlapped_backward_nccl(nccl):
    from paper_2312_03415_b200 import dp
    from paper_2312_03415_b200 import runlora as rl
    c = synth.case("dp_nccl", 0, 40, 1024, 1024, 768, 16, "bf16")
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    for bwd in (1, 5):
        g = dp.PackedAdapterGrads.create(c.k, c.r, c.m, "cuda")
        dX = torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda")
        work = dp.overlapped_backward(
            lambda: h.backward_params(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], g.dA, g.dB),
            lambda: h.backward_input(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX),
            g, comm_stream=torch.cuda.Stream())
        work.wait()
        torch.cuda.synchronize()
        dA = torch.empty(c.k, c.r, device="cuda")
        dB = torch.empty(c.r, c.m, device="cuda")
        dX2 = torch.empty_like(dX)
        h.backward(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX2, dA, dB)
        torch.cuda.synchronize()
        assert torch.equal(g.dA, dA) and torch.equal(g.dB, dB) and torch.equal(dX, dX2)


def test_stack_bucketed_sync_nccl(nccl):
    from paper_2312_03415_b200 import runlora as rl
    from paper_2312_03415_b200.stack import BucketedGradSync, LoRAStack, plan_model
    weights = synth.c5_weights(1, 256, d=1024, f=2816, r=16)
    x, dy = synth.c5_io(256, d=1024)
    ref = LoRAStack.from_weights(weights, "cuda")
    plan_model(ref, 256, rl.BY_FLOPS)
    xr = x.cuda().requires_grad_(True)
    ref(xr).backward(dy.cuda())
    model = LoRAStack.from_weights(weights, "cuda")
    plan_model(model, 256, rl.BY_FLOPS)
    sync = BucketedGradSync.for_model(model, bucket_bytes=64 << 10, comm_stream=torch.cuda.Stream(),
                                      always_reduce=True)
    sync.begin_step(1)
    xm = x.cuda().requires_grad_(True)
    model(xm).backward(dy.cuda())
    assert len(sync.works) == len(sync.buckets) > 1  # every bucket's collective launched
    sync.finish()
    torch.cuda.synchronize()
    for (_, _, a), (_, _, b) in zip(ref.linears(), model.linears()):
        assert torch.equal(a.A.grad.float(), b.sink.dA.to(torch.bfloat16).float())
        assert torch.equal(a.B.grad.float(), b.sink.dB.to(torch.bfloat16).float())
    assert torch.equal(xr.grad, xm.grad)
