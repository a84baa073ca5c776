"""One-shot fixed-order allreduce of the packed adapter gradients (runlora_allreduce_sum_f32;
SURVEY §8(a) a8, §8(f) NEXT-2).

This box has one GPU, so P ranks are emulated as P buffers on it and ONE launch sums them
(the profiling guide's advice: never run ranks that wait on one another as separate
launches on one GPU).  Each element is the fp32 sum in rank order 0..P-1, so the expected
value is the same left-to-right fp32 sum done by torch: bit-exact.  The symmetric-memory
transport (dp.SymmetricAllreduce: rendezvous, peer pointers, the two barriers) runs end to
end at P = 1 in a subprocess."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    return runlora


@pytest.mark.parametrize("P", [1, 2, 3, 8, 16])
@pytest.mark.parametrize("n", [1, 7, 4096 + 3, 1 << 20, (4096 + 4096) * 16])
def test_fixed_order_sum_bit_exact(rl, P, n):
    h = rl.handle(0)
    g = torch.Generator(device="cuda").manual_seed(1000 * P + n % 997)
    bufs = [torch.randn(n, device="cuda", generator=g) * (10.0 ** (q % 5 - 2)) for q in range(P)]
    out = torch.full((n,), float("nan"), device="cuda")
    h.allreduce_sum_f32([b.data_ptr() for b in bufs], out)
    torch.cuda.synchronize()
    want = bufs[0].clone()
    for b in bufs[1:]:
        want += b
    assert torch.equal(out, want)


def test_zero_length_and_errors(rl):
    h = rl.handle(0)
    a = torch.ones(64, device="cuda")
    out = torch.zeros(64, device="cuda")
    h.allreduce_sum_f32([a.data_ptr()], out, n=0)  # no-op
    torch.cuda.synchronize()
    assert torch.equal(out, torch.zeros(64, device="cuda"))
    for ptrs, o, st in (([], out, 1),                                  # P = 0
                        ([a.data_ptr()] * 17, out, 1),                 # P > 16
                        ([a.data_ptr(), out.data_ptr()], out, 1),      # out aliases a peer
                        ([a.data_ptr() + 4], out, 6)):                 # misaligned peer
        with pytest.raises(rl.RunLoRAError) as e:
            h.allreduce_sum_f32(ptrs, o, n=16)
        assert e.value.status == st


_CHILD = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, {root!r})
from paper_2312_03415_b200 import runlora as rl, dp
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29561", RANK="0", WORLD_SIZE="1")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
h = rl.handle(0)
k, r, m = 1000, 16, 776
sy = dp.SymmetricAllreduce(k, r, m, dev, h)
comm = torch.cuda.Stream(dev)
for step in range(3):
    src = torch.randn(k * r + r * m, device=dev)
    work = dp.overlapped_backward(lambda: sy.grads.flat.copy_(src), lambda: None, sy.grads, comm_stream=comm,
                                  exchange=sy)
    work.wait()
    torch.cuda.synchronize()
    assert torch.equal(sy.result.flat, src), step
    assert sy.result.dA.shape == (k, r) and sy.result.dB.shape == (r, m)
dist.destroy_process_group()
print("ok")
"""


def test_symmetric_memory_transport_p1(tmp_path):
    script = tmp_path / "child.py"
    script.write_text(_CHILD.format(root=ROOT))
    p = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "ok" in p.stdout, (p.stdout[-2000:], p.stderr[-3000:])
