"""The fused data-parallel exchange (include/runlora.h
runlora_backward_exchange): the adapter gradients' token-split slabs are reduced in fixed
order and summed across ranks by the dX GEMM launch's idle warps over peer memory.

dA and dB are sums over tokens (Eq. 3): the sum over ranks of the ranks'
partial sums is the full-batch gradient.

1. P in {1, 2, 4, 8} ranks EMULATED on one GPU: one cooperative launch runs every rank's
   exchange code (the profiling guide: never several ranks' waiting kernels as separate
   launches on one GPU).  Every rank's dA, dB must equal, bit for bit, the rank-order sum of
   the ranks' split-order slab sums (computed here with the same fp32 additions), on every
   rank alike, for consecutive epochs (alternating buffer halves, reused flags).
2. P = 1 through the real entry point: runlora_backward_exchange equals runlora_backward bit
   for bit (dX, dA, dB), for every executable variant.
"""
import ctypes as C

import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    return runlora


def _emulate(rl, h, P, k, m, r, splits, sA, sB, epoch, bufs, flags):
    f = rl._lib.runlora_debug_exchange_emulate
    f.restype = C.c_int
    V = C.c_void_p
    f.argtypes = [V, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.POINTER(V), C.POINTER(V), C.POINTER(V),
                  C.POINTER(V), C.POINTER(V), C.POINTER(V), C.c_uint32]
    arr = lambda ts: (V * P)(*[t.data_ptr() for t in ts])
    dA = [torch.full((k, r), float("nan"), device="cuda") for _ in range(P)]
    dB = [torch.full((r, m), float("nan"), device="cuda") for _ in range(P)]
    st = f(h._h, P, k, m, r, splits, arr(sA), arr(sB), arr(dA), arr(dB), arr(bufs), arr(flags), epoch)
    assert st == 0, rl._lib.runlora_last_error()
    return dA, dB


def test_emulated_exchange_long_run(rl):
    """200 consecutive epochs of the 8-rank emulated exchange on the same buffers (alternating
    halves, reused flags): every epoch bit-identical to the first — a flag or buffer-half race
    would show up as a changed bit or a hang (bounded by the pytest timeout)."""
    P, k, m, r, splits = 8, 520, 392, 16, 3
    h = rl.handle(0)
    buf_bytes, flag_bytes = rl.exchange_sizes(k, m, r, P)
    bufs = [torch.zeros(buf_bytes // 4, device="cuda") for _ in range(P)]
    flags = [torch.zeros(flag_bytes // 4, dtype=torch.int32, device="cuda") for _ in range(P)]
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    sA = [torch.randn(splits, k, r, device="cuda", generator=g) for _ in range(P)]
    sB = [torch.randn(splits, m, r, device="cuda", generator=g) for _ in range(P)]
    ref = None
    for epoch in range(1, 201):
        dA, dB = _emulate(rl, h, P, k, m, r, splits, sA, sB, epoch, bufs, flags)
        if ref is None:
            ref = (dA[0].clone(), dB[0].clone())
        for q in range(P):
            assert torch.equal(dA[q], ref[0]) and torch.equal(dB[q], ref[1]), (epoch, q)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_emulated_exchange_bit_exact(rl, P):
    k, m, r, splits = 520, 392, 16, 3
    h = rl.handle(0)
    buf_bytes, flag_bytes = rl.exchange_sizes(k, m, r, P)
    bufs = [torch.zeros(buf_bytes // 4, device="cuda") for _ in range(P)]
    flags = [torch.zeros(flag_bytes // 4, dtype=torch.int32, device="cuda") for _ in range(P)]
    g = torch.Generator(device="cuda")
    for epoch in (1, 2, 3):
        g.manual_seed(100 * P + epoch)
        sA = [torch.randn(splits, k, r, device="cuda", generator=g) for _ in range(P)]
        sB = [torch.randn(splits, m, r, device="cuda", generator=g) for _ in range(P)]
        dA, dB = _emulate(rl, h, P, k, m, r, splits, sA, sB, epoch, bufs, flags)
        # the same fp32 additions: split order within a rank, then rank order
        loc = [(s[0].clone(), t[0].clone()) for s, t in zip(sA, sB)]
        for q in range(P):
            for sp in range(1, splits):
                loc[q][0].add_(sA[q][sp])
                loc[q][1].add_(sB[q][sp])
        wA, wB = loc[0][0].clone(), loc[0][1].clone()
        for q in range(1, P):
            wA.add_(loc[q][0])
            wB.add_(loc[q][1])
        for q in range(P):
            assert torch.equal(dA[q], wA), (P, epoch, q)
            assert torch.equal(dB[q], wB.t()), (P, epoch, q)
        # and against the fp64 sum of everything (the reduction is a plain sum, Eq. 3)
        fA = sum(s.double().sum(0) for s in sA)
        assert O.rel_fro(dA[0].double().cpu().numpy(), fA.cpu().numpy()) < 1e-6


CASES = [synth.case("xchg_zsplit", 0, 60, 1024, 1024, 768, 16, "bf16"),   # K-split Z blocks, folded slabs
         synth.case("xchg_plain", 0, 61, 2048, 512, 640, 64, "bf16")]     # plain token-split slabs


@pytest.mark.parametrize("c", CASES, ids=lambda c: c.name)
def test_backward_exchange_p1_equals_backward(rl, c):
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    buf_bytes, flag_bytes = rl.exchange_sizes(c.k, c.m, c.r, 1)
    buf = torch.zeros(buf_bytes // 4, device="cuda")
    flags = torch.zeros(flag_bytes // 4, dtype=torch.int32, device="cuda")
    x = h.exchange_create(1, 0, c.k, c.m, c.r, [buf.data_ptr()], [flags.data_ptr()])
    try:
        epoch = 0
        for bwd in (1, 2, 3, 4, 5):
            ref = [torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda"), torch.empty(c.k, c.r, device="cuda"),
                   torch.empty(c.r, c.m, device="cuda")]
            h.backward(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], ref[0], ref[1], ref[2])
            for _ in range(2):  # two epochs: both buffer halves
                epoch += 1
                got = [torch.full_like(t, float("nan")) for t in ref]
                h.backward_exchange(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], got[0], got[1], got[2], x,
                                    epoch)
                torch.cuda.synchronize()
                for a, b in zip(ref, got):
                    assert torch.equal(a, b), (c.name, bwd, epoch)
    finally:
        rl.exchange_destroy(x)


def test_backward_exchange_errors(rl):
    c = CASES[0]
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    buf_bytes, flag_bytes = rl.exchange_sizes(c.k, c.m, c.r, 1)
    buf = torch.zeros(buf_bytes // 4, device="cuda")
    flags = torch.zeros(flag_bytes // 4, dtype=torch.int32, device="cuda")
    x = h.exchange_create(1, 0, c.k, c.m, c.r, [buf.data_ptr()], [flags.data_ptr()])
    dX = torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda")
    dA, dB = torch.empty(c.k, c.r, device="cuda"), torch.empty(c.r, c.m, device="cuda")
    try:
        with pytest.raises(rl.RunLoRAError) as e:
            h.backward_exchange(1, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB, x, 0)
        assert e.value.status == 1  # epochs start at 1
        with pytest.raises(rl.RunLoRAError) as e:
            h.backward_exchange(1, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], None, dA, dB, x, 1)
        assert e.value.status == 1  # the exchange rides on the dX GEMM
        other = rl.make_shape(c.n, c.k, c.m + 8, c.r, rl.BF16)
        with pytest.raises(rl.RunLoRAError) as e:
            h.backward_exchange(1, other, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB, x, 1)
        assert e.value.status in (1, 2)
    finally:
        rl.exchange_destroy(x)


_CHILD = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, {root!r})
import synth
from paper_2312_03415_b200 import runlora as rl, dp
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29562", RANK="0", WORLD_SIZE="1")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
h = rl.handle(0)
c = synth.case("xchg_symm", 0, 62, 1024, 1024, 768, 16, "bf16")
d = {{k: v.cuda() for k, v in synth.operands(c).items()}}
shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
out = []
for multicast in (False, True):
    fx = dp.FusedExchange(c.k, c.r, c.m, dev, h, multicast=multicast)
    if multicast and not fx.multicast:
        print("multicast unavailable")
        continue
    for bwd in (1, 5):
        ref = [torch.empty(c.n, c.k, dtype=torch.bfloat16, device=dev), torch.empty(c.k, c.r, device=dev),
               torch.empty(c.r, c.m, device=dev)]
        h.backward(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], *ref)
        for _ in range(3):
            got = [torch.full_like(t, float("nan")) for t in ref]
            fx.backward(bwd, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], *got)
            torch.cuda.synchronize()
            for a, b in zip(ref, got):
                assert torch.equal(a, b), (multicast, bwd)
    print("ok multicast" if multicast else "ok peer")
    fx.close()
dist.destroy_process_group()
"""


def test_fused_exchange_symmetric_memory_p1(tmp_path):
    """dp.FusedExchange over torch symmetric memory in a 1-rank group: the full path
    (rendezvous, descriptor, backward_exchange) equals the plain backward bit for bit; the
    multicast (NVLS) read is exercised when the handle reports a multicast address."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "child.py"
    script.write_text(_CHILD.format(root=root))
    p = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "ok peer" in p.stdout, (p.stdout[-2000:], p.stderr[-3000:])
    print(p.stdout)
