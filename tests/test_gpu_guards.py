"""Memory safety without compute-sanitizer (closed on this GPU pool, profiles/r02/sanitizer.md):
every buffer the library writes is embedded in a larger allocation whose guard regions carry a
byte pattern; after every variant, the split backward, the quantized-W entry points and the
fused exchange, the guards must be untouched — on ragged shapes (tails in every dimension)
and on a K-split shape (repeated A/B side jobs, folded slabs, side-job reduction, split fix-up)."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
G = 1 << 16  # guard bytes on each side
PAT = 0xA5


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    return runlora


class Guarded:
    def __init__(self, nbytes):
        self.buf = torch.full((nbytes + 2 * G,), PAT, dtype=torch.uint8, device="cuda")
        self.nbytes = nbytes

    def view(self, shape, dtype):
        return self.buf[G:G + self.nbytes].view(dtype).view(*shape)

    def intact(self):
        return bool((self.buf[:G] == PAT).all()) and bool((self.buf[G + self.nbytes:] == PAT).all())


def _outputs(c):
    g = {"Y": Guarded(c.n * c.m * 2), "dX": Guarded(c.n * c.k * 2), "dA": Guarded(c.k * c.r * 4),
         "dB": Guarded(c.r * c.m * 4)}
    t = {"Y": g["Y"].view((c.n, c.m), torch.bfloat16), "dX": g["dX"].view((c.n, c.k), torch.bfloat16),
         "dA": g["dA"].view((c.k, c.r), torch.float32), "dB": g["dB"].view((c.r, c.m), torch.float32)}
    return g, t


CASES = [synth.case("guard_ragged", 0, 70, 1000, 1032, 1552, 8, "bf16"),   # non-K-split, ragged tiles
         synth.case("guard_zsplit", 0, 71, 1024, 512, 512, 16, "bf16"),     # K-split Z blocks (sz = 4)
         synth.case("guard_r72", 0, 72, 777, 264, 392, 72, "bf16")]         # r beyond a 64-wide tile


@pytest.mark.parametrize("c", CASES, ids=lambda c: c.name)
def test_guards_all_variants(rl, c):
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    wsg = Guarded(rl.workspace_size_wq(shape))
    ws = wsg.view((rl.workspace_size_wq(shape),), torch.uint8)
    g, t = _outputs(c)
    for f in (1, 2):
        h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], t["Y"], ws=ws)
    for b in (1, 2, 3, 4, 5):
        h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], t["dX"], t["dA"], t["dB"], ws=ws)
        h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], None, t["dA"], t["dB"], accumulate=True, ws=ws)
        h.backward_params(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], t["dA"], t["dB"], ws=ws)
        h.backward_input(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], t["dX"], ws=ws)
    if c.m % 16 == 0:
        qw = h.quantize_w(d["W"])
        for f in (1, 2):
            h.forward_wq(f, shape, d["X"], qw, d["A"], d["B"], t["Y"], ws=ws)
        for b in (1, 4, 5):
            h.backward_wq(b, shape, d["X"], qw, d["A"], d["B"], d["dY"], t["dX"], t["dA"], t["dB"], ws=ws)
    torch.cuda.synchronize()
    assert wsg.intact(), "workspace guards"
    for k, gg in g.items():
        assert gg.intact(), k
    # bf16 adapter gradients (2-byte outputs of the reductions)
    gA, gB = Guarded(c.k * c.r * 2), Guarded(c.r * c.m * 2)
    for b in (1, 5):
        h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], t["dX"], gA.view((c.k, c.r), torch.bfloat16),
                   gB.view((c.r, c.m), torch.bfloat16), ws=ws)
    torch.cuda.synchronize()
    assert gA.intact() and gB.intact()


def test_guards_fused_exchange(rl):
    c = CASES[1]
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    bb, fb = rl.exchange_sizes(c.k, c.m, c.r, 1)
    bufg, flg = Guarded(bb), Guarded(fb)
    buf, fl = bufg.view((bb // 4,), torch.float32), flg.view((fb // 4,), torch.int32)
    buf.zero_()
    fl.zero_()
    x = h.exchange_create(1, 0, c.k, c.m, c.r, [buf.data_ptr()], [fl.data_ptr()])
    try:
        g, t = _outputs(c)
        for e in (1, 2, 3):
            for b in (1, 5):
                h.backward_exchange(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], t["dX"], t["dA"], t["dB"], x,
                                    2 * e - (b == 1))
        torch.cuda.synchronize()
        assert bufg.intact() and flg.intact()
        for k in ("dX", "dA", "dB"):
            assert g[k].intact(), k
    finally:
        rl.exchange_destroy(x)


@pytest.mark.parametrize("c", CASES[:2], ids=lambda c: c.name)
def test_guards_forward2_halves(rl, c):
    """runlora_wprime_t / _wq write exactly the m x k W'ᵀ; runlora_forward_wprime exactly Y."""
    d = {k: v.cuda() for k, v in synth.operands(c).items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    wg = Guarded(c.m * c.k * 2)
    Wpt = wg.view((c.m, c.k), torch.bfloat16)
    g, t = _outputs(c)
    h.wprime_t(shape, d["W"], d["A"], d["B"], Wpt)
    h.forward_wprime(shape, d["X"], Wpt, t["Y"])
    if c.m % 16 == 0:
        h.wprime_t(shape, h.quantize_w(d["W"]), d["A"], d["B"], Wpt)
        h.forward_wprime(shape, d["X"], Wpt, t["Y"])
    torch.cuda.synchronize()
    assert wg.intact() and g["Y"].intact()
