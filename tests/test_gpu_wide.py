"""512-wide main-GEMM tiles: the planner's split and parity of every
executable variant on shapes where it mixes 512- and 256-wide tiles, with ragged rows,
a ragged last column tile of one MMA half (N = 3304: 232 columns) and of two halves
(N = 3512: 440 columns), and the concat-K tail of dX — against the fp64 oracle
(relative Frobenius <= 2e-2 per tensor, healthy < 5e-3)."""
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


def _rows(rl, h, M, N, K, b_mn=0):
    f = rl._lib.runlora_debug_wide_rows
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
    return f(h._h, M, N, K, b_mn)


def _np(t):
    return t.detach().to(torch.float64).cpu().numpy()


def test_planner_split(rl):
    h = rl.handle(0)
    # Y GEMM of case W1 (M = n, N = m, K = k): wide rows then narrow rows (ragged M)
    r = _rows(rl, h, 3000, 3304, 2048)
    assert 0 < r < 3000 and r % 256 == 0
    # C2: most rows wide (measured planner choice 6912 of 8192)
    r = _rows(rl, h, 8192, 4096, 4096)
    assert 4096 <= r < 8192 and r % 256 == 0
    # MN-major B (forward1's Y GEMM) and single-round shapes stay 256-wide
    assert _rows(rl, h, 8192, 4096, 4096, b_mn=1) == 0
    assert _rows(rl, h, 512, 512, 512) == 0
    # short K: with the tile held in registers the wide tiles pay even at 13 k-blocks; the
    # planner mixes them with 256-wide rows (measured 31.7 µs mixed vs 33.8 either pure,
    # DESIGN.md §5)
    r = _rows(rl, h, 4096, 3000, 776)
    assert 0 < r < 4096 and r % 256 == 0


CASES = [synth.case("wide_w1", 0, 40, 3000, 2048, 3304, 16, "bf16"),
         synth.case("wide_w2", 0, 41, 2600, 3512, 2048, 8, "bf16")]


@pytest.mark.parametrize("c", CASES, ids=lambda c: c.name)
def test_wide_all_variants_match_oracle(rl, c):
    h = rl.handle(0)
    # both main GEMMs of the case take the wide path
    assert _rows(rl, h, c.n, c.m, c.k) > 0 and _rows(rl, h, c.n, c.k, c.m + c.r) > 0
    ops = synth.operands(c)
    d = {k: v.cuda() for k, v in ops.items()}
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    X, W, A, B, dY = (_np(ops[k]) for k in ("X", "W", "A", "B", "dY"))
    wY = O.forward(1, X, W, A, B)
    wA, wB, wX = O.reference_backward(X, W, A, B, dY)
    errs = {}
    for f in (1, 2):
        Y = torch.full((c.n, c.m), float("nan"), dtype=torch.bfloat16, device="cuda")
        h.forward(f, shape, d["X"], d["W"], d["A"], d["B"], Y)
        torch.cuda.synchronize()
        errs[f"F{f}"] = O.rel_fro(_np(Y), wY)
    for b in (1, 2, 3, 4, 5):
        dX = torch.full((c.n, c.k), float("nan"), dtype=torch.bfloat16, device="cuda")
        dA = torch.full((c.k, c.r), float("nan"), device="cuda")
        dB = torch.full((c.r, c.m), float("nan"), device="cuda")
        h.backward(b, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB)
        torch.cuda.synchronize()
        errs[f"B{b}"] = max(O.rel_fro(_np(dA), wA), O.rel_fro(_np(dB), wB), O.rel_fro(_np(dX), wX))
    assert all(e <= 2e-2 for e in errs.values()), errs
    assert max(errs.values()) < 5e-3, errs


_CHILD = r"""
import sys, torch
sys.path.insert(0, {root!r})
import synth
from paper_2312_03415_b200 import runlora as rl
c = synth.case("wide_w1", 0, 40, 3000, 2048, 3304, 16, "bf16")
d = {{k: v.cuda() for k, v in synth.operands(c).items()}}
h = rl.handle(0)
shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
Y = torch.empty(c.n, c.m, dtype=torch.bfloat16, device="cuda")
dX = torch.empty(c.n, c.k, dtype=torch.bfloat16, device="cuda")
dA = torch.empty(c.k, c.r, device="cuda"); dB = torch.empty(c.r, c.m, device="cuda")
h.forward(2, shape, d["X"], d["W"], d["A"], d["B"], Y)
h.backward(1, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB)
torch.save({{"Y": Y.cpu(), "dX": dX.cpu(), "dA": dA.cpu(), "dB": dB.cpu()}}, sys.argv[1])
"""


def test_wide_reduced_stages_bit_exact(tmp_path):
    """RUNLORA_MAIN_STAGES < 7 (set by bench.py under data parallelism) applies to the dX GEMM
    only — the one the adapter-gradient allreduce overlaps: its 512-wide launch runs on 3 of
    the 4 ring stages (48 KB less shared memory, RUNLORA_DEBUG_LAUNCH), the Y GEMM keeps the
    full ring, and the arithmetic is unchanged, so every output is bit-identical."""
    import os
    import re
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "child.py"
    script.write_text(_CHILD.format(root=root))
    outs, smem = [], []
    for st in ("", "6"):
        env = dict(os.environ)
        env.pop("RUNLORA_MAIN_STAGES", None)
        env["RUNLORA_DEBUG_LAUNCH"] = "1"
        if st:
            env["RUNLORA_MAIN_STAGES"] = st
        f = tmp_path / f"out{st or 'default'}.pt"
        p = subprocess.run([sys.executable, str(script), str(f)], env=env, capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(torch.load(f))
        # the two 512-wide main-GEMM launches of the child, in order: Y (forward), dX (backward)
        wide = [int(m.group(1)) for m in re.finditer(r"tc_gemm<512,2,[^>]*> grid \d+ smem (\d+)", p.stderr)]
        assert len(wide) == 2, p.stderr[-2000:]
        smem.append(wide)
    assert smem[0][0] == smem[0][1]                      # default: both on the full ring
    assert smem[1][0] == smem[0][0]                      # reduced: the Y GEMM keeps it
    assert smem[0][1] - smem[1][1] == 48 * 1024          # the dX GEMM drops one 48 KB stage
    for k in ("Y", "dX", "dA", "dB"):
        assert torch.equal(outs[0][k], outs[1][k]), k


def test_wide_outputs_stay_in_bounds(rl):
    """Y and dX live inside larger buffers filled with a sentinel: the wide/narrow launches
    (ragged rows and a ragged last column tile) must not write outside [0, n·m)."""
    c = CASES[0]
    ops = synth.operands(c)
    d = {k: v.cuda() for k, v in ops.items()}
    h = rl.handle(0)
    shape = rl.make_shape(c.n, c.k, c.m, c.r, rl.BF16)
    pad = 4096
    sentinel = torch.tensor(-12345.0, dtype=torch.bfloat16)
    ybuf = torch.full((c.n * c.m + 2 * pad,), sentinel.item(), dtype=torch.bfloat16, device="cuda")
    xbuf = torch.full((c.n * c.k + 2 * pad,), sentinel.item(), dtype=torch.bfloat16, device="cuda")
    Y = ybuf[pad:pad + c.n * c.m].view(c.n, c.m)
    dX = xbuf[pad:pad + c.n * c.k].view(c.n, c.k)
    dA = torch.empty(c.k, c.r, device="cuda")
    dB = torch.empty(c.r, c.m, device="cuda")
    h.forward(2, shape, d["X"], d["W"], d["A"], d["B"], Y)
    h.backward(1, shape, d["X"], d["W"], d["A"], d["B"], d["dY"], dX, dA, dB)
    torch.cuda.synchronize()
    for buf, n_in in ((ybuf, c.n * c.m), (xbuf, c.n * c.k)):
        assert bool((buf[:pad] == sentinel.item()).all()) and bool((buf[pad + n_in:] == sentinel.item()).all())
        assert not bool((buf[pad:pad + n_in] == sentinel.item()).any())  # every element written


def test_comm_sms_leave_sms_free_for_the_collective(tmp_path):
    """RUNLORA_COMM_SMS = 2 (bench.py sets it under NCCL data parallelism): the dX GEMM — the
    launch the adapter-gradient allreduce overlaps — runs its persistent grid on 146 of the
    148 SMs (the 512/256-wide split re-planned for 73 pairs), the Y GEMM keeps all of them,
    and the outputs stay parity-green (tile order changes the K direction of some tiles,
    so they are not bit-identical)."""
    import os
    import re
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "child.py"
    # enough units that the persistent grid is bounded by the SMs (C4 per-rank size at P = 4)
    script.write_text(_CHILD.format(root=root).replace('synth.case("wide_w1", 0, 40, 3000, 2048, 3304, 16, "bf16")',
                                                      'synth.case("comm", 0, 42, 8192, 2048, 2048, 16, "bf16")'))
    outs, grids = [], []
    for cs in ("", "2"):
        env = dict(os.environ)
        env.pop("RUNLORA_COMM_SMS", None)
        env.pop("RUNLORA_MAIN_STAGES", None)
        env["RUNLORA_DEBUG_LAUNCH"] = "1"
        if cs:
            env["RUNLORA_COMM_SMS"] = cs
        f = tmp_path / f"out{cs or 'default'}.pt"
        p = subprocess.run([sys.executable, str(script), str(f)], env=env, capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(torch.load(f))
        grids.append([int(m.group(1)) for m in re.finditer(r"tc_gemm<512,2,[^>]*> grid (\d+)", p.stderr)])
    assert grids[0] == [148, 148] and grids[1] == [148, 146], grids
    for k in ("Y", "dA", "dB"):
        assert torch.equal(outs[0][k], outs[1][k]), k  # the Y GEMM and the adapter gradients are untouched
    d = (outs[0]["dX"].double() - outs[1]["dX"].double()).norm() / outs[0]["dX"].double().norm()
    assert d < 1e-3, d
