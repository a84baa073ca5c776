"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports every
symbol include/*.h declares, and its Table 1 cost model / FLOP selector / Eq. 5
predicate agree with the oracle exactly."""
import ctypes as C
import os
import random
import re

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rl():
    from paper_2312_03415_b200 import runlora
    return runlora


def _declared():
    names = set()
    for h in ("runlora.h", "runlora_testing.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names.update(re.findall(r"\b(runlora_[a-z_]+)\s*\(", src))
    return sorted(names)


def test_library_exports_every_declared_symbol(rl):
    lib = C.CDLL(rl.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert len(_declared()) >= 18
    assert "sm_100a" in rl.version()


def test_flops_match_table1(rl):
    rnd = random.Random(3)
    shapes = [(256, 256, 256, 8), (200, 512, 512, 32), (8192, 4096, 11008, 16), (1, 1, 1, 1)]
    shapes += [(rnd.randint(1, 1 << 17), rnd.randint(1, 1 << 14), rnd.randint(1, 1 << 14), rnd.randint(1, 512))
               for _ in range(300)]
    for n, k, m, r in shapes:
        s = rl.make_shape(n, k, m, r, rl.BF16)
        for v in (1, 2):
            assert rl.flops(s, False, v) == O.flops_forward(v, n, k, m, r)
        for v in range(1, 9):
            assert rl.flops(s, True, v) == O.flops_backward(v, n, k, m, r)
        assert rl.param_reduction(s) == O.param_reduction(k, m, r)


def test_flops_overflow_and_bad_variant(rl):
    s = rl.make_shape(1 << 30, 1 << 30, 1 << 30, 1 << 20, rl.BF16)
    with pytest.raises(rl.RunLoRAError) as e:
        rl.flops(s, True, 6)
    assert e.value.status == 5
    s = rl.make_shape(8, 8, 8, 8)
    with pytest.raises(rl.RunLoRAError) as e:
        rl.flops(s, False, 3)
    assert e.value.status == 1
    with pytest.raises(rl.RunLoRAError):
        rl.flops(rl.make_shape(0, 8, 8, 8), False, 1)


def test_select_by_flops_matches_oracle(rl):
    rnd = random.Random(9)
    for _ in range(2000):
        n, k, m = rnd.randint(1, 1 << 16), rnd.randint(1, 1 << 13), rnd.randint(1, 1 << 13)
        r = rnd.randint(1, 256)
        p = rl.select_by_flops(rl.make_shape(n, k, m, r, rl.F32))
        assert (p.fwd, p.bwd) == O.select_by_flops(n, k, m, r), (n, k, m, r)
        assert (p.flops_fwd_pick, p.flops_bwd_pick) == (p.fwd, p.bwd)
        assert bool(p.param_reduction) == O.param_reduction(k, m, r)
    # SPEC worked selections
    assert (rl.select_by_flops(rl.make_shape(200, 512, 512, 32)).fwd,
            rl.select_by_flops(rl.make_shape(200, 512, 512, 32)).bwd) == (1, 1)
    assert rl.select_by_flops(rl.make_shape(20480, 512, 512, 32)).fwd == 2


def test_workspace_size_and_validation(rl):
    s = rl.make_shape(8192, 4096, 4096, 16, rl.BF16)
    ws = rl.workspace_size(s, 2, 5)
    assert ws >= 4096 * 4096 * 2 + 2 * 8192 * 16 * 2  # W' plus Z1, Z2
    with pytest.raises(rl.RunLoRAError) as e:
        rl.workspace_size(rl.make_shape(100, 4100, 4096, 16, rl.BF16), 1, 1)
    assert e.value.status == 6  # bf16 needs k, m, r multiples of 8 (TMA strides)
    with pytest.raises(rl.RunLoRAError) as e:
        rl.workspace_size(s, 1, 7)
    assert e.value.status == 4  # backward7 is cost-model only
    # fp32 shapes need no alignment
    assert rl.workspace_size(rl.make_shape(333, 200, 150, 5, rl.F32), 1, 1) > 0


def test_status_strings(rl):
    for st in range(11):
        assert rl._lib.runlora_status_string(st)


def test_null_handle_is_invalid_arg(rl):
    """Every entry point that takes a handle returns RUNLORA_ERR_INVALID_ARG for NULL before
    touching anything (include/runlora.h "Errors"); no launch, no dereference."""
    lib = rl._lib
    s = rl.make_shape(256, 256, 256, 8, rl.BF16)
    p = C.c_void_p(4096)  # never dereferenced: the handle check comes first
    S = C.byref(s)
    assert lib.runlora_forward(None, 1, S, p, p, p, p, p, p, 1 << 20, None) == 1
    assert lib.runlora_backward(None, 1, S, p, p, p, p, p, p, p, p, 0, 0, p, 1 << 20, None) == 1
    assert lib.runlora_backward_params(None, 1, S, p, p, p, p, p, p, p, 0, 0, p, 1 << 20, None) == 1
    assert lib.runlora_backward_input(None, 1, S, p, p, p, p, p, p, p, 1 << 20, None) == 1
    st = rl.HostStep(1, 1, 0, 0, *([4096] * 15))
    assert lib.runlora_step_host(None, S, C.byref(st), p, 1 << 20, None) == 1
    assert lib.runlora_select(None, S, rl.BY_TIME, None, p, 1 << 20, None, C.byref(rl.Plan())) == 1
    assert lib.runlora_profile_enable(None, 1) == 1
    assert lib.runlora_wprime_t(None, S, p, p, p, p, None) == 1
    assert lib.runlora_wprime_t_wq(None, S, p, p, p, p, p, p, None) == 1
    assert lib.runlora_forward_wprime(None, S, p, p, p, p, 1 << 20, None) == 1
    assert "handle" in lib.runlora_last_error().decode()


def test_host_step_struct_matches_header(rl):
    """ABI version 2: runlora_host_step_t ends with the exchange hook (function pointer + user)."""
    src = open(os.path.join(ROOT, "include", "runlora.h")).read()
    assert "#define RUNLORA_ABI_VERSION 2" in src
    assert [f[0] for f in rl.HostStep._fields_][-2:] == ["exchange", "exchange_user"]
    assert C.sizeof(rl.HostStep) == 4 * 4 + 15 * 8 + 2 * 8


def test_exchange_sizes_and_null_handle(rl):
    """Fused exchange geometry (include/runlora.h): two epoch halves of r(k+m) fp32 (rounded up
    to 64 floats) per rank, one flag per 64-row chunk and rank; argument checks before any
    device work."""
    buf, flags = rl.exchange_sizes(4096, 4096, 16, 8)
    assert buf == 2 * 16 * 8192 * 4 and flags == (8192 // 64) * 8 * 4
    buf, flags = rl.exchange_sizes(1000, 24, 8, 3)
    assert buf == 2 * ((1024 * 8 + 63) // 64 * 64) * 4 and flags == 16 * 3 * 4
    for bad in [(0, 8, 8, 1), (8, 8, 6, 1), (8, 8, 8, 0), (8, 8, 8, 17)]:
        with pytest.raises(rl.RunLoRAError) as e:
            rl.exchange_sizes(*bad)
        assert e.value.status == 1
    x = C.c_void_p()
    arr = (C.c_void_p * 1)(4096)
    assert rl._lib.runlora_exchange_create(None, 1, 0, 8, 8, 8, arr, arr, None, C.byref(x)) == 1
    s = rl.make_shape(256, 256, 256, 8, rl.BF16)
    p = C.c_void_p(4096)
    assert rl._lib.runlora_backward_exchange(None, 1, C.byref(s), p, p, p, p, p, p, p, p, 0, 0, p, 1, p, 1 << 20,
                                             None) == 1
