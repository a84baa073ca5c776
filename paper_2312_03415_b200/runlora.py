"""Thin ctypes binding of librunlora.so (include/runlora.h).

Argument marshalling only: every step of the LoRA forward/backward runs in the
library's sm_100a kernels.  PyTorch supplies device memory (``data_ptr()``) and
streams.  If the shared library is missing the import of this module fails
loudly — there is no CPU or eager-PyTorch fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# the in-tree build; RUNLORA_LIB overrides it (e.g. tools/ab_lib.py loads two builds side by side)
LIB_PATH = os.environ.get("RUNLORA_LIB") or os.path.join(_PKG, "lib", "librunlora.so")

F32, BF16 = 0, 1
BY_FLOPS, BY_TIME, HYBRID = 0, 1, 2
STATUS = {0: "ok", 1: "invalid argument", 2: "shape mismatch", 3: "unsupported dtype", 4: "unsupported variant",
          5: "FLOP overflow", 6: "alignment", 7: "workspace too small", 8: "CUDA error", 9: "timing failure",
          10: "unsupported device"}

_DT = {torch.float32: F32, torch.bfloat16: BF16}
_TORCH = {F32: torch.float32, BF16: torch.bfloat16}


class Shape(C.Structure):
    _fields_ = [("n", C.c_int64), ("k", C.c_int64), ("m", C.c_int64), ("r", C.c_int64), ("dtype", C.c_int32)]


class Plan(C.Structure):
    _fields_ = [("fwd", C.c_int32), ("bwd", C.c_int32), ("criterion", C.c_int32), ("param_reduction", C.c_int32),
                ("flops_fwd", C.c_uint64 * 3), ("flops_bwd", C.c_uint64 * 9),
                ("time_fwd_us", C.c_float * 3), ("time_bwd_us", C.c_float * 9),
                ("flops_fwd_pick", C.c_int32), ("flops_bwd_pick", C.c_int32)]

    def as_dict(self):
        nan_to_none = lambda x: None if math.isnan(x) else float(x)
        return {"fwd": self.fwd, "bwd": self.bwd, "criterion": self.criterion,
                "param_reduction": bool(self.param_reduction),
                "flops_fwd": {v: int(self.flops_fwd[v]) for v in (1, 2)},
                "flops_bwd": {v: int(self.flops_bwd[v]) for v in range(1, 9)},
                "time_fwd_us": {v: nan_to_none(self.time_fwd_us[v]) for v in (1, 2)},
                "time_bwd_us": {v: nan_to_none(self.time_bwd_us[v]) for v in range(1, 6)},
                "flops_pick": (self.flops_fwd_pick, self.flops_bwd_pick)}


class Operands(C.Structure):
    _fields_ = [("X", C.c_void_p), ("W", C.c_void_p), ("A", C.c_void_p), ("B", C.c_void_p), ("dY", C.c_void_p),
                ("Y", C.c_void_p), ("dX", C.c_void_p), ("dA", C.c_void_p), ("dB", C.c_void_p),
                ("grad_dtype", C.c_int32)]


EXCHANGE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)  # runlora_exchange_fn(user, stream)


class HostStep(C.Structure):
    _fields_ = [("fwd", C.c_int32), ("bwd", C.c_int32), ("grad_dtype", C.c_int32), ("accumulate", C.c_int32),
                ("X_host", C.c_void_p), ("dY_host", C.c_void_p), ("Y_host", C.c_void_p), ("dX_host", C.c_void_p),
                ("dA_host", C.c_void_p), ("dB_host", C.c_void_p),
                ("W", C.c_void_p), ("A", C.c_void_p), ("B", C.c_void_p),
                ("X", C.c_void_p), ("dY", C.c_void_p), ("Y", C.c_void_p), ("dX", C.c_void_p),
                ("dA", C.c_void_p), ("dB", C.c_void_p), ("exchange", EXCHANGE_FN), ("exchange_user", C.c_void_p)]


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_uint64), ("total_ms", C.c_double)]


EXPORTS = ["runlora_version", "runlora_create", "runlora_destroy", "runlora_flops", "runlora_param_reduction",
           "runlora_workspace_size", "runlora_select", "runlora_forward", "runlora_backward",
           "runlora_backward_params", "runlora_backward_input", "runlora_step_host", "runlora_profile_enable",
           "runlora_profile_read", "runlora_launch_count", "runlora_status_string", "runlora_last_error",
           "runlora_quantize_w_e4m3", "runlora_workspace_size_wq", "runlora_forward_wq", "runlora_backward_wq",
           "runlora_allreduce_sum_f32", "runlora_exchange_sizes", "runlora_exchange_create", "runlora_exchange_destroy",
           "runlora_backward_exchange", "runlora_wprime_t", "runlora_wprime_t_wq", "runlora_forward_wprime"]


def _load():
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2312_03415_b200.build` "
                           "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I, U64, SZ = C.c_void_p, C.c_int, C.c_uint64, C.c_size_t
    S = C.POINTER(Shape)
    sig = {
        "runlora_version": (C.c_char_p, []),
        "runlora_create": (I, [C.POINTER(P), I]),
        "runlora_destroy": (I, [P]),
        "runlora_flops": (I, [S, I, I, C.POINTER(U64)]),
        "runlora_param_reduction": (I, [S]),
        "runlora_workspace_size": (I, [S, I, I, C.POINTER(SZ)]),
        "runlora_select": (I, [P, S, I, C.POINTER(Operands), P, SZ, P, C.POINTER(Plan)]),
        "runlora_forward": (I, [P, I, S, P, P, P, P, P, P, SZ, P]),
        "runlora_backward": (I, [P, I, S, P, P, P, P, P, P, P, P, I, I, P, SZ, P]),
        "runlora_backward_params": (I, [P, I, S, P, P, P, P, P, P, P, I, I, P, SZ, P]),
        "runlora_backward_input": (I, [P, I, S, P, P, P, P, P, P, P, SZ, P]),
        "runlora_step_host": (I, [P, S, C.POINTER(HostStep), P, SZ, P]),
        "runlora_profile_enable": (I, [P, I]),
        "runlora_profile_read": (I, [P, C.POINTER(KernelStat), I, C.POINTER(I), I]),
        "runlora_launch_count": (U64, [P]),
        "runlora_status_string": (C.c_char_p, [I]),
        "runlora_last_error": (C.c_char_p, []),
        "runlora_quantize_w_e4m3": (I, [P, C.c_int64, C.c_int64, P, P, P, P, P]),
        "runlora_workspace_size_wq": (I, [S, I, I, C.POINTER(SZ)]),
        "runlora_forward_wq": (I, [P, I, S, P, P, P, P, P, P, P, P, SZ, P]),
        "runlora_backward_wq": (I, [P, I, S, P, P, P, P, P, P, P, P, P, P, I, I, P, SZ, P]),
        "runlora_allreduce_sum_f32": (I, [P, C.POINTER(P), I, P, C.c_int64, P]),
        "runlora_exchange_sizes": (I, [C.c_int64, C.c_int64, C.c_int64, I, C.POINTER(SZ), C.POINTER(SZ)]),
        "runlora_exchange_create": (I, [P, I, I, C.c_int64, C.c_int64, C.c_int64, C.POINTER(P), C.POINTER(P), P,
                                        C.POINTER(P)]),
        "runlora_exchange_destroy": (I, [P]),
        "runlora_backward_exchange": (I, [P, I, S, P, P, P, P, P, P, P, P, I, I, P, C.c_uint32, P, SZ, P]),
        "runlora_wprime_t": (I, [P, S, P, P, P, P, P]),
        "runlora_wprime_t_wq": (I, [P, S, P, P, P, P, P, P, P]),
        "runlora_forward_wprime": (I, [P, S, P, P, P, P, SZ, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


class RunLoRAError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = _lib.runlora_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)} — {msg}")


def _check(st, where):
    if st != 0:
        raise RunLoRAError(st, where)


def version() -> str:
    return _lib.runlora_version().decode()


def make_shape(n, k, m, r, dtype=BF16) -> Shape:
    if isinstance(dtype, torch.dtype):
        dtype = _DT[dtype]
    return Shape(int(n), int(k), int(m), int(r), int(dtype))


def flops(shape: Shape, is_backward: bool, variant: int) -> int:
    out = C.c_uint64()
    _check(_lib.runlora_flops(C.byref(shape), int(is_backward), int(variant), C.byref(out)), "runlora_flops")
    return int(out.value)


def param_reduction(shape: Shape) -> bool:
    return bool(_lib.runlora_param_reduction(C.byref(shape)))


def workspace_size(shape: Shape, fwd: int = 0, bwd: int = 0) -> int:
    out = C.c_size_t()
    _check(_lib.runlora_workspace_size(C.byref(shape), int(fwd), int(bwd), C.byref(out)), "runlora_workspace_size")
    return int(out.value)


class QuantizedWeight:
    """A frozen W [k, m] stored as FP8 E4M3 bytes `q` with one power-of-two fp32 `scale` per
    output column and their E5M2 diagonal `diag` [m, 128] (R18); `shape` is (k, m)."""

    def __init__(self, q: torch.Tensor, scale: torch.Tensor, diag: torch.Tensor):
        self.q, self.scale, self.diag = q, scale, diag

    @property
    def shape(self):
        return tuple(self.q.shape)

    @property
    def device(self):
        return self.q.device


def workspace_size_wq(shape: Shape) -> int:
    out = C.c_size_t()
    _check(_lib.runlora_workspace_size_wq(C.byref(shape), 0, 0, C.byref(out)), "runlora_workspace_size_wq")
    return out.value


def exchange_sizes(k, m, r, P):
    """(buffer bytes, flag bytes) of each rank's fused-exchange buffers (runlora_exchange_sizes)."""
    b, f = C.c_size_t(), C.c_size_t()
    _check(_lib.runlora_exchange_sizes(int(k), int(m), int(r), int(P), C.byref(b), C.byref(f)),
           "runlora_exchange_sizes")
    return int(b.value), int(f.value)


def exchange_destroy(x):
    _lib.runlora_exchange_destroy(x)


def select_by_flops(shape: Shape) -> Plan:
    p = Plan()
    _check(_lib.runlora_select(None, C.byref(shape), BY_FLOPS, None, None, 0, None, C.byref(p)), "runlora_select")
    return p


def _ptr(t):
    # argtypes declare c_void_p: a plain int (or None) converts without a wrapper object
    return None if t is None else t.data_ptr()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(device):
    if _raw_stream is not None:
        return _raw_stream(device.index or 0)
    return torch.cuda.current_stream(device).cuda_stream


class Handle:
    """One library handle per CUDA device (host caches: TMA descriptors, plans)."""

    def __init__(self, device=0):
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        h = C.c_void_p()
        _check(_lib.runlora_create(C.byref(h), self.device.index or 0), "runlora_create")
        self._h = h
        self._ws = None

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None:
                _lib.runlora_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # workspace: plain device memory owned by the caller side of the ABI
    def workspace(self, shape: Shape, quantized_w: bool = False) -> torch.Tensor:
        need = workspace_size_wq(shape) if quantized_w else workspace_size(shape)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    # ------------------------------------------------- DP exchange (one-shot allreduce)
    def allreduce_sum_f32(self, peer_ptrs, out: torch.Tensor, n: int = None):
        """out[:n] = sum over peer_ptrs (device addresses of fp32 buffers, rank order) —
        runlora_allreduce_sum_f32; the cross-rank barriers are the caller's."""
        n = out.numel() if n is None else int(n)
        arr = (C.c_void_p * len(peer_ptrs))(*[int(p) for p in peer_ptrs])
        _check(_lib.runlora_allreduce_sum_f32(self._h, arr, len(peer_ptrs), _ptr(out), n, _stream(self.device)),
               "runlora_allreduce_sum_f32")

    # ------------------------------------------------- fused DP exchange (NEXT-2)
    def exchange_create(self, P, rank, k, m, r, buf_ptrs, flag_ptrs, mc_ptr=None):
        """runlora_exchange_create: this rank's view of the ranks' exchange buffers / flag arrays
        (device addresses in rank order, as mapped in this process)."""
        x = C.c_void_p()
        bufs = (C.c_void_p * P)(*[int(v) for v in buf_ptrs])
        flags = (C.c_void_p * P)(*[int(v) for v in flag_ptrs])
        _check(_lib.runlora_exchange_create(self._h, P, rank, k, m, r, bufs, flags, mc_ptr or None, C.byref(x)),
               "runlora_exchange_create")
        return x

    def backward_exchange(self, bwd, shape, X, W, A, B, dY, dX, dA, dB, xchg, epoch, accumulate=False, ws=None):
        """runlora_backward_exchange: the backward with dA, dB summed over the ranks by the dX
        GEMM launch's idle warps (fp32 gradients)."""
        ws = self.workspace(shape) if ws is None else ws
        _check(_lib.runlora_backward_exchange(self._h, int(bwd), C.byref(shape), _ptr(X), _ptr(W), _ptr(A), _ptr(B),
                                              _ptr(dY), _ptr(dX), _ptr(dA), _ptr(dB), F32, int(bool(accumulate)),
                                              xchg, int(epoch), _ptr(ws), ws.numel(), _stream(self.device)),
               "runlora_backward_exchange")

    # ------------------------------------------------- quantized frozen W (R18)
    def quantize_w(self, W: torch.Tensor):
        """W bf16 [k, m] -> QuantizedWeight (FP8 E4M3 bytes [k, m], fp32 scale [m])."""
        k, m = W.shape
        Wq = torch.empty(k, m, dtype=torch.uint8, device=W.device)
        scale = torch.empty(m, dtype=torch.float32, device=W.device)
        diag = torch.empty(m, 128, dtype=torch.uint8, device=W.device)
        _check(_lib.runlora_quantize_w_e4m3(self._h, k, m, _ptr(W), _ptr(Wq), _ptr(scale), _ptr(diag),
                                            _stream(self.device)), "runlora_quantize_w_e4m3")
        return QuantizedWeight(Wq, scale, diag)

    def forward_wq(self, fwd, shape, X, Wq, A, B, Y, ws=None):
        ws = self.workspace(shape, True) if ws is None else ws
        _check(_lib.runlora_forward_wq(self._h, int(fwd), C.byref(shape), _ptr(X), _ptr(Wq.q), _ptr(Wq.scale),
                                       _ptr(Wq.diag), _ptr(A), _ptr(B), _ptr(Y), _ptr(ws), ws.numel(),
                                       _stream(self.device)),
               "runlora_forward_wq")

    def backward_wq(self, bwd, shape, X, Wq, A, B, dY, dX, dA, dB, accumulate=False, ws=None):
        ws = self.workspace(shape, True) if ws is None else ws
        _check(_lib.runlora_backward_wq(self._h, int(bwd), C.byref(shape), _ptr(X), _ptr(Wq.q), _ptr(Wq.scale),
                                        _ptr(Wq.diag), _ptr(A), _ptr(B), _ptr(dY), _ptr(dX), _ptr(dA), _ptr(dB),
                                        _DT[dA.dtype],
                                        int(bool(accumulate)), _ptr(ws), ws.numel(), _stream(self.device)),
               "runlora_backward_wq")

    # ------------------------------------------------- forward2 in two halves
    def wprime_t(self, shape, W, A, B, Wpt):
        """runlora_wprime_t (or _wq for a QuantizedWeight): Wpt [m, k] = (W + A·B)ᵀ."""
        if isinstance(W, QuantizedWeight):
            _check(_lib.runlora_wprime_t_wq(self._h, C.byref(shape), _ptr(W.q), _ptr(W.scale), _ptr(W.diag),
                                            _ptr(A), _ptr(B), _ptr(Wpt), _stream(self.device)),
                   "runlora_wprime_t_wq")
        else:
            _check(_lib.runlora_wprime_t(self._h, C.byref(shape), _ptr(W), _ptr(A), _ptr(B), _ptr(Wpt),
                                         _stream(self.device)), "runlora_wprime_t")

    def forward_wprime(self, shape, X, Wpt, Y, ws=None):
        """runlora_forward_wprime: Y = X·W' from a W'ᵀ built by wprime_t."""
        ws = self.workspace(shape) if ws is None else ws
        _check(_lib.runlora_forward_wprime(self._h, C.byref(shape), _ptr(X), _ptr(Wpt), _ptr(Y), _ptr(ws),
                                           ws.numel(), _stream(self.device)), "runlora_forward_wprime")

    def select(self, shape: Shape, criterion=BY_FLOPS, ops: dict | None = None, grad_dtype=F32) -> Plan:
        p = Plan()
        o = None
        ws, wsb = None, 0
        if criterion != BY_FLOPS:
            o = Operands(*[_ptr(ops.get(k)) for k in ("X", "W", "A", "B", "dY", "Y", "dX", "dA", "dB")],
                         int(grad_dtype))
            w = self.workspace(shape)
            ws, wsb = _ptr(w), w.numel()
        _check(_lib.runlora_select(self._h, C.byref(shape), int(criterion), C.byref(o) if o is not None else None,
                                   ws, wsb, _stream(self.device), C.byref(p)), "runlora_select")
        return p

    def forward(self, fwd, shape, X, W, A, B, Y, ws=None):
        ws = self.workspace(shape) if ws is None else ws
        _check(_lib.runlora_forward(self._h, int(fwd), C.byref(shape), _ptr(X), _ptr(W), _ptr(A), _ptr(B), _ptr(Y),
                                    _ptr(ws), ws.numel(), _stream(self.device)), "runlora_forward")

    def backward(self, bwd, shape, X, W, A, B, dY, dX, dA, dB, accumulate=False, ws=None):
        ws = self.workspace(shape) if ws is None else ws
        _check(_lib.runlora_backward(self._h, int(bwd), C.byref(shape), _ptr(X), _ptr(W), _ptr(A), _ptr(B), _ptr(dY),
                                     _ptr(dX), _ptr(dA), _ptr(dB), _DT[dA.dtype], int(bool(accumulate)), _ptr(ws),
                                     ws.numel(), _stream(self.device)), "runlora_backward")

    def backward_params(self, bwd, shape, X, W, A, B, dY, dA, dB, accumulate=False, ws=None):
        ws = self.workspace(shape) if ws is None else ws
        _check(_lib.runlora_backward_params(self._h, int(bwd), C.byref(shape), _ptr(X), _ptr(W), _ptr(A), _ptr(B),
                                            _ptr(dY), _ptr(dA), _ptr(dB), _DT[dA.dtype], int(bool(accumulate)),
                                            _ptr(ws), ws.numel(), _stream(self.device)), "runlora_backward_params")

    def backward_input(self, bwd, shape, X, W, A, B, dY, dX, ws=None):
        ws = self.workspace(shape) if ws is None else ws
        _check(_lib.runlora_backward_input(self._h, int(bwd), C.byref(shape), _ptr(X), _ptr(W), _ptr(A), _ptr(B),
                                           _ptr(dY), _ptr(dX), _ptr(ws), ws.numel(), _stream(self.device)),
               "runlora_backward_input")

    def step_host(self, shape, fwd, bwd, host: dict, dev: dict, grad_dtype, accumulate=False, ws=None,
                  exchange=None):
        """runlora_step_host.  `exchange`: optional callable run after the backward is enqueued
        and before the D2H copies (e.g. the data-parallel allreduce of dA, dB on the current
        stream), so the host buffers receive its result."""
        ws = self.workspace(shape) if ws is None else ws
        cb = EXCHANGE_FN(lambda user, stream: exchange()) if exchange is not None else EXCHANGE_FN()
        st = HostStep(int(fwd), int(bwd), int(grad_dtype), int(bool(accumulate)),
                      _ptr(host["X"]), _ptr(host["dY"]), _ptr(host.get("Y")), _ptr(host.get("dX")),
                      _ptr(host["dA"]), _ptr(host["dB"]),
                      _ptr(dev["W"]), _ptr(dev["A"]), _ptr(dev["B"]),
                      _ptr(dev["X"]), _ptr(dev["dY"]), _ptr(dev["Y"]), _ptr(dev["dX"]), _ptr(dev["dA"]),
                      _ptr(dev["dB"]), cb, None)
        _check(_lib.runlora_step_host(self._h, C.byref(shape), C.byref(st), _ptr(ws), ws.numel(),
                                      _stream(self.device)), "runlora_step_host")

    def profile_enable(self, on=True):
        _check(_lib.runlora_profile_enable(self._h, int(bool(on))), "runlora_profile_enable")

    def profile_read(self, reset=True) -> dict:
        arr = (KernelStat * 32)()
        cnt = C.c_int()
        _check(_lib.runlora_profile_read(self._h, arr, 32, C.byref(cnt), int(bool(reset))), "runlora_profile_read")
        return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms)) for i in range(cnt.value)}

    def launch_count(self) -> int:
        return int(_lib.runlora_launch_count(self._h))


_handles: dict = {}
_hlock = threading.Lock()


def handle(device=None) -> Handle:
    """Process-wide handle for a CUDA device."""
    dev = torch.cuda.current_device() if device is None else (device if isinstance(device, int) else device.index)
    with _hlock:
        h = _handles.get(dev)
        if h is None:
            h = _handles[dev] = Handle(dev)
        return h
