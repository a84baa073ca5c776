"""B200-native (sm_100a) RunLoRA hot path: forward/backward of a LoRA-adapted
linear layer with variant selection (arXiv 2312.03415).

Layout: csrc/ (CUDA kernels + C ABI, built into lib/librunlora.so),
runlora.py (ctypes binding), lora.py (autograd op), dp.py (token-sharded DP),
stack.py (C5 stack: model-level planning, bucketed gradient sync).
"""
__all__ = ["runlora", "lora", "dp", "stack", "build"]
