"""B200-native (sm_100a) MoE-layer hot path: router, permute, grouped-GEMM SwiGLU
experts, combine and the expert-parallel dispatcher.

A drop-in for the function API of the reference ``moelab.routing`` module
(reference pkg/src/moelab/routing.py), backed by hand-written CUDA kernels in
``libmoe_b200.so`` (C-ABI, include/moe_b200.h). There is no CPU fallback.
"""
__version__ = "0.1.0"
