timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py tests/test_layer_scale_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do python tools/gemm_kinds.py mixtral fc1_fwd 10 2>&1 | grep -v "^{"; python tools/gemm_kinds.py qwen3 fc1_fwd 10 2>&1 | grep -v "^{"; done
MOE_NVCC_EXTRA=-DMOE_SWIGLU_TMA=0 python -m paper_2603_07685_b200.build --force > /dev/null 2>&1 && echo "== no-TMA SwiGLU build" && for i in 1 2; do python tools/gemm_kinds.py mixtral fc1_fwd 10 2>&1 | grep -v "^{"; python tools/gemm_kinds.py qwen3 fc1_fwd 10 2>&1 | grep -v "^{"; done
