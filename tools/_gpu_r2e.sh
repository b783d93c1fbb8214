python tools/gemm_kinds.py mixtral all 10 2>&1 | grep -v "^{" ; echo "== qwen3"; python tools/gemm_kinds.py qwen3 all 10 2>&1 | grep -v "^{"
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py tests/test_layer_scale_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
echo "== 4-warp dSwiGLU build"
MOE_NVCC_EXTRA=-DMOE_DSWIGLU_WARPS=4 python -m paper_2603_07685_b200.build --force > /dev/null 2>&1 && python tools/gemm_kinds.py mixtral fc2_dgrad 10 2>&1 | grep -v "^{"; python tools/gemm_kinds.py qwen3 fc2_dgrad 10 2>&1 | grep -v "^{"
