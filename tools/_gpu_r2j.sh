timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py tests/test_layer_scale_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
python tools/gemm_kinds.py deepseek all 10 2>&1 | grep -v "^{"
python tools/gemm_kinds.py mixtral fc2_wgrad 10 2>&1 | grep -v "^{"
