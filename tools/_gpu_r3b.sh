timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
cd tools
echo "== evict-first"; POWER_NO_CUBLAS=1 python power_probe.py 2>&1 | grep -v "^{" | tail -6
cd ..; MOE_NVCC_EXTRA=-DMOE_EPI_EVICT_FIRST=0 python -m paper_2603_07685_b200.build --force > /dev/null 2>&1; cd tools
echo "== normal"; POWER_NO_CUBLAS=1 python power_probe.py 2>&1 | grep -v "^{" | tail -6
