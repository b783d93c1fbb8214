# small-N router (fp32 fast selection, warp-uniform exact fallback): parity tests, probe, ncu
export MOE_TEST_TIMEOUT=120
timeout 240 python -m pytest tests/test_router_gpu.py -x -q -p no:cacheprovider > gpurun_out/r4e_pytest_router.log 2>&1; echo rc=$?; tail -2 gpurun_out/r4e_pytest_router.log
grep -E "^FAILED|^E  " gpurun_out/r4e_pytest_router.log | head -10
nvidia-smi --query-gpu=utilization.gpu --format=csv
timeout 300 python -m pytest tests/test_routing_api_gpu.py -x -q -p no:cacheprovider > gpurun_out/r4e_pytest_api.log 2>&1; echo rc=$?; tail -2 gpurun_out/r4e_pytest_api.log
grep -E "^FAILED|^E  " gpurun_out/r4e_pytest_api.log | head -10
timeout 600 python -m pytest tests/test_layer_gpu.py tests/test_layer_scale_gpu.py -x -q -p no:cacheprovider > gpurun_out/r4e_pytest_layer.log 2>&1; echo rc=$?; tail -2 gpurun_out/r4e_pytest_layer.log
grep -E "^FAILED|^E  " gpurun_out/r4e_pytest_layer.log | head -10
timeout 200 python tools/router_probe.py 2>&1 | grep -v small | tail -14
for c in mixtral qwen3 deepseek; do
  timeout 200 ncu --set full --clock-control none --import-source on -k regex:router_tc_kernel -s 2 -c 2 -o gpurun_out/r4e_router_$c python tools/router_one.py $c 3 > gpurun_out/r4e_ncu_$c.log 2>&1
  tail -1 gpurun_out/r4e_ncu_$c.log
done
