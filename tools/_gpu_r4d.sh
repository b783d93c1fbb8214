# small-N router (fp32 fast selection): parity tests, probe, ncu of the fused forward
export MOE_TEST_TIMEOUT=150
timeout 900 python -m pytest tests/test_router_gpu.py tests/test_routing_api_gpu.py tests/test_layer_gpu.py tests/test_layer_scale_gpu.py -x -q -p no:cacheprovider > gpurun_out/r4d_pytest.log 2>&1; tail -3 gpurun_out/r4d_pytest.log
grep -E "^FAILED|^E  " gpurun_out/r4d_pytest.log | head -20
timeout 300 python tools/router_probe.py 2>&1 | grep -v small | tail -14
for c in mixtral qwen3 deepseek; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:router_tc_kernel -s 2 -c 2 -o gpurun_out/r4d_router_$c python tools/router_one.py $c 3 > gpurun_out/r4d_ncu_$c.log 2>&1
  tail -1 gpurun_out/r4d_ncu_$c.log
done
