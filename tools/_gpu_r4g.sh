# small-N router, smem-resident logits tile: parity, probe, ncu summaries
export MOE_TEST_TIMEOUT=120
timeout 240 python -m pytest tests/test_router_gpu.py tests/test_routing_api_gpu.py -x -q -p no:cacheprovider > gpurun_out/r4g_pytest_router.log 2>&1; echo rc=$?; tail -2 gpurun_out/r4g_pytest_router.log
grep -E "^FAILED|^E  " gpurun_out/r4g_pytest_router.log | head -10
timeout 600 python -m pytest tests/test_layer_gpu.py tests/test_layer_scale_gpu.py -x -q -p no:cacheprovider > gpurun_out/r4g_pytest_layer.log 2>&1; echo rc=$?; tail -2 gpurun_out/r4g_pytest_layer.log
timeout 200 python tools/router_probe.py 2>&1 | grep -v small | tail -14
for c in qwen3 deepseek mixtral; do
  timeout 200 ncu --set full --clock-control none --import-source on -k regex:router_tc_kernel -s 2 -c 2 -o /tmp/r4g_$c python tools/router_one.py $c 3 > gpurun_out/r4g_ncu_$c.log 2>&1
  NCU_TOP_SASS=25 python tools/ncu_summary.py /tmp/r4g_$c.ncu-rep "router_tc $c" > gpurun_out/r4g_router_$c.txt 2>&1
  grep -E "kernel:|duration|dram_thr|issue_slots|warp-stall" gpurun_out/r4g_router_$c.txt
done
