# small-N router: parity tests + probe; wave-sync lag matrix on the grouped-M kinds; HBM probe
export MOE_TEST_TIMEOUT=150
timeout 900 python -m pytest tests/test_router_gpu.py tests/test_routing_api_gpu.py tests/test_layer_gpu.py tests/test_layer_scale_gpu.py -x -q -p no:cacheprovider > gpurun_out/r4c_pytest.log 2>&1; tail -3 gpurun_out/r4c_pytest.log
grep -E "FAIL|Error|error" gpurun_out/r4c_pytest.log | head -20
timeout 300 python tools/router_probe.py 2>&1 | tail -14
export POWER_NO_CUBLAS=1 POWER_KINDS=fc1_fwd,fc2_fwd,fc2_dgrad,fc1_dgrad
cd tools
for cfg in mixtral qwen3; do
  for v in "0 0 0" "1 64 0" "1 64 1" "1 32 1" "1 32 2" "1 16 2"; do set -- $v
    echo "== $cfg sync=$1 kb=$2 lag=$3"
    POWER_CONFIG=$cfg MOE_B200_WAVE_SYNC=$1 MOE_B200_SYNC_KB=$2 MOE_B200_SYNC_LAG=$3 timeout 300 python power_probe.py 2>&1 | grep -v "^{" | tail -4
  done
done
cd ..
timeout 300 python tools/hbm_probe.py 2>&1 | tail -12
