export MOE_TEST_TIMEOUT=150
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py tests/test_layer_scale_gpu.py tests/test_ep_loopback_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
export POWER_NO_CUBLAS=1 POWER_KINDS=fc1_fwd,fc2_fwd,fc2_dgrad,fc1_dgrad
cd tools
for cfg in qwen3 mixtral; do echo "== $cfg auto band"; POWER_CONFIG=$cfg timeout 200 python power_probe.py 2>&1 | grep -v "^{" | tail -4; echo "== $cfg band 16"; MOE_B200_BAND=16 POWER_CONFIG=$cfg timeout 200 python power_probe.py 2>&1 | grep -v "^{" | tail -4; done
cd ..
for c in qwen3 mixtral; do timeout 400 python bench.py --config $c > gpurun_out/r4y_bench_$c.json 2> gpurun_out/r4y_bench_$c.err; python -c "import json;d=json.loads(open('gpurun_out/r4y_bench_$c.json').read().strip().splitlines()[-1]);print('$c', d.get('value'), d.get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('roofline') or {}).get('frac_vs'), d['kernel_ms_per_step'].get('moe_zero_pad_rows'))"; done
