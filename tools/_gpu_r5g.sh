export MOE_TEST_TIMEOUT=150
timeout 600 python -m pytest tests/test_layer_gpu.py tests/test_layer_scale_gpu.py tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2 3 4; do
  for pd in 1 0; do MOE_B200_WGRAD_PDL=$pd timeout 400 python bench.py --no-cpu-baseline --no-dropin --steps 30 > gpurun_out/r5g_$pd.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r5g_$pd.json').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];g=sum(v for x,v in k.items() if x.startswith('moe_gg'));print('wgrad_pdl=$pd', d.get('ms_per_step'), 'gemm', round(g,3), 'mhz', (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))"; done
done
