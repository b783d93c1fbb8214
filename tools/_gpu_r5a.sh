export MOE_TEST_TIMEOUT=150
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_layer_scale_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
for c in mixtral qwen3; do
  for sp in 1 0; do MOE_B200_SPLIT_UNITS=$sp timeout 400 python bench.py --config $c --no-cpu-baseline --no-dropin > gpurun_out/r5a_bench_${c}_$sp.json 2> gpurun_out/r5a_bench_${c}_$sp.err; python -c "import json;d=json.loads(open('gpurun_out/r5a_bench_${c}_$sp.json').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('$c split=$sp', d.get('value'), d.get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('roofline') or {}).get('frac_vs',{}).get('clock_adjusted_dense'), {x: k[x] for x in k if x.startswith('moe_gg')})"; done
done
