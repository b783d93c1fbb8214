for i in 1 2 3 4; do
  for sp in 2 0; do MOE_B200_SPLIT_UNITS=$sp timeout 400 python bench.py --config qwen3 --no-cpu-baseline --no-dropin --steps 30 > gpurun_out/r5f_$sp.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r5f_$sp.json').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];g=sum(v for x,v in k.items() if x.startswith('moe_gg'));print('qwen3 split=$sp', d.get('ms_per_step'), 'gemm', round(g,3), 'mhz', (d.get('clocks') or {}).get('sm_mhz'))"; done
done
