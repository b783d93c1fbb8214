# split units A/B, alternating runs on one box
for c in mixtral qwen3; do
  for i in 1 2 3; do
    for sp in 1 0; do MOE_B200_SPLIT_UNITS=$sp timeout 400 python bench.py --config $c --no-cpu-baseline --no-dropin --steps 30 > gpurun_out/r5b_$c_$sp.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r5b_$c_$sp.json').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];g=sum(v for x,v in k.items() if x.startswith('moe_gg'));print('$c split=$sp', d.get('ms_per_step'), 'gemm', round(g,3), 'mhz', (d.get('clocks') or {}).get('sm_mhz'), 'clk-adj', (d.get('roofline') or {}).get('frac_vs',{}).get('clock_adjusted_dense'))"; done
  done
done
