for i in 1 2 3 4; do
  for g in "--graph" ""; do timeout 400 python bench.py --no-cpu-baseline --no-dropin --steps 30 $g > gpurun_out/r5i.json 2>gpurun_out/r5i.err; python -c "import json;d=json.loads(open('gpurun_out/r5i.json').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];g=sum(v for x,v in k.items() if x.startswith('moe_gg'));print('graph=$g', d.get('ms_per_step'), 'gemm', round(g,3), 'mhz', (d.get('clocks') or {}).get('sm_mhz'), 'e2e', d['e2e']['ms_per_step'], 'launches', d.get('gpu_launches'))" || tail -5 gpurun_out/r5i.err; done
done
