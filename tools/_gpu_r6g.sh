# Qwen3 split units A/B at the 60-step window, alternating
for rep in 1 2; do
for v in 1 2; do
  MOE_B200_SPLIT_UNITS=$v timeout 400 python bench.py --config qwen3 --no-cpu-baseline --no-dropin > gpurun_out/r6g_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r6g_$v.json').read().strip().splitlines()[-1]);print('split=$v', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['gemm_ms_per_step'])"
done
done
