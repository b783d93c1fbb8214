# in-step A/B: streaming epilogue stores (MOE_B200_EPI_CS) and, at Qwen3, the 128-row plan
for i in 1 2; do
  for v in "0 256" "1 256" "0 128"; do set -- $v
    MOE_B200_EPI_CS=$1 MOE_B200_ALIGN=$2 timeout 300 python bench.py --config qwen3 --no-cpu-baseline --no-dropin --steps 30 > gpurun_out/r5r.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r5r.json').read().strip().splitlines()[-1]);print('qwen3 cs=$1 align=$2', d.get('ms_per_step'), 'mhz', (d.get('clocks') or {}).get('sm_mhz'))"
  done
  for cs in 0 1; do MOE_B200_EPI_CS=$cs timeout 300 python bench.py --no-cpu-baseline --no-dropin --steps 30 > gpurun_out/r5r.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r5r.json').read().strip().splitlines()[-1]);print('mixtral cs=$cs', d.get('ms_per_step'), 'mhz', (d.get('clocks') or {}).get('sm_mhz'))"; done
done
