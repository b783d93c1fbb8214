# timed-region length vs the power limiter: ms_per_step and the last step's kernel sum
for s in 20 60 20 100; do
  timeout 400 python bench.py --steps $s --no-cpu-baseline --no-dropin > gpurun_out/r6f_s$s.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r6f_s$s.json').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('steps $s', d['value'], d['ms_per_step'], round(sum(k.values()),3), d['clocks']['sm_mhz'], d['roofline']['frac'])"
done
