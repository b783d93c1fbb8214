# DeepSeek (1-CTA engine, ~1.5 M units per expert) raster band A/B through the bench step,
# alternating; plus the new roofline floor model on the bench line
for b in 0 4 8 32 0 8; do
  if [ $b = 0 ]; then unset MOE_B200_BAND; else export MOE_B200_BAND=$b; fi
  timeout 400 python bench.py --config deepseek --no-cpu-baseline --no-dropin > gpurun_out/r5y_ds_b$b.json 2>gpurun_out/r5y_ds_b$b.err
  python -c "import json;d=json.loads(open('gpurun_out/r5y_ds_b$b.json').read().strip().splitlines()[-1]);r=d['roofline'];print('band $b', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], r['bound'], r['frac'], r['floor_model']['frac_of_floor'], {k:v['measured_ms'] for k,v in r['floor_model']['per_gemm'].items()})" || tail -3 gpurun_out/r5y_ds_b$b.err
done
unset MOE_B200_BAND
timeout 300 python bench.py --config mixtral --no-cpu-baseline --no-dropin > gpurun_out/r5y_mixtral.json 2>gpurun_out/r5y_mixtral.err
python -c "import json;d=json.loads(open('gpurun_out/r5y_mixtral.json').read().strip().splitlines()[-1]);r=d['roofline'];print('mixtral', d['value'], r['bound'], r['frac'], r['floor_model']['frac_of_floor'])" || tail -3 gpurun_out/r5y_mixtral.err
