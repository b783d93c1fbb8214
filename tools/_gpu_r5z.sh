# bench with the GEMM busy time as the union of the GEMM event spans + the floor model
timeout 300 python -m pytest tests/test_bench_contract.py -x -q -m gpu > gpurun_out/r5z_pytest.log 2>&1; tail -2 gpurun_out/r5z_pytest.log
for c in mixtral qwen3 deepseek; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --no-dropin > gpurun_out/r5z_$c.json 2>gpurun_out/r5z_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/r5z_$c.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$c', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], r['bound'], r['frac'], r['gemm_ms_per_step'], r['floor_model']['floor_ms'], r['floor_model']['frac_of_floor'], d['gemm_exclusive_ms_per_step'])" || tail -3 gpurun_out/r5z_$c.err
done
