timeout 300 python -m pytest tests/test_bench_contract.py tests/test_abi.py -x -q -m gpu > gpurun_out/r6a_pytest.log 2>&1; tail -2 gpurun_out/r6a_pytest.log
for c in qwen3 mixtral; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --no-dropin > gpurun_out/r6a_$c.json 2>gpurun_out/r6a_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/r6a_$c.json').read().strip().splitlines()[-1]);h=d['hbm_kernels'];print('$c', d['value'], h['_peaks'], {k:(v['frac_of_measured_hbm'],v['frac_of_bound']) for k,v in h.items() if k!='_peaks'})" || tail -3 gpurun_out/r6a_$c.err
done
