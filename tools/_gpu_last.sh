export MOE_TEST_TIMEOUT=150
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/last_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/last_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/last_smoke.log
python bench.py > gpurun_out/last_bench1.json 2> gpurun_out/last_bench1.err
tail -3 gpurun_out/last_pytest.log; cat gpurun_out/last_smoke.log
python -c "import json;d=json.loads(open('gpurun_out/last_bench1.json').read().strip().splitlines()[-1]);print('bench1', d['value'], d['ms_per_step'], d['clocks'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'])"
