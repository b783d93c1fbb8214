# Last check of the final tree on one B200: GPU suite, smoke, default bench line
export MOE_TEST_TIMEOUT=150
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin9_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/fin9_pytest.log
tail -2 gpurun_out/fin9_pytest.log; grep -E "^FAILED" gpurun_out/fin9_pytest.log | head
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin9_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/fin9_smoke.log; tail -2 gpurun_out/fin9_smoke.log
python bench.py > gpurun_out/fin9_bench1.json 2> gpurun_out/fin9_bench1.err
python -c "import json;d=json.loads(open('gpurun_out/fin9_bench1.json').read().strip().splitlines()[-1]);print('fin9', d['value'], d['ms_per_step'], d['steps'], d['clocks'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['cpu_baseline']['value'])"
