# full validation after the small-N router + wave sync (1 GPU)
export MOE_TEST_TIMEOUT=150
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r4q_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r4q_pytest.log
tail -3 gpurun_out/r4q_pytest.log; grep -E "^FAILED" gpurun_out/r4q_pytest.log | head
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4q_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/r4q_smoke.log; tail -2 gpurun_out/r4q_smoke.log
for c in mixtral qwen3 deepseek; do timeout 400 python bench.py --config $c > gpurun_out/r4q_bench_$c.json 2> gpurun_out/r4q_bench_$c.err; done
for f in r4q_bench_mixtral r4q_bench_qwen3 r4q_bench_deepseek; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value')); print(json.dumps(d.get('hbm_kernels')))"; done
