# Validation of HEAD after the epilogue-TMA / raster / evict-first commits (1 GPU)
export MOE_TEST_TIMEOUT=150
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r4a_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r4a_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4a_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/r4a_smoke.log
for c in mixtral qwen3 deepseek; do timeout 400 python bench.py --config $c > gpurun_out/r4a_bench_$c.json 2> gpurun_out/r4a_bench_$c.err; done
timeout 400 python bench.py --impl reference > gpurun_out/r4a_ref.json 2> gpurun_out/r4a_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r4a_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/r4a_ncu.log 2>&1
tail -3 gpurun_out/r4a_pytest.log; tail -3 gpurun_out/r4a_smoke.log
for f in r4a_bench_mixtral r4a_bench_qwen3 r4a_bench_deepseek r4a_ref; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('kernel_ms_per_step'))"; done
