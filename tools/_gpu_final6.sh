# Final validation (6), end of session (write probe, GEMM busy-time union, floor model): GPU tests, smoke, bench lines (default Mixtral with the
# CPU baseline and drop-in timing, Qwen3, DeepSeek), reference arm, ncu launch list
export MOE_TEST_TIMEOUT=150
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin6_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/fin6_pytest.log
tail -3 gpurun_out/fin6_pytest.log; grep -E "^FAILED" gpurun_out/fin6_pytest.log | head
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin6_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/fin6_smoke.log; tail -2 gpurun_out/fin6_smoke.log
python bench.py > gpurun_out/fin6_bench1.json 2> gpurun_out/fin6_bench1.err
for c in qwen3 deepseek; do timeout 400 python bench.py --config $c > gpurun_out/fin6_bench1_$c.json 2> gpurun_out/fin6_bench1_$c.err; done
python bench.py --impl reference > gpurun_out/fin6_ref1.json 2> gpurun_out/fin6_ref1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin6_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/fin6_ncu.log 2>&1
for f in fin6_bench1 fin6_bench1_qwen3 fin6_bench1_deepseek fin6_ref1; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('gpu_launches'))"; done
