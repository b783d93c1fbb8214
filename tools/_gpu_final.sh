# Full validation: GPU tests (EP tests use all GPUs of the box), smoke, bench lines, ncu.
export MOE_TEST_TIMEOUT=150
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/fin_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/fin_smoke.log
python bench.py > gpurun_out/fin_bench1.json 2> gpurun_out/fin_bench1.err
python bench.py --impl reference > gpurun_out/fin_ref1.json 2> gpurun_out/fin_ref1.err
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 4"
timeout 400 $TR > gpurun_out/fin_bench4_mixtral.json 2> gpurun_out/fin_bench4_mixtral.err
timeout 400 $TR --config qwen3 > gpurun_out/fin_bench4_qwen3.json 2> gpurun_out/fin_bench4_qwen3.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mxfp8_gemm_kernel -s 6 -c 1 -o gpurun_out/fin_ncu_mxfp8 python tools/mxfp8_probe.py > gpurun_out/fin_ncu_mxfp8.log 2>&1
tail -3 gpurun_out/fin_pytest.log; cat gpurun_out/fin_smoke.log
for f in fin_bench1 fin_ref1 fin_bench4_mixtral fin_bench4_qwen3; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), d.get('clocks'), (d.get('roofline') or {}).get('frac'))"; done
