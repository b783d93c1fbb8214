# Full validation of the committed state: GPU tests (EP tests use all GPUs of the box),
# smoke, bench lines at N = 1, 2, 4 and the reference arm.
export MOE_TEST_TIMEOUT=150
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin2_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/fin2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/fin2_smoke.log
python bench.py > gpurun_out/fin2_bench1.json 2> gpurun_out/fin2_bench1.err
python bench.py --impl reference > gpurun_out/fin2_ref1.json 2> gpurun_out/fin2_ref1.err
for n in 2 4; do timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n > gpurun_out/fin2_bench$n.json 2> gpurun_out/fin2_bench$n.err; done
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29529 bench.py --gpus 4 --graph > gpurun_out/fin2_bench4_graph.json 2> gpurun_out/fin2_bench4_graph.err
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29530 bench.py --gpus 2 --impl reference > gpurun_out/fin2_ref2.json 2> gpurun_out/fin2_ref2.err
tail -3 gpurun_out/fin2_pytest.log; cat gpurun_out/fin2_smoke.log
for f in fin2_bench1 fin2_ref1 fin2_bench2 fin2_bench4 fin2_bench4_graph fin2_ref2; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), d.get('n_gpus'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('samples'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))"; done
