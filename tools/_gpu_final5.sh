# Final EP validation (2) on a 4-GPU box with the end-of-round code
# bench lines at N=2 and N=4 (Mixtral, Qwen3, DeepSeek at 4), CUDA-graph EP=4, reference arm
export MOE_TEST_TIMEOUT=200
nvidia-smi --query-gpu=index,name --format=csv
MOE_TEST_WORKER_LOG=gpurun_out/fin5_workers timeout 2400 python -m pytest tests/test_ep_gpu.py tests/test_ep_plan_gpu.py -q -p no:cacheprovider > gpurun_out/fin5_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/fin5_pytest.log
tail -3 gpurun_out/fin5_pytest.log; grep -E "^FAILED" gpurun_out/fin5_pytest.log | head
for n in 2 4; do timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n bench.py --gpus $n > gpurun_out/fin5_bench$n.json 2> gpurun_out/fin5_bench$n.err; done
for c in qwen3 deepseek; do timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 4 --config $c > gpurun_out/fin5_bench4_$c.json 2> gpurun_out/fin5_bench4_$c.err; done
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 bench.py --gpus 4 --graph > gpurun_out/fin5_bench4_graph.json 2> gpurun_out/fin5_bench4_graph.err
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29693 bench.py --gpus 4 --impl reference > gpurun_out/fin5_ref4.json 2> gpurun_out/fin5_ref4.err
for f in fin5_bench2 fin5_bench4 fin5_bench4_qwen3 fin5_bench4_deepseek fin5_bench4_graph fin5_ref4; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), d.get('n_gpus'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))"; done
