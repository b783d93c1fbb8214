# Final EP validation on a 4-GPU box: EP parity tests at EP=4 (and the rest of the GPU suite),
# bench lines at N=2 and N=4 (Mixtral, Qwen3, DeepSeek at 4), CUDA-graph EP=4, reference arm
export MOE_TEST_TIMEOUT=200
nvidia-smi --query-gpu=index,name --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin4_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/fin4_pytest.log
tail -3 gpurun_out/fin4_pytest.log; grep -E "^FAILED" gpurun_out/fin4_pytest.log | head
for n in 2 4; do timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n > gpurun_out/fin4_bench$n.json 2> gpurun_out/fin4_bench$n.err; done
for c in qwen3 deepseek; do timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --config $c > gpurun_out/fin4_bench4_$c.json 2> gpurun_out/fin4_bench4_$c.err; done
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 --graph > gpurun_out/fin4_bench4_graph.json 2> gpurun_out/fin4_bench4_graph.err
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29583 bench.py --gpus 4 --impl reference > gpurun_out/fin4_ref4.json 2> gpurun_out/fin4_ref4.err
for f in fin4_bench2 fin4_bench4 fin4_bench4_qwen3 fin4_bench4_deepseek fin4_bench4_graph fin4_ref4; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), d.get('n_gpus'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))"; done
