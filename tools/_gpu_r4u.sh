# EP on 2 GPUs with the small-N router: EP parity tests, N=2 bench (Mixtral), reference arm
export MOE_TEST_TIMEOUT=200
timeout 1500 python -m pytest tests/test_ep_gpu.py tests/test_ep_plan_gpu.py -q -p no:cacheprovider > gpurun_out/r4u_pytest_ep2.log 2>&1; echo pytest_rc=$? >> gpurun_out/r4u_pytest_ep2.log
tail -3 gpurun_out/r4u_pytest_ep2.log; grep -E "^FAILED" gpurun_out/r4u_pytest_ep2.log | head
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 > gpurun_out/r4u_bench2.json 2> gpurun_out/r4u_bench2.err
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --config qwen3 > gpurun_out/r4u_bench2_qwen3.json 2> gpurun_out/r4u_bench2_qwen3.err
for f in r4u_bench2 r4u_bench2_qwen3; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))"; done
tail -3 gpurun_out/r4u_bench2.err
