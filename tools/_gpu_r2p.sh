nvidia-smi --query-gpu=index,name --format=csv,noheader | head
timeout 1800 python -m pytest tests/test_ep_gpu.py -x -q -p no:cacheprovider --timeout 600 > gpurun_out/r2p_ep_tests.log 2>&1; echo ep_rc=$?
tail -3 gpurun_out/r2p_ep_tests.log
for cfg in mixtral qwen3 deepseek; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 10 --warmup 3 --config $cfg > gpurun_out/r2p_bench4_$cfg.json 2> gpurun_out/r2p_bench4_$cfg.err; echo $cfg rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r2p_bench4_$cfg.json')); print('$cfg', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], d['nvlink']['achieved_GBps_per_direction'] if d.get('nvlink') else None)"
done
