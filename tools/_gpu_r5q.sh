# EP with the weight gradients as programmatic dependent launches: loopback EP tests (1 GPU
# process, 2 GPUs of the box for the real EP tests), EP=2 bench A/B
export MOE_TEST_TIMEOUT=200
timeout 900 python -m pytest tests/test_ep_loopback_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_ep_gpu.py -q -p no:cacheprovider -k "layer_matches and (p2p or nccl)" 2>&1 | tail -2
for i in 1 2; do for pd in 1 0; do MOE_B200_WGRAD_PDL=$pd timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2971$pd bench.py --gpus 2 --no-cpu-baseline --no-dropin > gpurun_out/r5q_$pd.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r5q_$pd.json').read().strip().splitlines()[-1]);print('ep2 wgrad_pdl=$pd', d.get('value'), d.get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'))"; done; done
