export MOE_TEST_TIMEOUT=150
timeout 900 python -m pytest tests/test_ep_gpu.py -q -p no:cacheprovider -k "mxfp8 or (dropless and p2p)" > gpurun_out/mxep.log 2>&1; echo rc=$? >> gpurun_out/mxep.log
timeout 300 python -m pytest tests/test_layer_gpu.py tests/test_mxfp8.py -q -p no:cacheprovider 2>&1 | tail -1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 10 --no-cpu-baseline"
for pr in bf16 mxfp8; do timeout 300 $TR --precision $pr > gpurun_out/mxep_$pr.json 2> gpurun_out/mxep_$pr.err; python -c "import json;d=json.loads(open('gpurun_out/mxep_$pr.json').read().strip().splitlines()[-1]);print('$pr', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; done
tail -4 gpurun_out/mxep.log
