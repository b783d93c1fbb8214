# A/B of the EP transports at EP=4 + EP parity tests (p2p variants)
python -m pytest tests/test_ep_gpu.py -x -q -p no:cacheprovider -k "p2p and not pull and not dedup" > gpurun_out/ab3_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/ab3_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 10 --no-cpu-baseline"
for cfg in qwen3 mixtral deepseek; do for tr in p2p p2p_sync p2p_dedup; do
  timeout 300 $TR --config $cfg --ep-transport $tr > gpurun_out/ab3_${cfg}_${tr}.json 2> gpurun_out/ab3_${cfg}_${tr}.err
done; done
tail -2 gpurun_out/ab3_pytest.log
