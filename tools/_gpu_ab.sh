python -m pytest tests/test_ep_plan_gpu.py -x -q -p no:cacheprovider > gpurun_out/ab4_plan.log 2>&1; echo rc=$? >> gpurun_out/ab4_plan.log
timeout 900 python -m pytest tests/test_ep_gpu.py -x -q -p no:cacheprovider -k "p2p and not pull and not dedup and not overlap" > gpurun_out/ab4_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/ab4_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 10 --no-cpu-baseline"
for cfg in qwen3 mixtral; do
  timeout 300 $TR --config $cfg > gpurun_out/ab4_${cfg}_p2p.json 2> gpurun_out/ab4_${cfg}_p2p.err
  timeout 300 $TR --config $cfg --sync-free > gpurun_out/ab4_${cfg}_sf.json 2> gpurun_out/ab4_${cfg}_sf.err
  timeout 300 $TR --config $cfg --graph > gpurun_out/ab4_${cfg}_graph.json 2> gpurun_out/ab4_${cfg}_graph.err
done
tail -2 gpurun_out/ab4_plan.log gpurun_out/ab4_pytest.log
