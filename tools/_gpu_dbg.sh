TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515"
timeout 150 $TR tools/ep_overlap_debug.py --config qwen3 --tokens 4096 > gpurun_out/dbg_small.out 2>&1
cat gpurun_out/dbg_rank*.log > gpurun_out/dbg_small.log
timeout 200 $TR tools/ep_overlap_debug.py --config qwen3 > gpurun_out/dbg_full.out 2>&1
cat gpurun_out/dbg_rank*.log > gpurun_out/dbg_full.log
cat gpurun_out/dbg_small.log gpurun_out/dbg_full.log
