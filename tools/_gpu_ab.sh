timeout 600 python -m pytest tests/test_mxfp8.py tests/test_layer_gpu.py -q -p no:cacheprovider > gpurun_out/ab7_mx.log 2>&1; echo rc=$? >> gpurun_out/ab7_mx.log
timeout 300 python tools/mxfp8_probe.py > gpurun_out/ab7_mx_probe.json 2> gpurun_out/ab7_mx_probe.err
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517"
timeout 400 $TR tools/stash_demo.py --config mixtral --layers 8 --mode plain > gpurun_out/ab7_stash_plain.json 2> gpurun_out/ab7_stash_plain.err
timeout 400 $TR tools/stash_demo.py --config mixtral --layers 8 --mode stash > gpurun_out/ab7_stash_stash.json 2> gpurun_out/ab7_stash_stash.err
tail -3 gpurun_out/ab7_mx.log; cat gpurun_out/ab7_mx_probe.json; cat gpurun_out/ab7_stash_*.json; tail -3 gpurun_out/ab7_mx_probe.err
