export MOE_TEST_TIMEOUT=120
timeout 1200 python -m pytest tests/test_ep_gpu.py -q -p no:cacheprovider -k "p2p and not pull and not dedup" > gpurun_out/ab5_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/ab5_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517"
timeout 400 $TR tools/stash_demo.py --config mixtral --layers 8 --mode plain > gpurun_out/ab5_stash_plain.json 2> gpurun_out/ab5_stash_plain.err
timeout 400 $TR tools/stash_demo.py --config mixtral --layers 8 --mode stash > gpurun_out/ab5_stash_stash.json 2> gpurun_out/ab5_stash_stash.err
timeout 400 $TR tools/stash_demo.py --config mixtral --layers 2 --mode both --steps 1 > gpurun_out/ab5_stash_both.json 2> gpurun_out/ab5_stash_both.err
tail -3 gpurun_out/ab5_pytest.log; cat gpurun_out/ab5_stash_*.json
