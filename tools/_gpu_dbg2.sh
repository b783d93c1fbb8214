MOE_TEST_TIMEOUT=60 timeout 250 python -m pytest tests/test_ep_gpu.py -x -q -p no:cacheprovider -k "mem_efficient and p2p_sync_free" > gpurun_out/dbg2_me.log 2>&1; echo rc=$? >> gpurun_out/dbg2_me.log
tail -60 gpurun_out/dbg2_me.log
