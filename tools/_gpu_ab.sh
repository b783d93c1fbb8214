export MOE_TEST_TIMEOUT=150
timeout 400 python -m pytest tests/test_ep_gpu.py -q -p no:cacheprovider -k stash > gpurun_out/so_pytest.log 2>&1; echo rc=$? >> gpurun_out/so_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541"
timeout 400 $TR tools/stash_demo.py --config mixtral --layers 8 --mode stash_overlap > gpurun_out/so_demo_ov.json 2> gpurun_out/so_demo_ov.err
timeout 400 $TR tools/stash_demo.py --config mixtral --layers 8 --mode stash > gpurun_out/so_demo_st.json 2> gpurun_out/so_demo_st.err
tail -3 gpurun_out/so_pytest.log; cat gpurun_out/so_demo_ov.json gpurun_out/so_demo_st.json; grep -E "Error|error" gpurun_out/so_demo_ov.err | head -3
