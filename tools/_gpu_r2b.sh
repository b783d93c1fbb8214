timeout 1700 python -m pytest tests/test_ep_loopback_gpu.py -x -q -p no:cacheprovider --timeout 400 -rA > gpurun_out/r2b_loopback.log 2>&1; echo loopback_rc=$?
tail -40 gpurun_out/r2b_loopback.log
