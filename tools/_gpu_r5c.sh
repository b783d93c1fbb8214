# re-run the EP layer tests at EP=4 with per-worker logs and hang stack dumps
export MOE_TEST_TIMEOUT=150 MOE_TEST_WORKER_LOG=gpurun_out/r5c_workers
timeout 2000 python -m pytest tests/test_ep_gpu.py -q -p no:cacheprovider -k "layer_matches" > gpurun_out/r5c_pytest.log 2>&1; echo rc=$?
tail -3 gpurun_out/r5c_pytest.log; grep -E "^FAILED" gpurun_out/r5c_pytest.log
for f in gpurun_out/r5c_workers/*.log; do if grep -q "Thread\|Traceback\|Error" $f; then echo "== $f"; head -60 $f; fi; done 2>/dev/null | head -150
