# EP=4 test file again with per-rank logs and hang stack dumps (flakiness check)
export MOE_TEST_TIMEOUT=150 MOE_TEST_WORKER_LOG=gpurun_out/r5v_workers
timeout 2400 python -m pytest tests/test_ep_gpu.py -q -p no:cacheprovider -rw > gpurun_out/r5v_pytest.log 2>&1; echo rc=$?
tail -4 gpurun_out/r5v_pytest.log; grep -E "^FAILED|retrying" gpurun_out/r5v_pytest.log | head
for f in gpurun_out/r5v_workers/*.log; do if grep -q "Thread 0x\|Current thread" $f; then echo "== $f"; grep -A25 "Current thread\|Thread 0x" $f | head -40; fi; done 2>/dev/null | head -120
