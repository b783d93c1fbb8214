# Final full GPU suite on a 4-GPU box with the end-of-session code (EP tests at every
# visible GPU), per-rank worker logs
export MOE_TEST_TIMEOUT=200
nvidia-smi --query-gpu=index,name --format=csv
MOE_TEST_WORKER_LOG=gpurun_out/fin8_workers timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin8_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/fin8_pytest.log
tail -3 gpurun_out/fin8_pytest.log; grep -E "^FAILED" gpurun_out/fin8_pytest.log | head
