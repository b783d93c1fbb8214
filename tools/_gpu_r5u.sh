# the reference's own test suite / moe-check on the B200 drop-in, with the end-of-round code
timeout 900 python tools/run_reference_suite.py > gpurun_out/r5u_refsuite.log 2>&1; echo rc=$?
grep -E "passed|failed" gpurun_out/r5u_refsuite.log | tail -3
tail -12 gpurun_out/r5u_refsuite.log
