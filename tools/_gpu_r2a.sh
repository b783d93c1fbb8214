set -x
nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests/test_layer_scale_gpu.py tests/test_layer_gpu.py -x -q -s -p no:cacheprovider > gpurun_out/r2a_scale.log 2>&1; echo scale_rc=$?
tail -30 gpurun_out/r2a_scale.log
tail -3 gpurun_out/r2a_smoke.log
