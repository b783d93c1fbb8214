timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 > gpurun_out/r2c_gpu.log 2>&1; echo gpu_rc=$?
tail -15 gpurun_out/r2c_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
