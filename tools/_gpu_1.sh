timeout 600 python -m pytest tests/test_mxfp8.py tests/test_layer_gpu.py -q -p no:cacheprovider -x > gpurun_out/mx_pytest.log 2>&1; echo rc=$? >> gpurun_out/mx_pytest.log
timeout 300 python tools/mxfp8_probe.py > gpurun_out/mx_probe.json 2> gpurun_out/mx_probe.err
tail -30 gpurun_out/mx_pytest.log; cat gpurun_out/mx_probe.json; tail -5 gpurun_out/mx_probe.err
