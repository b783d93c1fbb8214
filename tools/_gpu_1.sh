timeout 300 python -m pytest tests/test_mxfp8.py tests/test_layer_gpu.py -q -p no:cacheprovider > gpurun_out/mx5.log 2>&1; tail -3 gpurun_out/mx5.log
python bench.py --steps 10 --no-cpu-baseline > gpurun_out/mx5_bf16.json 2> gpurun_out/mx5_bf16.err
python bench.py --steps 10 --no-cpu-baseline --precision mxfp8 > gpurun_out/mx5_mxfp8.json 2> gpurun_out/mx5_mxfp8.err
python bench.py --steps 10 --no-cpu-baseline > gpurun_out/mx5_bf16b.json 2> gpurun_out/mx5_bf16b.err
for f in mx5_bf16 mx5_mxfp8 mx5_bf16b; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'], d['ms_per_step'], {k: round(v,2) for k,v in d['kernel_ms_per_step'].items() if v > 0.3}, d['clocks']['sm_mhz'])"; done
