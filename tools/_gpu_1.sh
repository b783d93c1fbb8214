timeout 300 python -m pytest tests/test_layer_gpu.py -q -p no:cacheprovider -k mxfp8 > gpurun_out/mx3.log 2>&1; tail -2 gpurun_out/mx3.log
python bench.py --steps 10 --no-cpu-baseline > gpurun_out/mx3_bf16.json 2> gpurun_out/mx3_bf16.err
python bench.py --steps 10 --no-cpu-baseline --precision mxfp8 > gpurun_out/mx3_mxfp8.json 2> gpurun_out/mx3_mxfp8.err
python bench.py --steps 10 --no-cpu-baseline > gpurun_out/mx3_bf16b.json 2> gpurun_out/mx3_bf16b.err
for f in mx3_bf16 mx3_mxfp8 mx3_bf16b; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d['value'], d['ms_per_step'], d['clocks'])"; done
