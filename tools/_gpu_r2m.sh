timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_layer_scale_gpu.py -x -q -p no:cacheprovider -k "wgrad or deepseek or fc" 2>&1 | tail -2
for it in 1 10; do python tools/gemm_kinds.py deepseek fc1_wgrad $it 2>&1 | grep -v "^{"; python tools/gemm_kinds.py deepseek fc2_wgrad $it 2>&1 | grep -v "^{"; done
python bench.py --config deepseek --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/r2m_ds.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r2m_ds.json')); print(d['value'], d['ms_per_step'], d['clocks']['sm_mhz']); print(d['kernel_ms_per_step'])"
