timeout 600 python -m pytest tests/test_router_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -15
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r2g_bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz']); print(d['kernel_ms_per_step'])"
python bench.py --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/r2g_bench_qwen3.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r2g_bench_qwen3.json')); print(d['value'], d['ms_per_step'], d['clocks']['sm_mhz']); print(d['kernel_ms_per_step'])"
