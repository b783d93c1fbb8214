timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r2t_bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'], d['roofline']['frac_vs']); print(d['kernel_ms_per_step']); print(d['hbm_kernels']); print(d.get('dropin')); print(d['cpu_baseline'])"
python bench.py --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/r2t_bench_qwen3.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r2t_bench_qwen3.json')); print('qwen3', d['value'], d['ms_per_step'], d['clocks']['sm_mhz']); print(d['kernel_ms_per_step']); print(d['hbm_kernels'])"
