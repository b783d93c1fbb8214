timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo bench_rc=$?
cat gpurun_out/r2f_bench.json
python bench.py --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/r2f_bench_qwen3.json 2>&1; echo q_rc=$?
python bench.py --config deepseek --steps 10 --warmup 3 --no-cpu-baseline --no-dropin > gpurun_out/r2f_bench_deepseek.json 2>&1; echo d_rc=$?
