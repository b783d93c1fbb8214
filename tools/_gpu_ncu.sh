python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pre1.json 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 1 -c 1 -o gpurun_out/ncu_fc1_pair python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_fc1_pair.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 4 -c 1 -o gpurun_out/ncu_wgrad_pair python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_wgrad_pair.log 2>&1
ls -la gpurun_out/ncu_*pair*
