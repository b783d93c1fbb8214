python tools/gemm_kinds.py deepseek all 10 2>&1 | grep -v "^{"
python tools/gemm_kinds.py deepseek fc1_wgrad 1 > gpurun_out/r2i_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 4 -c 1 -o gpurun_out/r2i_ds_fc1_wgrad python tools/gemm_kinds.py deepseek fc1_wgrad 1 > gpurun_out/r2i_ncu.log 2>&1
tail -3 gpurun_out/r2i_ncu.log
