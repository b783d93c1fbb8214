python tools/gemm_kinds.py mixtral all 10 > gpurun_out/r2d_kinds_mixtral.log 2>&1; echo kinds_rc=$?
cat gpurun_out/r2d_kinds_mixtral.log
python tools/gemm_kinds.py mixtral fc2_dgrad 1 > gpurun_out/r2d_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 4 -c 1 -o gpurun_out/r2d_fc2_dgrad python tools/gemm_kinds.py mixtral fc2_dgrad 1 > gpurun_out/r2d_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 4 -c 1 -o gpurun_out/r2d_fc1_dgrad python tools/gemm_kinds.py mixtral fc1_dgrad 1 > gpurun_out/r2d_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 4 -c 1 -o gpurun_out/r2d_fc2_fwd python tools/gemm_kinds.py mixtral fc2_fwd 1 > gpurun_out/r2d_ncu3.log 2>&1
ls -la gpurun_out/r2d_*
