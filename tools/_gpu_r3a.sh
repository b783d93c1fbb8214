python tools/gemm_kinds.py mixtral fc2_dgrad 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 4 -c 1 -o gpurun_out/r3a_fc2_dgrad python tools/gemm_kinds.py mixtral fc2_dgrad 1 > gpurun_out/r3a_ncu.log 2>&1
python tools/gemm_kinds.py mixtral fc1_dgrad 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 4 -c 1 -o gpurun_out/r3a_fc1_dgrad python tools/gemm_kinds.py mixtral fc1_dgrad 1 > gpurun_out/r3a_ncu2.log 2>&1
tail -1 gpurun_out/r3a_ncu.log
