# end-of-round ncu (full) of the weight gradient (dW1, the largest launch of the step) and
# the wave-synced fc1 data-gradient, Mixtral shape; text summaries only
for k in fc1_wgrad fc1_dgrad fc2_fwd; do
  python tools/gemm_kinds.py mixtral $k 1 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 4 -c 1 -o /tmp/r5n_$k python tools/gemm_kinds.py mixtral $k 1 > gpurun_out/r5n_ncu_$k.log 2>&1
  NCU_TOP_SASS=20 python tools/ncu_summary.py /tmp/r5n_$k.ncu-rep "Mixtral $k (end of round 2)" > gpurun_out/r5n_ncu_$k.txt 2>&1
  head -16 gpurun_out/r5n_ncu_$k.txt
done
