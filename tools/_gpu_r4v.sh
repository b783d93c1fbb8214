# refresh the per-launch DRAM traffic of one step (roofline.traffic source) + full ncu of
# the two epilogue-heavy GEMMs (text summaries only)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
for cfg in mixtral qwen3 deepseek; do
  python tools/layer_step.py $cfg 4 > gpurun_out/r4v_plain_$cfg.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -c 600 --csv --log-file gpurun_out/r4v_step_$cfg.csv python tools/layer_step.py $cfg 4 > gpurun_out/r4v_ncu_$cfg.log 2>&1; echo $cfg rc=$?
  python tools/step_traffic.py gpurun_out/r4v_step_$cfg.csv $cfg gpurun_out/r4v_step_traffic_$cfg.json > /dev/null 2>&1; echo traffic rc=$?
done
for k in fc2_dgrad fc1_fwd; do
  python tools/gemm_kinds.py mixtral $k 1 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_kernel -s 4 -c 1 -o /tmp/r4v_$k python tools/gemm_kinds.py mixtral $k 1 > gpurun_out/r4v_ncu_$k.log 2>&1
  NCU_TOP_SASS=30 python tools/ncu_summary.py /tmp/r4v_$k.ncu-rep "Mixtral $k (round-2 final kernels)" > gpurun_out/r4v_ncu_$k.txt 2>&1
  head -16 gpurun_out/r4v_ncu_$k.txt
done
