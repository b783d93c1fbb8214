# per-launch DRAM traffic of one step at the end of the session (roofline.traffic source)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
for cfg in mixtral qwen3 deepseek; do
  python tools/layer_step.py $cfg 4 > /dev/null 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -c 700 --csv --log-file gpurun_out/r5x_step_$cfg.csv python tools/layer_step.py $cfg 4 > gpurun_out/r5x_ncu_$cfg.log 2>&1; echo $cfg rc=$?
  python tools/step_traffic.py gpurun_out/r5x_step_$cfg.csv $cfg gpurun_out/r5x_step_traffic_$cfg.json
done
