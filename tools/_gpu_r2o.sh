M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
for cfg in mixtral qwen3 deepseek; do
python tools/layer_step.py $cfg 4 > gpurun_out/r2o_plain_$cfg.log 2>&1 && \
ncu --metrics $M --clock-control none -c 600 --csv --log-file gpurun_out/r2o_step_$cfg.csv python tools/layer_step.py $cfg 4 > gpurun_out/r2o_ncu_$cfg.log 2>&1; echo $cfg rc=$?
done
ls -la gpurun_out/r2o_*csv
