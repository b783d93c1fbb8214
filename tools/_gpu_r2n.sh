nvidia-smi topo -m | head -5
python tools/nvlink_probe.py 20 > gpurun_out/r2n_nvlink.json 2> gpurun_out/r2n_nvlink.err; echo rc=$?; cat gpurun_out/r2n_nvlink.json; tail -3 gpurun_out/r2n_nvlink.err
python tools/nvlink_probe.py 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dispatch_push|grouped_gemm" --csv --log-file gpurun_out/r2n_ncu_nvlink.csv python tools/nvlink_probe.py 1 > gpurun_out/r2n_ncu.log 2>&1; echo ncu_rc=$?
tail -2 gpurun_out/r2n_ncu.log
