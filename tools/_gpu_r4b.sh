# Wave-sync A/B: per-kind GEMM time, power, clock (power_probe) and DRAM bytes (ncu)
export POWER_NO_CUBLAS=1
cd tools
for cfg in mixtral qwen3; do
  for v in "0 0" "1 0" "1 64" "1 16"; do set -- $v
    echo "== $cfg sync=$1 kb=$2"
    POWER_CONFIG=$cfg MOE_B200_WAVE_SYNC=$1 MOE_B200_SYNC_KB=$2 timeout 300 python power_probe.py 2>&1 | grep -v "^{" | tail -6
  done
done
cd ..
for v in "0 0" "1 0" "1 64"; do set -- $v
  for cfg in mixtral qwen3; do
  MOE_B200_WAVE_SYNC=$1 MOE_B200_SYNC_KB=$2 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:grouped_gemm_kernel --csv python tools/gemm_kinds.py $cfg all 1 > gpurun_out/r4b_ncu_${cfg}_$1_$2.csv 2> gpurun_out/r4b_ncu_${cfg}_$1_$2.err
  done
done
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py tests/test_layer_scale_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
