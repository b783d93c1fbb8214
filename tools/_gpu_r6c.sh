# DeepSeek weight gradients (routed counts): pair vs 1-CTA SK engine, raster order; alternating
export GEMM_KINDS_COUNTS=random
for rep in 1 2; do
for v in "" "MOE_B200_WGRAD_PAIR=0" "MOE_B200_GK_RASTER=nb" "MOE_B200_GK_RASTER=mu" "MOE_B200_WGRAD_PAIR=0 MOE_B200_GK_RASTER=nb"; do
  for k in fc1_wgrad fc2_wgrad; do
    env $v timeout 200 python tools/gemm_kinds.py deepseek $k 10 2>&1 | grep -v "^{" | sed "s/^/[$v] /"
  done
done
done
