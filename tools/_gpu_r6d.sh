# DeepSeek dW1 / dW2 (routed counts): component costs of the SK weight-gradient engine
export GEMM_KINDS_COUNTS=random
for rep in 1 2; do
for d in 0 1 2 4 5 6; do
  for k in fc1_wgrad fc2_wgrad; do
    MOE_B200_DEBUG_SKIP=$d timeout 200 python tools/gemm_kinds.py deepseek $k 10 2>&1 | grep -v "^{" | sed "s/^/[skip $d] /"
  done
done
done
