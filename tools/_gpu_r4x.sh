# raster band A/B (MOE_B200_BAND = M units per swept n-block band), grouped-M kinds
export POWER_NO_CUBLAS=1 POWER_KINDS=fc1_fwd,fc2_fwd,fc2_dgrad,fc1_dgrad
cd tools
for cfg in mixtral qwen3; do
  for b in 16 8 32 4; do echo "== $cfg band=$b"; MOE_B200_BAND=$b POWER_CONFIG=$cfg timeout 200 python power_probe.py 2>&1 | grep -v "^{" | tail -4; done
done
