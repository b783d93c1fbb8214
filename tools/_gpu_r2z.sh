cd tools
for b in 4 8 16 32; do echo "== band $b"; MOE_B200_BAND=$b POWER_NO_CUBLAS=1 POWER_KINDS=fc1_dgrad,fc2_fwd,fc1_fwd,fc2_dgrad python power_probe.py 2>&1 | grep -v "^{" | tail -4; done
