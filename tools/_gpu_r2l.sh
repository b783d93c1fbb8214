for it in 1 3 10; do python tools/gemm_kinds.py deepseek fc1_wgrad $it 2>&1 | grep -v "^{"; done
for it in 1 10; do python tools/gemm_kinds.py deepseek fc2_wgrad $it 2>&1 | grep -v "^{"; done
nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu --format=csv
