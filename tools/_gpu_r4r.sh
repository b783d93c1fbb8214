# epilogue A/B: TMA staging (smem) vs direct per-thread global loads/stores
export POWER_NO_CUBLAS=1 POWER_KINDS=fc1_fwd,fc2_dgrad
cd tools
for cfg in mixtral qwen3; do echo "== $cfg TMA epilogues (default)"; POWER_CONFIG=$cfg timeout 200 python power_probe.py 2>&1 | grep -v "^{" | tail -2; done
cd ..; MOE_NVCC_EXTRA="-DMOE_DSWIGLU_TMA=0 -DMOE_SWIGLU_TMA=0" python -m paper_2603_07685_b200.build --force > /dev/null 2>&1; cd tools
for cfg in mixtral qwen3; do echo "== $cfg direct epilogues"; POWER_CONFIG=$cfg timeout 200 python power_probe.py 2>&1 | grep -v "^{" | tail -2; done
cd ..; MOE_NVCC_EXTRA="-DMOE_DSWIGLU_TMA=1 -DMOE_SWIGLU_TMA=0" python -m paper_2603_07685_b200.build --force > /dev/null 2>&1; cd tools
for cfg in mixtral qwen3; do echo "== $cfg swiglu direct, dswiglu TMA"; POWER_CONFIG=$cfg timeout 200 python power_probe.py 2>&1 | grep -v "^{" | tail -2; done
cd ..; MOE_NVCC_EXTRA="-DMOE_DSWIGLU_TMA=0 -DMOE_SWIGLU_TMA=1" python -m paper_2603_07685_b200.build --force > /dev/null 2>&1; cd tools
for cfg in mixtral qwen3; do echo "== $cfg swiglu TMA, dswiglu direct"; POWER_CONFIG=$cfg timeout 200 python power_probe.py 2>&1 | grep -v "^{" | tail -2; done
