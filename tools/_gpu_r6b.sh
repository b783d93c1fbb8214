# DeepSeek weight gradients: uniform vs routed counts, SK vs per-thread stores, ncu of dW1
for cnt in uniform random; do
  GEMM_KINDS_COUNTS=$cnt timeout 200 python tools/gemm_kinds.py deepseek all 10 2>&1 | grep -v "^{" | sed "s/^/$cnt /"
done
MOE_B200_WGRAD_BULK=0 GEMM_KINDS_COUNTS=random timeout 200 python tools/gemm_kinds.py deepseek fc1_wgrad 10 2>&1 | grep -v "^{" | sed "s/^/random nobulk /"
GEMM_KINDS_COUNTS=random timeout 300 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 3 -c 1 -o /tmp/r6b_w1 python tools/gemm_kinds.py deepseek fc1_wgrad 3 > gpurun_out/r6b_ncu.log 2>&1
NCU_TOP_SASS=30 python tools/ncu_summary.py /tmp/r6b_w1.ncu-rep "DeepSeek dW1 routed counts" > gpurun_out/r6b_w1.txt 2>&1
cat gpurun_out/r6b_w1.txt | head -60
