# ncu of the small-N router forward (Qwen3 and Mixtral shapes): text summaries only
for c in qwen3 mixtral; do
  timeout 200 ncu --set full --clock-control none --import-source on -k regex:router_tc_kernel -s 2 -c 1 -o /tmp/r4f_$c python tools/router_one.py $c 3 > gpurun_out/r4f_ncu_$c.log 2>&1
  NCU_TOP_SASS=40 python tools/ncu_summary.py /tmp/r4f_$c.ncu-rep "router_tc $c" > gpurun_out/r4f_router_$c.txt 2>&1
  head -30 gpurun_out/r4f_router_$c.txt
done
