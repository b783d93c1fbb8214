timeout 200 python -m pytest tests/test_router_gpu.py tests/test_routing_api_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 200 python tools/router_probe.py 2>&1 | grep -v small | grep tc
for c in deepseek qwen3; do
  timeout 200 ncu --set full --clock-control none --import-source on -k regex:router_tc_kernel -s 2 -c 1 -o /tmp/r4i_$c python tools/router_one.py $c 3 > gpurun_out/r4i_ncu_$c.log 2>&1
  NCU_TOP_SASS=30 python tools/ncu_summary.py /tmp/r4i_$c.ncu-rep "router_tc $c" > gpurun_out/r4i_router_$c.txt 2>&1
  grep -E "duration|dram_thr|issue_slots|warp-stall" gpurun_out/r4i_router_$c.txt
done
