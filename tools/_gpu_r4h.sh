timeout 120 python -m pytest tests/test_router_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 200 python tools/router_probe.py 2>&1 | grep -v small | grep tc
for c in deepseek qwen3; do
  timeout 200 ncu --set full --clock-control none --import-source on -k regex:router_tc_kernel -s 2 -c 1 -o /tmp/r4h_$c python tools/router_one.py $c 3 > gpurun_out/r4h_ncu_$c.log 2>&1
  NCU_TOP_SASS=40 python tools/ncu_summary.py /tmp/r4h_$c.ncu-rep "router_tc $c" > gpurun_out/r4h_router_$c.txt 2>&1
  ncu -i /tmp/r4h_$c.ncu-rep --page source --csv --print-source=cuda > gpurun_out/r4h_src_$c.csv 2>&1
done
