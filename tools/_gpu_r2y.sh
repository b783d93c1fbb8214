timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
echo "== raster auto"; python tools/gemm_kinds.py mixtral fc2_wgrad 10 | grep -v "^{"; python tools/gemm_kinds.py qwen3 fc1_wgrad 10 | grep -v "^{"
echo "== raster nb"; MOE_B200_GK_RASTER=nb python tools/gemm_kinds.py mixtral fc2_wgrad 10 | grep -v "^{"; MOE_B200_GK_RASTER=nb python tools/gemm_kinds.py qwen3 fc1_wgrad 10 | grep -v "^{"
python tools/gemm_kinds.py mixtral fc2_wgrad 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:grouped_gemm_kernel -s 4 -c 1 --csv python tools/gemm_kinds.py mixtral fc2_wgrad 1 2>/dev/null | grep -E "dram|duration" | cut -d, -f13-15
cd tools && python power_probe.py 2>&1 | grep -v "^{" | tail -8
