timeout 600 python -m pytest tests/test_layer_gpu.py tests/test_routing_api_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
echo "== chunk gather"; python tools/hbm_probe.py 20 | grep gather
echo "== token gather"; MOE_B200_GATHER=token python tools/hbm_probe.py 20 | grep gather
echo "== tma gather"; MOE_B200_GATHER=tma python tools/hbm_probe.py 20 | grep gather
