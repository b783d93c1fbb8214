timeout 600 python -m pytest tests/test_layer_gpu.py tests/test_routing_api_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
echo "== TMA gather"; python tools/hbm_probe.py 20
echo "== SIMT gather"; MOE_B200_GATHER_TMA=0 python tools/hbm_probe.py 20 | grep gather
