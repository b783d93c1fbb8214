timeout 200 python -m pytest tests/test_router_gpu.py tests/test_routing_api_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
python tools/router_bench.py tc
python tools/router_bench.py gemm
