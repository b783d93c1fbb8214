timeout 200 python -m pytest tests/test_router_gpu.py tests/test_routing_api_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
python tools/router_bench.py tc
MOE_ROUTER_TC_DEBUG_SKIP=1 python tools/router_bench.py tc 2>&1 | sed 's/^/skip-selection /'
