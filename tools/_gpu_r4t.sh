timeout 300 python -m pytest tests/test_router_gpu.py tests/test_routing_api_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
python tools/router_bench.py tc 2>&1 | sed 's/^/subk2 /'
MOE_ROUTER_TC_DEBUG_SKIP=1 python tools/router_bench.py tc 2>&1 | sed 's/^/subk2 skip /'
MOE_NVCC_EXTRA=-DMOE_ROUTER_SUBK=4 python -m paper_2603_07685_b200.build --force > /dev/null 2>&1
python tools/router_bench.py tc 2>&1 | sed 's/^/subk4 /'
MOE_NVCC_EXTRA=-DMOE_ROUTER_SUBK=1 python -m paper_2603_07685_b200.build --force > /dev/null 2>&1
python tools/router_bench.py tc 2>&1 | sed 's/^/subk1 /'
