timeout 200 python -m pytest tests/test_router_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
python tools/router_bench.py tc 2>&1 | sed 's/^/box64 /'
MOE_ROUTER_TC_DEBUG_SKIP=1 python tools/router_bench.py tc 2>&1 | sed 's/^/box64 skip /'
MOE_NVCC_EXTRA=-DMOE_ROUTER_BOX_ROWS=128 python -m paper_2603_07685_b200.build --force > /dev/null 2>&1
python tools/router_bench.py tc 2>&1 | sed 's/^/box128 /'
MOE_ROUTER_TC_DEBUG_SKIP=1 python tools/router_bench.py tc 2>&1 | sed 's/^/box128 skip /'
MOE_NVCC_EXTRA="-DMOE_ROUTER_BOX_ROWS=32" python -m paper_2603_07685_b200.build --force > /dev/null 2>&1
python tools/router_bench.py tc 2>&1 | sed 's/^/box32 /'
