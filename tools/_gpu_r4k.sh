python tools/router_bench.py gemm
python tools/router_bench.py tc
MOE_ROUTER_TC_DEBUG_SKIP=1 python tools/router_bench.py tc 2>&1 | sed 's/^/skip-selection /'
MOE_NVCC_EXTRA=-DMOE_ROUTER_RING_KB=160 python -m paper_2603_07685_b200.build --force > /dev/null 2>&1
python tools/router_bench.py tc 2>&1 | sed 's/^/ring160 /'
MOE_ROUTER_TC_DEBUG_SKIP=1 python tools/router_bench.py tc 2>&1 | sed 's/^/ring160 skip-selection /'
