timeout 120 python -m pytest tests/test_router_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
python tools/router_bench.py tc
timeout 300 python tools/hbm_probe.py 2>&1 | tail -16
