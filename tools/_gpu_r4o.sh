for cs in 1 2 4 8; do MOE_ROUTER_TC_CS=$cs python tools/router_bench.py tc 2>&1 | sed "s/^/cs$cs /"; done
