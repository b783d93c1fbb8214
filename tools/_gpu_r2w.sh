timeout 1500 python -m pytest tests/test_ep_loopback_gpu.py -x -q -p no:cacheprovider --timeout 600 -k "ep8 or unequal or two_ranks" 2>&1 | tail -3
