timeout 600 python -m pytest tests/test_bench_contract.py -q -m gpu -p no:cacheprovider 2>&1 | tail -3
