timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider -o faulthandler_timeout=300 2>&1 | tail -2
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
