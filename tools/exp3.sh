timeout 900 python -m pytest tests/test_gpu_comm_one_rank.py -q -x -p no:cacheprovider 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "solve or lookahead or reduce" 2>&1 | tail -3
