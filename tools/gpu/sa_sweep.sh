timeout 300 python tools/sa_time.py cfg3 100 2>&1 | tail -1
timeout 300 python tools/sa_time.py cfg2 100 2>&1 | tail -1
SA_CHAINS=8192 timeout 300 python tools/sa_time.py cfg3 100 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sa or fused or algorithm or rank_split or config3" 2>&1 | tail -2
