for cfg in cfg3 cfg2; do
  timeout 300 python tools/sa_time.py $cfg 100 2>&1 | tail -1
done
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
