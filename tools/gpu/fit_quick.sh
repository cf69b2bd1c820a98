# fit parity tests + bench step breakdown (quick)
timeout 600 python -m pytest tests -m gpu -x -q -k "fit or algorithm1 or config4" 2>&1 | tail -15
timeout 300 python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], {k: round(v/3,3) for k,v in d['kernel_ms'].items()})"
AT_FIT_FUSED=2 timeout 300 python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v2', d['value'], d['ms_per_step'], {k: round(v/3,3) for k,v in d['kernel_ms'].items()})"
