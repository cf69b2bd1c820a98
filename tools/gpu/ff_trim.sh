timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fit or algorithm or fused" 2>&1 | tail -2
for t in 0 1 0 1; do
AT_FIT_NT_TRIM=$t timeout 600 python bench.py --steps 3 --warmup 3 --quick 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('trim', $t, d['value'], d['ms_per_step'], round(d['kernel_ms']['fit_graph']/3, 3), d['topk_sha'])"
done
