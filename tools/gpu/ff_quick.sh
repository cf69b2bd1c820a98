timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fit or algorithm or fused" 2>&1 | tail -2
for r in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 3 --quick 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], round(d['kernel_ms']['fit_graph']/3, 3), d['topk_sha'])"
done
timeout 600 python tools/fit_phases.py 2>&1 | grep -v ptxas | grep "level work\|ns/tree" | head -4
