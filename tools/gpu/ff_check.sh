timeout 600 python bench.py --steps 2 --warmup 1 --quick > gpurun_out/plain.log 2>&1; python -c "import json; d=json.load(open('gpurun_out/plain.log')); print(d['value'], d['kernel_ms'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fit" 2>&1 | tail -2
