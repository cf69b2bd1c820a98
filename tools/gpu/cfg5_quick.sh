set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_scoring or config5" > gpurun_out/pytest_c5.log 2>&1; tail -3 gpurun_out/pytest_c5.log
timeout 900 python bench_configs.py --only cfg5 > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err; cat gpurun_out/cfg5.json; tail -3 gpurun_out/cfg5.err
