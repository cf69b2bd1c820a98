# refit paths: parity tests + config-4 timing (subtraction path vs plain level-by-level)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fit or config4" > gpurun_out/pytest_fit.log 2>&1; tail -5 gpurun_out/pytest_fit.log
timeout 300 python bench_configs.py --only cfg4 > gpurun_out/cfg4_sub.json 2>&1; cat gpurun_out/cfg4_sub.json
AT_FIT_SUB=0 timeout 300 python bench_configs.py --only cfg4 > gpurun_out/cfg4_plain.json 2>&1; cat gpurun_out/cfg4_plain.json
