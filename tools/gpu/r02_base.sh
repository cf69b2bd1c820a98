# round-2 baseline: GPU tests, config 3 at 500 steps, config-3 SA ncu capture
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench_configs.py --only cfg3 --steps3 500 > gpurun_out/cfg3_500.json 2> gpurun_out/cfg3_500.err; cat gpurun_out/cfg3_500.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sa_kernel -c 1 -o gpurun_out/sa3 python bench_configs.py --only cfg3 --steps3 20 > gpurun_out/ncu_sa3.log 2>&1; tail -3 gpurun_out/ncu_sa3.log
