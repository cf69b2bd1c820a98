set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_forest -c 1 -o gpurun_out/ff python bench.py --steps 1 --warmup 1 --quick > gpurun_out/ncu_ff.log 2>&1; tail -3 gpurun_out/ncu_ff.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sa_kernel -c 1 -o gpurun_out/sa python bench.py --steps 1 --warmup 1 --quick > gpurun_out/ncu_sa.log 2>&1; tail -3 gpurun_out/ncu_sa.log
