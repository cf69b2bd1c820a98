# round-2 evidence: GPU tests, smoke, bench line, launch list, ncu captures of the top kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 600 python bench.py --steps 2 --warmup 1 --quick > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sa_kernel -c 1 -o gpurun_out/sa3 \
    python bench.py --steps 1 --warmup 1 --quick > gpurun_out/ncu_sa3.log 2>&1; tail -1 gpurun_out/ncu_sa3.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_forest -c 1 -o gpurun_out/ff3 \
    python bench.py --steps 1 --warmup 1 --quick > gpurun_out/ncu_ff3.log 2>&1; tail -1 gpurun_out/ncu_ff3.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/reference.json 2> gpurun_out/reference.err; cat gpurun_out/reference.json
