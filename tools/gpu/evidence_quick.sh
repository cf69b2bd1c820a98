# bench line + launch list + fused-forest / SA ncu captures (after a kernel change)
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 2 --warmup 1 --quick > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_forest -c 1 -o gpurun_out/ff \
    python bench.py --steps 1 --warmup 1 --quick > gpurun_out/ncu_ff.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sa_kernel -c 1 -o gpurun_out/sa \
    python bench.py --steps 1 --warmup 1 --quick > gpurun_out/ncu_sa.log 2>&1
timeout 900 python bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err
