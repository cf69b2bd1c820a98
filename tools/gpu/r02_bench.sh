# bench line + launch list of the config-3 step
set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 600 python bench.py --steps 2 --warmup 1 --quick > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
