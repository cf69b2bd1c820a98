# Round evidence: full bench line, reference arm, per-config numbers, launch list, ncu captures.
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/reference.json 2> gpurun_out/reference.err
timeout 900 python bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err
python bench.py --steps 2 --warmup 1 --quick > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --quick > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sa_kernel -c 1 -o gpurun_out/sa \
    python bench.py --steps 1 --warmup 1 --quick > gpurun_out/ncu_sa.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_forest -c 1 -o gpurun_out/ff \
    python bench.py --steps 1 --warmup 1 --quick > gpurun_out/ncu_ff.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"predict_kernel|features_kernel" -c 4 -o gpurun_out/scoring \
    python tools/prof_scoring.py > gpurun_out/ncu_scoring.log 2>&1
ls -la gpurun_out
ncu --set full --clock-control none --import-source on -k regex:sub_hist_kernel -c 2 -o gpurun_out/subhist \
    python tools/prof_fit.py 1 > gpurun_out/ncu_subhist.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fit_launches.csv \
    python tools/prof_fit.py 5 > gpurun_out/ncu_fit.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:predict_kernel -s 1 -c 1 -o gpurun_out/pred5rk \
    python tools/prof_cfg5.py > gpurun_out/ncu_pred5rk.log 2>&1
ls -la gpurun_out
