# refit subtraction path: parity, config-4 timing, launch list of a 5-tree fit
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fit or config4" > gpurun_out/pytest_fit.log 2>&1; tail -5 gpurun_out/pytest_fit.log
timeout 300 python bench_configs.py --only cfg4 > gpurun_out/cfg4_sub.json 2>&1; cat gpurun_out/cfg4_sub.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fit_launches.csv python tools/prof_fit.py 5 > gpurun_out/ncu_fit.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sub_hist_kernel -c 2 -o gpurun_out/subhist python tools/prof_fit.py 1 > gpurun_out/ncu_subhist.log 2>&1
