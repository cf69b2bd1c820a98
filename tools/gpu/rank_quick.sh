set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "predict or config5 or fused_scoring or gbt or acq or concat" > gpurun_out/pytest_rank.log 2>&1; tail -3 gpurun_out/pytest_rank.log
timeout 600 python bench_configs.py --only cfg5 > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err; cat gpurun_out/cfg5.json; tail -3 gpurun_out/cfg5.err
ncu --set full --clock-control none --import-source on -k regex:predict_kernel -s 1 -c 1 -o gpurun_out/pred5rk python tools/prof_cfg5.py > gpurun_out/ncu_pred5rk.log 2>&1
