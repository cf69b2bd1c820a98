set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "predict or config5 or fused_scoring or gbt or acq or concat" > gpurun_out/pytest_rank.log 2>&1; tail -3 gpurun_out/pytest_rank.log
AT_RK_GRP=4 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "predict_rank or scores_and_slots" > gpurun_out/pytest_rank2.log 2>&1; tail -3 gpurun_out/pytest_rank2.log
timeout 600 python bench_configs.py --only cfg5 > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err; cat gpurun_out/cfg5.json | cut -c1-400
AT_RK_GRP=4 timeout 600 python bench_configs.py --only cfg5 > gpurun_out/cfg5_g4.json 2> gpurun_out/cfg5_g4.err; cat gpurun_out/cfg5_g4.json | cut -c1-400
