set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sa or topk or merge or config3 or config2 or select or tune or fused_scoring or smoke or rank" > gpurun_out/pytest_topk.log 2>&1; tail -2 gpurun_out/pytest_topk.log
timeout 600 python bench_configs.py --only cfg3,cfg2a > gpurun_out/c3.json 2>&1; cat gpurun_out/c3.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python bench_configs.py --only cfg3 --steps3 100 > gpurun_out/ncu_c3.log 2>&1
