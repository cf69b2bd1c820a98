for eb in 0 1; do AT_PRED_EB=$eb bash tools/gpu/pred_check.sh 2>&1 | head -1 | python -c "import json,sys; print($eb, json.loads(sys.stdin.read())['cfg5_sweep_1e7'])"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "predict or rank or gbt or fused or score or config5" 2>&1 | tail -2
