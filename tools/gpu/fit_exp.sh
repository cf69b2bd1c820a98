set -x
for lib in paper_1805_08166_b200/libautotvm_b200_old.so paper_1805_08166_b200/libautotvm_b200.so; do
for r in 290 400 ; do
AT_LIB=$lib AT_SUB_ROWS=$r timeout 600 python - <<'PY'
import sys, json, os; sys.path.insert(0, ".")
import torch, bench
from paper_1805_08166_b200 import build
build.build(); torch.cuda.set_device(0)
r = bench.other_configs(torch.device("cuda", 0), torch.cuda.current_stream(), bench._peaks())
print(os.environ.get("AT_LIB")[-12:], os.environ.get("AT_SUB_ROWS"), json.dumps(r["cfg4_refit"]))
PY
done
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fit_new.csv python tools/prof_fit.py 5 > /dev/null 2>&1
python tools/launches.py gpurun_out/fit_new.csv 2>/dev/null | head -14
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rank_invariance or fit" 2>&1 | tail -3
