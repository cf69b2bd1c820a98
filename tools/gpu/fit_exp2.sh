for nr in 2 15; do
AT_SUB_NRMAX=$nr ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fit_nr$nr.csv python tools/prof_fit.py 5 > /dev/null 2>&1
python tools/launches.py gpurun_out/fit_nr$nr.csv 2>/dev/null | head -3
AT_SUB_NRMAX=$nr timeout 600 python - <<'PY'
import sys, json, os; sys.path.insert(0, ".")
import torch, bench
from paper_1805_08166_b200 import build
build.build(); torch.cuda.set_device(0)
r = bench.other_configs(torch.device("cuda", 0), torch.cuda.current_stream(), bench._peaks())
print(os.environ.get("AT_SUB_NRMAX"), json.dumps(r["cfg4_refit"]))
PY
done
