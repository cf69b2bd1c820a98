timeout 600 python - <<'PY'
import sys, json; sys.path.insert(0, ".")
import torch, bench
from paper_1805_08166_b200 import build
build.build(); torch.cuda.set_device(0)
r = bench.other_configs(torch.device("cuda", 0), torch.cuda.current_stream(), bench._peaks())
r.pop("cfg4_refit", None)
print(json.dumps(r))
PY
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "predict or gbt or rank or acq or fused or score" 2>&1 | tail -2
