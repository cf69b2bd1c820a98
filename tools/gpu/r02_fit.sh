set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rank_invariance or fit" 2>&1 | tail -5
timeout 600 python - <<'PY'
import sys, json; sys.path.insert(0, ".")
import torch, bench
from paper_1805_08166_b200 import build
build.build(); torch.cuda.set_device(0)
r = bench.other_configs(torch.device("cuda", 0), torch.cuda.current_stream(), bench._peaks())
print(json.dumps(r["cfg4_refit"]))
PY
