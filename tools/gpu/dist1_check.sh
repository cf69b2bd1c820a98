timeout 900 python bench.py --dist --steps 2 --warmup 3 --quick > gpurun_out/q_dist.json 2>/dev/null
timeout 900 python bench.py --steps 2 --warmup 3 --quick > gpurun_out/q_plain.json 2>/dev/null
python - <<'PY'
import json
a=json.load(open("gpurun_out/q_dist.json")); b=json.load(open("gpurun_out/q_plain.json"))
print("dist", a["value"], a["topk_sha"], a["gpu_launches"]); print("plain", b["value"], b["topk_sha"], b["gpu_launches"])
PY
