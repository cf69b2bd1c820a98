# A/B of the config-5 sweep: current library vs AT_LIB=libautotvm_b200_alt.so
for lib in paper_1805_08166_b200/libautotvm_b200_alt.so paper_1805_08166_b200/libautotvm_b200.so paper_1805_08166_b200/libautotvm_b200_alt.so paper_1805_08166_b200/libautotvm_b200.so; do
AT_LIB=$lib timeout 600 python - <<'PY'
import os, sys, json; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_08166_b200 import at, synth
sp = at.Space(synth.ALL_RESNET); ens = synth.ensemble(2000, 8, seed=1805)
g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
n = 10_000_000
idx = torch.from_numpy(synth.sweep_indices(sp.size(), 0, n).view(np.int64)).cuda()
X = sp.features(idx); torch.cuda.synchronize()
for _ in range(2): g.predict(X, n=n)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): g.predict(X, n=n)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(os.environ["AT_LIB"][-10:], "predict 1e7 ms", round(ms, 2), "cand/s", round(n / ms * 1e3 / 1e6, 1), "M")
PY
done
