for gr in 2 4; do
AT_RK_GRP=$gr timeout 600 python - <<'PY'
import os, sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_08166_b200 import at, synth
sp = at.Space(synth.ALL_RESNET); ens = synth.ensemble(2000, 8, seed=1805)
g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
n = 10_000_000
X = sp.features(torch.from_numpy(synth.sweep_indices(sp.size(), 0, n).view(np.int64)).cuda())
g.predict(X, n=n); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): g.predict(X, n=n)
b.record(); torch.cuda.synchronize()
print("RK_GRP", os.environ["AT_RK_GRP"], round(a.elapsed_time(b) / 5, 2))
PY
done
