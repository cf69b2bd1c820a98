# A/B of gbt_predict (config 5 rank form at 10^7, config-2 fp32 at 2^20) and the config-3 SA: alt vs current
for lib in alt "" alt ""; do
L=paper_1805_08166_b200/libautotvm_b200${lib:+_$lib}.so
AT_LIB=$L timeout 600 python - <<'PY'
import os, sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_08166_b200 import at, synth
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
sp = at.Space(synth.ALL_RESNET); ens = synth.ensemble(2000, 8, seed=1805)
g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
n = 10_000_000
X = sp.features(torch.from_numpy(synth.sweep_indices(sp.size(), 0, n).view(np.int64)).cuda())
m5 = t(lambda: g.predict(X, n=n))
del X
sp2 = at.Space([synth.CFG2A]); e2 = synth.ensemble(500, 6, seed=1805)
g2 = at.Gbt(e2["feat"], e2["thresh"], e2["leaf"])
n2 = 1 << 20
X2 = sp2.features(torch.from_numpy(synth.uniform_indices(sp2.size(), n2, seed=3).view(np.int64)).cuda())
m2 = t(lambda: g2.predict(X2, n=n2), reps=20)
print(os.environ["AT_LIB"][-10:], "cfg5 predict ms", round(m5, 2), "cfg2 predict ms", round(m2, 4))
PY
AT_LIB=$L timeout 600 python tools/sa_time.py cfg3 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sa', d['ms'], d['accept_digest'])"
done
