import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_08166_b200.at as at
at.LIB_PATH = at.PKG.parent / "dbg" / "libautotvm_b200.so"
from paper_1805_08166_b200 import synth
sp = at.Space([synth.CFG2A])
n = 151250
idx = torch.from_numpy(synth.uniform_indices(sp.size(), n, seed=1).view(np.int64)).cuda()
X = sp.features(idx)
for T, D in ((100, 6), (500, 6), (1000, 8)):
    ens = synth.ensemble(T, D)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    g.predict(X, n=n); torch.cuda.synchronize()
