"""Small driver for ncu captures of the scoring kernels: features_extract + gbt_predict on the
config-1 space (all 151,250 schedules, 100 trees d6) and 2^20 config-2 candidates (500 trees d6)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08166_b200 import at, build, synth  # noqa: E402

build.build()
for wl, T, n in ((synth.MATMUL_512, 100, 151250), (synth.CFG2A, 500, 1 << 20)):
    sp = at.Space([wl])
    ens = synth.ensemble(T, 6, seed=1805)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    idx = np.arange(n, dtype=np.uint64) if n == sp.size() else synth.uniform_indices(sp.size(), n, seed=7)
    idx = torch.from_numpy(idx.view(np.int64)).cuda()
    X = sp.features(idx)
    s = g.predict(X, n=n)
    torch.cuda.synchronize()
print("ok")
