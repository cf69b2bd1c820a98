"""Config-5 scoring (2^16 sweep candidates over the 12 ResNet spaces, 2000 trees depth 8) for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08166_b200 import at, build, synth  # noqa: E402

build.build()
sp = at.Space(synth.ALL_RESNET)
ens = synth.ensemble(2000, 8, seed=1805)
g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
n = 1 << 20
idx = torch.from_numpy(synth.sweep_indices(sp.size(), 0, n).view(np.int64)).cuda()
X = sp.features(idx)
for _ in range(2):
    s = g.predict(X, n=n)
torch.cuda.synchronize()
print("ok")
