"""One config-4 refit (10^5 samples over the 9 MobileNet depthwise spaces) for ncu launch lists:
python tools/prof_fit.py [trees]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08166_b200 import at, build, synth  # noqa: E402

build.build()
trees = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = 100000
sp = at.Space(synth.ALL_DW)
key = synth.group_keys(n, 9, seed=4)
sizes = np.array([sp.size(w) for w in range(9)], dtype=np.uint64)
loc = synth.uniform_indices(1 << 62, n, seed=5) % sizes[key]
idx = torch.from_numpy((loc + np.array(sp.offsets[:9], dtype=np.uint64)[key]).view(np.int64)).cuda()
X = sp.features(idx)
cost = torch.from_numpy(synth.labels(X[:, :n].T.cpu().numpy(), seed=6)).cuda()
kg = torch.from_numpy(key.view(np.int16)).cuda()
at.gbt_fit_hist(X, n, cost, kg, n_trees=trees, depth=6)
torch.cuda.synchronize()
print("ok")
