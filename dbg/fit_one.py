import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_08166_b200.at as at
from paper_1805_08166_b200 import synth
sp = at.Space([synth.CFG2A])
n = int(os.environ.get("FIT_N", "1024"))
idx = torch.from_numpy(synth.uniform_indices(sp.size(), n, seed=3).view(np.int64)).cuda()
X = sp.features(idx)
c = torch.from_numpy(synth.labels(X[:, :n].T.cpu().numpy(), seed=6)).cuda()
key = torch.zeros(n, dtype=torch.int16, device="cuda")
at.gbt_fit_hist(X, n, c, key, n_trees=20, depth=6); torch.cuda.synchronize()
print("ok")
