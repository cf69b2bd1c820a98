import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_08166_b200.at as at
if os.environ.get("DBG_LIB", "1") == "1":
    at.LIB_PATH = at.PKG.parent / "dbg" / "libautotvm_b200.so"
from paper_1805_08166_b200 import synth
sp = at.Space([synth.CFG2A])
for n in (1024, 2048, 256):
    idx = torch.from_numpy(synth.uniform_indices(sp.size(), n, seed=3).view(np.int64)).cuda()
    X = sp.features(idx)
    c = torch.from_numpy(synth.labels(X[:, :n].T.cpu().numpy(), seed=6)).cuda()
    key = torch.zeros(n, dtype=torch.int16, device="cuda")
    for env in ("1", "0"):
        os.environ["AT_FIT_FUSED"] = env
        at.gbt_fit_hist(X, n, c, key, n_trees=100, depth=6); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); at.gbt_fit_hist(X, n, c, key, n_trees=100, depth=6); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"n={n} fused={env} ms={sorted(ts)[1]:.3f}", flush=True)
