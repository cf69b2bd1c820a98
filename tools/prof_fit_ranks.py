"""Per-class kernel time of the config-4 refit through the multi-rank subtraction path, rank 0's share at
R = 1, 2, 4, 8 (the exchange replaced by a no-op: compute only), from the library's CUDA-event profiler."""
import json, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_08166_b200 import at, build, synth, dist as D
build.build(); torch.cuda.set_device(0)
n = 100000
sp = at.Space(synth.ALL_DW)
key = synth.group_keys(n, 9, seed=4)
sizes = np.array([sp.size(w) for w in range(9)], dtype=np.uint64)
loc = synth.uniform_indices(1 << 62, n, seed=5) % sizes[key]
idx = torch.from_numpy((loc + np.array(sp.offsets[:9], dtype=np.uint64)[key]).view(np.int64)).cuda()
X = sp.features(idx)
cost = torch.from_numpy(synth.labels(X[:, :n].T.cpu().numpy(), seed=6)).cuda()
kg = torch.from_numpy(key.view(np.int16)).cuda()
out = {}
for R in (1, 2, 4, 8):
    hr = D.sample_slice(n, 0, R)
    at.gbt_fit_hist(X, n, cost, kg, n_trees=10, depth=6, hist_range=hr, allreduce=lambda t: None)
    torch.cuda.synchronize()
    at.prof_reset(); at.prof_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    at.gbt_fit_hist(X, n, cost, kg, n_trees=100, depth=6, hist_range=hr, allreduce=lambda t: None)
    e1.record(); torch.cuda.synchronize()
    at.prof_enable(False)
    out[R] = {"wall_ms": round(e0.elapsed_time(e1), 2), **{k: round(at.prof_query(k)[1], 2) for k in at.AT_K if at.prof_query(k)[0]}}
print(json.dumps(out))
