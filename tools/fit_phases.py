"""Phase timing of the fused forest (instrumented build, -DAT_FIT_TIMING): ns per tree of the gradient
phase, its grid sync, the levels' block work and syncs, the leaves (block 0) -- config 3's |D| = 1536
(12 workloads) and config 2's |D| = 1024."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_08166_b200 import build
lib = build.build(defines=("-DAT_FIT_TIMING",), lib=build.PKG / "libautotvm_b200_fittime.so")
from paper_1805_08166_b200 import at, synth
at.LIB_PATH = lib
for name, wls, nper in (("cfg3", synth.ALL_RESNET, 128), ("cfg2", [synth.CFG2A], 1024)):
    sp = at.Space(wls)
    nw = len(wls)
    n = nw * nper if nw > 1 else nper
    key = (np.arange(n) % nw).astype(np.uint16)
    sizes = np.array([sp.size(w) for w in range(nw)], dtype=np.uint64)
    loc = synth.uniform_indices(1 << 62, n, seed=1806) % sizes[key]
    idx = loc + np.array(sp.offsets[:nw], dtype=np.uint64)[key]
    X = sp.features(torch.from_numpy(idx.view(np.int64)).cuda())
    c = torch.from_numpy(synth.labels(X[:, :n].T.cpu().numpy(), seed=1807)).cuda()
    k = torch.from_numpy(key.view(np.int16)).cuda()
    print(name, n, flush=True)
    at.gbt_fit_hist(X, n, c, k, n_trees=100, depth=6)
    torch.cuda.synchronize()
