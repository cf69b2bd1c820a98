"""A small pass over every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
features, streamed + resident + rank-form predict, SA (1 and 2 groups, measured drop over several
rounds), top-k merge, select, the fused-forest / subtraction / level-by-level refits (incl. the grid
barrier and the 128-bit CAS), bootstrap, acquisition.  Sizes are tiny; the point is the checkers."""
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_08166_b200 import at, build, synth
build.build(); torch.cuda.set_device(0)
u64 = lambda a: torch.from_numpy(np.asarray(a, dtype=np.uint64).view(np.int64)).cuda()
sp = at.Space([synth.CFG2A])
ens = synth.ensemble(300, 6, seed=1)                      # streamed (2 chunks+), GRP = 1
g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
idx = u64(synth.uniform_indices(sp.size(), 700, seed=2))
X = sp.features(idx)
s = g.predict(X, n=700, slots=True)
small = synth.ensemble(20, 4, seed=3)                     # resident
gs = at.Gbt(small["feat"], small["thresh"], small["leaf"])
gs.predict(X, n=700)
deep = synth.ensemble(40, 8, seed=4)                      # depth 8: rank form
gd = at.Gbt(deep["feat"], deep["thresh"], deep["leaf"])
gd.predict(X, n=700)
temps = torch.from_numpy(synth.temperatures(6, 0.3)).cuda()
ci = torch.zeros(64, dtype=torch.int64, device="cuda")
r = at.sa_explore(sp, g, ci, temps, seed=1, round_=0, k_out=32, init=True, accept_bits=True)
r = at.sa_explore(sp, g, ci, temps, seed=1, round_=1, k_out=32, measured=torch.sort(r["out_idx"][0][:20])[0])
spu = at.Space(synth.ALL_RESNET[:3])
cw = torch.from_numpy((np.arange(96) % 3).astype(np.int16)).cuda()
r3 = at.sa_explore(spu, gd, torch.zeros(96, dtype=torch.int64, device="cuda"), temps, seed=2, round_=0, k_out=16,
                   chain_workload=cw, init=True)
mi, ms, mn = at.topk_merge(spu, r3["out_idx"][None].repeat(2, 1, 1).contiguous(), r3["out_score"][None].repeat(2, 1, 1).contiguous(),
                           r3["out_n"][None].repeat(2, 1).contiguous(), 16)
at.select_topk(sp, 0, r["out_idx"][0], r["out_score"][0], b=16, eps=0.25, alpha=0.1, seed=3, round_=0)
c = torch.from_numpy(synth.labels(X[:, :700].T.cpu().numpy(), seed=5)).cuda()
key = torch.zeros(700, dtype=torch.int16, device="cuda")
at.gbt_fit_hist(X, 700, c, key, n_trees=3, depth=5)                               # fused forest
os.environ["AT_FIT_FUSED"] = "0"
idx2 = u64(synth.uniform_indices(sp.size(), 2500, seed=6))
X2 = sp.features(idx2)
c2 = torch.from_numpy(synth.labels(X2[:, :2500].T.cpu().numpy(), seed=7)).cuda()
k2 = torch.zeros(2500, dtype=torch.int16, device="cuda")
at.gbt_fit_hist(X2, 2500, c2, k2, n_trees=2, depth=5)                              # subtraction path
os.environ["AT_FIT_SUB"] = "0"
at.gbt_fit_hist(X2, 2500, c2, k2, n_trees=2, depth=4)                              # level-by-level
Xb, cb, kb, _ = at.bootstrap_resample(X, 700, c, key, 1)
g.concat(gs).predict_acq(X, 700, 1, kind="ucb")
torch.cuda.synchronize()
sp.check()
print("sanitize run ok, launches:", at.launch_count(), "library:", at.LIB_PATH.name)
