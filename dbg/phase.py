import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_08166_b200.at as at
at.LIB_PATH = at.PKG.parent / "dbg" / "libautotvm_b200.so"
from paper_1805_08166_b200 import synth
sp = at.Space([synth.CFG2A])
for T, D, nch, st in ((500, 6, 4096, 200), (128, 6, 4096, 200), (1000, 8, 4096, 50), (1000, 8, 65536, 20), (500, 6, 65536, 20)):
    ens = synth.ensemble(T, D)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    t = torch.from_numpy(synth.temperatures(st, synth.energy_scale(T))).cuda()
    ci = torch.zeros(nch, dtype=torch.int64, device="cuda")
    at.sa_explore(sp, g, ci, t, seed=1, round_=0, k_out=128, init=True); torch.cuda.synchronize()
