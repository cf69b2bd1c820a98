"""Phase timing of the SA kernel (instrumented build, -DAT_SA_PHASE_TIMING): per-step cycles of the
proposal, feature and walk phases and, per warp, tree-wait / walk / barrier cycles (block 0)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_08166_b200 import build
lib = build.build(defines=("-DAT_SA_PHASE_TIMING",), lib=build.PKG / "libautotvm_b200_phase.so")
from paper_1805_08166_b200 import at, synth
at.LIB_PATH = lib
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
if cfg == "cfg3":
    wls, T, D, C, cw = synth.ALL_RESNET, 1000, 8, 65536, (np.arange(65536) % 12).astype(np.int16)
else:
    wls, T, D, C, cw = [synth.CFG2A], 500, 6, 4096, None
sp = at.Space(wls)
ens = synth.ensemble(T, D, seed=1805)
g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
steps = 40
temps = torch.from_numpy(synth.temperatures(steps, synth.energy_scale(T))).cuda()
ci = torch.zeros(C, dtype=torch.int64, device="cuda")
at.sa_explore(sp, g, ci, temps, seed=1805, round_=0, k_out=128, init=True,
              chain_workload=None if cw is None else torch.from_numpy(cw).cuda())
torch.cuda.synchronize()
