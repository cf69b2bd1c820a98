"""Time sa_explore on config 3 (12 ResNet spaces, 1000 trees d8, 65,536 chains) or config 2 (CFG2A, 500 trees
d6, 4096 chains) for STEPS steps; prints chain-steps/s.  Env knobs (AT_SA_NBUF, AT_SA_RING) pass through."""
import json, os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_08166_b200 import at, build, synth
build.build(); torch.cuda.set_device(0)
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
C3 = int(os.environ.get("SA_CHAINS", "65536"))
if cfg == "cfg3":
    wls, T, D, C, cw = synth.ALL_RESNET, 1000, 8, C3, torch.from_numpy((np.arange(C3) % 12).astype(np.int16)).cuda()
else:
    wls, T, D, C, cw = [synth.CFG2A], 500, 6, 4096, None
sp = at.Space(wls)
ens = synth.ensemble(T, D, seed=1805)
g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
temps = torch.from_numpy(synth.temperatures(steps, synth.energy_scale(T))).cuda()
ci = torch.zeros(C, dtype=torch.int64, device="cuda")
r = at.sa_explore(sp, g, ci, temps, seed=1805, round_=0, k_out=128, init=True, chain_workload=cw, accept_bits=True)
ref_bits = r["accept_bits"].clone()
ts = []
for rep in range(3):
    ci.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = at.sa_explore(sp, g, ci, temps, seed=1805, round_=0, k_out=128, init=True, chain_workload=cw, accept_bits=True)
    b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
    assert torch.equal(r["accept_bits"], ref_bits)
ms = min(ts)
print(json.dumps({"cfg": cfg, "nbuf": os.environ.get("AT_SA_NBUF"), "ring": os.environ.get("AT_SA_RING"), "lg": os.environ.get("AT_SA_LG"), "grp": os.environ.get("AT_SA_GRP"), "np": os.environ.get("AT_SA_NP"), "eb": os.environ.get("AT_SA_EB"), "chains": C,
                  "ms": round(ms, 3), "chain_steps_per_s": round(C * (steps + 1) / ms * 1e3, 1),
                  "accept_digest": int(ref_bits.sum().item())}))
