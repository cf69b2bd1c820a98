#!/usr/bin/env python
"""Algorithm 1 against random search on a synthetic cost (the qualitative claim of
P:356-361: the model-guided search finds better schedules than random search for the same number
of measurements).

The "hardware" is a fixed synthetic cost over the config-2 conv2d space: a random log-linear model
of the schedule's loop-context features (paper_1805_08166_b200.synth.labels) -- a stand-in for
f(g(e, s)) of P:63, not a model of any real GPU.  Both searches get the same trial budget.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08166_b200 import at, build, synth  # noqa: E402
from paper_1805_08166_b200.tune import TuneConfig, Tuner  # noqa: E402


def main(budget=512, seeds=(1, 2, 3)):
    build.build()
    wl = synth.CFG2A
    sp = at.Space([wl])
    # a fixed synthetic cost: labels() of the GPU features, one draw per configuration (seeded by idx)
    def cost(idx):
        idx = np.asarray(idx, dtype=np.uint64)
        X = sp.features(torch.from_numpy(idx.view(np.int64)).cuda())[:, :len(idx)].T.cpu().numpy()
        base = synth.labels(X, seed=2024)             # random log-linear model of the features
        noise = np.array([np.random.default_rng(int(i)).normal(0, 0.05) for i in idx])
        return (base * np.exp(noise)).astype(np.float32)

    out = {"budget": budget, "space": int(sp.size()), "tuner": [], "random": []}
    for seed in seeds:
        ens0 = synth.ensemble(100, 6, seed=seed)      # untrained initial energy (no history)
        cfg = TuneConfig(n_chains=128, n_steps=500, b=64, seed=seed)
        t = Tuner(wl, at.Gbt(ens0["feat"], ens0["thresh"], ens0["leaf"]), cost, cfg)
        best_idx, best = t.run(budget)
        curve = np.minimum.accumulate(np.array(t.state.costs)).tolist()
        rnd = cost(synth.uniform_indices(sp.size(), budget, seed=1000 + seed))
        out["tuner"].append({"seed": seed, "best": best, "best_at": [curve[i - 1] for i in (64, 128, 256, budget)]})
        rc = np.minimum.accumulate(rnd)
        out["random"].append({"seed": seed, "best": float(rc[-1]), "best_at": [float(rc[i - 1]) for i in (64, 128, 256, budget)]})
    out["tuner_median_best"] = float(np.median([r["best"] for r in out["tuner"]]))
    out["random_median_best"] = float(np.median([r["best"] for r in out["random"]]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
