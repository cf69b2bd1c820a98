"""Algorithm 1 of the paper driven over the C-ABI: the model-guided tuning loop.

    D <- {}
    while n_trials < max_n_trials:
        Q <- parallel SA over S_e with energy f-hat                  (sa_explore)
        S <- greedy Eq. 3 (1 - eps) b from the top lambda b  + eps b random  (select_topk)
        for s in S: c <- f(g(e, s)); D <- D U {(e, s, c)}            (measure: caller-supplied f)
        update f-hat using D                                         (gbt_fit_hist, Eq. 2)
    s* <- history best

Chains persist across rounds.  Before the first refit f-hat is the caller's initial model
(e.g. a transferred / synthetic ensemble).  The measurement f is a callable on global indices that
returns costs (the hardware run of P:63); features of the measured configurations come from
features_extract.  Everything numeric runs in the library's kernels; this module only sequences
the calls and keeps the database.  Single GPU (the multi-GPU pieces are in dist.py / bench.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class TuneConfig:
    n_chains: int = 128          # n_sa
    n_steps: int = 500           # step_sa
    b: int = 64                  # b_GBT
    lam: int = 2                 # pool = lam * b (reading Q24)
    eps: float = 0.05
    alpha: float = 0.1           # reading Q24
    n_trees: int = 100           # refit (reading Q16)
    depth: int = 6
    t_ratio: float = 0.05        # geometric temperature schedule T0 -> t_ratio T0 (reading Q21)
    seed: int = 1805


@dataclass
class TuneState:
    chain_idx: object = None                      # device int64 [n_chains], persistent
    measured: list = field(default_factory=list)  # global indices in measurement order
    costs: list = field(default_factory=list)
    best_idx: int = -1
    best_cost: float = float("inf")
    history: list = field(default_factory=list)   # per round: (selected, costs)


class Tuner:
    def __init__(self, workload: dict, model, measure, cfg: TuneConfig = TuneConfig()):
        import torch

        from . import at
        self.at = at
        self.torch = torch
        self.space = at.Space([workload])
        self.model = model
        self.measure = measure
        self.cfg = cfg
        self.state = TuneState(chain_idx=torch.zeros(cfg.n_chains, dtype=torch.int64, device="cuda"))
        self.round = 0

    def _temps(self):
        import torch
        from .synth import energy_scale, temperatures
        t0 = energy_scale(self.model.n_trees)
        return torch.from_numpy(temperatures(self.cfg.n_steps, t0, self.cfg.t_ratio)).cuda()

    def step(self):
        """One iteration of Algorithm 1; returns the selected global indices (numpy u64)."""
        at, torch, cfg, st = self.at, self.torch, self.cfg, self.state
        meas = None
        if st.measured:
            meas = torch.from_numpy(np.sort(np.array(st.measured, dtype=np.uint64)).view(np.int64)).cuda()
        res = at.sa_explore(self.space, self.model, st.chain_idx, self._temps(), seed=cfg.seed, round_=self.round,
                            k_out=cfg.lam * cfg.b, measured=meas, init=self.round == 0)
        n_pool = int(res["out_n"][0])
        sel, n_sel = at.select_topk(self.space, 0, res["out_idx"][0, :n_pool].contiguous(),
                                    res["out_score"][0, :n_pool].contiguous(), b=cfg.b, eps=cfg.eps,
                                    alpha=cfg.alpha, seed=cfg.seed, round_=self.round, measured=meas)
        selected = sel[:int(n_sel)].cpu().numpy().view(np.uint64).copy()
        costs = np.asarray(self.measure(selected), dtype=np.float32)
        st.measured += selected.tolist()
        st.costs += costs.tolist()
        st.history.append((selected, costs))
        i = int(np.argmin(costs)) if len(costs) else -1
        if i >= 0 and costs[i] < st.best_cost:
            st.best_cost, st.best_idx = float(costs[i]), int(selected[i])
        # update f-hat using D (rank loss, from scratch)
        idx = torch.from_numpy(np.array(st.measured, dtype=np.uint64).view(np.int64)).cuda()
        X = self.space.features(idx)
        c = torch.from_numpy(np.array(st.costs, dtype=np.float32)).cuda()
        key = torch.zeros(len(st.measured), dtype=torch.int16, device="cuda")
        self.model = at.gbt_fit_hist(X, len(st.measured), c, key, n_trees=cfg.n_trees, depth=cfg.depth,
                                     seed=cfg.seed + self.round)
        self.round += 1
        return selected

    def run(self, max_trials: int):
        while len(self.state.measured) < max_trials:
            before = len(self.state.measured)
            self.step()
            if len(self.state.measured) == before:      # space exhausted
                break
        return self.state.best_idx, self.state.best_cost
