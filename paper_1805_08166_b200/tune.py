"""Algorithm 1 of the paper driven over the C-ABI: the model-guided tuning loop.

    D <- {}
    while n_trials < max_n_trials:
        Q <- parallel SA over S_e with energy f-hat                  (sa_explore)
        S <- greedy Eq. 3 (1 - eps) b from the top lambda b  + eps b random  (select_topk)
        for s in S: c <- f(g(e, s)); D <- D U {(e, s, c)}            (measure: caller-supplied f)
        update f-hat using D                                         (gbt_fit_hist, Eq. 2)
    s* <- history best

Chains persist across rounds.  Before the first refit f-hat is the caller's initial model
(e.g. a transferred / synthetic ensemble).  Options:
  objective="reg"        the regression loss sum (f - c)^2 instead of Eq. 2;
  global_model=g         transfer learning, Eq. 4: f-hat = f_global + f_local, the local
                         fit on top of f_global's scores (base margin), scored as one ensemble;
  n_bootstrap=K, acq     K models on bootstrap multisets of D and an EI / UCB acquisition as the
                         SA energy.  The measurement f is a callable on global indices that
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
    objective: str = "rank"      # "rank" (Eq. 2) or "reg"
    n_bootstrap: int = 0         # K >= 2: bootstrap ensemble with an acquisition energy
    acq: str = "ucb"             # "ucb" | "ei" | "mean"
    kappa: float = 1.0


@dataclass
class TuneState:
    chain_idx: object = None                      # device int64 [n_chains], persistent
    measured: list = field(default_factory=list)  # global indices in measurement order
    costs: list = field(default_factory=list)
    best_idx: int = -1
    best_cost: float = float("inf")
    history: list = field(default_factory=list)   # per round: (selected, costs)


class Tuner:
    def __init__(self, workload: dict, model, measure, cfg: TuneConfig = TuneConfig(), global_model=None):
        import torch

        from . import at
        self.at = at
        self.torch = torch
        self.space = at.Space([workload])
        self.model = model
        self.global_model = global_model   # f_global of Eq. 4 (or None)
        self.acq = None                    # acquisition options of the current energy (bootstrap)
        self.measure = measure
        self.cfg = cfg
        self.state = TuneState(chain_idx=torch.zeros(cfg.n_chains, dtype=torch.int64, device="cuda"))
        self.round = 0

    def _temps(self, meas):
        """Reading Q21: geometric T0 -> t_ratio T0 with T0 = sigma of the round's initial chain energies
        under the current f-hat (synth.energy_sigma).  The energies come from a 0-step sa_explore, which
        scores the chain states and moves nothing; the 128 floats are read back (the round syncs for the
        measurement anyway) so that the schedule is the same fp64 arithmetic on every replay."""
        from .synth import energy_sigma, temperatures
        at, torch, cfg, st = self.at, self.torch, self.cfg, self.state
        empty = torch.empty(0, dtype=torch.float32, device=st.chain_idx.device)
        r0 = at.sa_explore(self.space, self.model, st.chain_idx, empty, seed=cfg.seed, round_=self.round, k_out=1,
                           measured=meas, init=self.round == 0, acq=self.acq)
        t0 = energy_sigma(r0["chain_energy"].cpu().numpy())
        return torch.from_numpy(temperatures(cfg.n_steps, t0, cfg.t_ratio)).cuda()

    def step(self):
        """One iteration of Algorithm 1; returns the selected global indices (numpy u64)."""
        at, torch, cfg, st = self.at, self.torch, self.cfg, self.state
        meas = None
        if st.measured:
            meas = torch.from_numpy(np.sort(np.array(st.measured, dtype=np.uint64)).view(np.int64)).cuda()
        res = at.sa_explore(self.space, self.model, st.chain_idx, self._temps(meas), seed=cfg.seed, round_=self.round,
                            k_out=cfg.lam * cfg.b, measured=meas, init=self.round == 0, acq=self.acq)
        n_pool = int(res["out_n"][0])
        sel, n_sel = at.select_topk(self.space, 0, res["out_idx"][0, :n_pool].contiguous(),
                                    res["out_score"][0, :n_pool].contiguous(), b=cfg.b, eps=cfg.eps,
                                    alpha=cfg.alpha, seed=cfg.seed, round_=self.round, measured=meas)
        selected = sel[:int(n_sel)].cpu().numpy().view(np.uint64).copy()
        costs = np.asarray(self.measure(selected), dtype=np.float32)
        st.measured += selected.tolist()
        st.costs += costs.tolist()
        st.history.append((selected, costs))
        fin = np.where(np.isfinite(costs), costs, np.inf)
        i = int(np.argmin(fin)) if len(costs) else -1
        if i >= 0 and fin[i] < st.best_cost:
            st.best_cost, st.best_idx = float(costs[i]), int(selected[i])
        # update f-hat using D (from scratch); failed measurements (non-finite cost) stay in D -- they
        # are never proposed again -- but are left out of the fit
        fit = self.refit()
        if fit is not None:
            self.model, self.acq = fit
        self.round += 1
        return selected

    def _fit(self, X, n, c, key):
        """One model on (X, c): f_local on top of f_global's scores when transferring (Eq. 4)."""
        at, cfg = self.at, self.cfg
        margin = self.global_model.predict(X, n) if self.global_model is not None else None
        local = at.gbt_fit_hist(X, n, c, key, n_trees=cfg.n_trees, depth=cfg.depth, seed=cfg.seed + self.round,
                                objective=cfg.objective, base_margin=margin)
        return self.global_model.concat(local) if self.global_model is not None else local

    def refit(self):
        """update f-hat using D: one model, or K bootstrap models concatenated for the acquisition."""
        at, torch, cfg, st = self.at, self.torch, self.cfg, self.state
        costs = np.array(st.costs, dtype=np.float32)
        ok = np.isfinite(costs)
        n = int(ok.sum())
        if n < 2:          # nothing to rank yet: keep the current f-hat
            return None
        idx = torch.from_numpy(np.array(st.measured, dtype=np.uint64)[ok].view(np.int64)).cuda()
        X = self.space.features(idx)
        c = torch.from_numpy(costs[ok]).cuda()
        key = torch.zeros(n, dtype=torch.int16, device="cuda")
        if cfg.n_bootstrap < 2:
            return self._fit(X, n, c, key), None
        model = None
        for k in range(cfg.n_bootstrap):
            Xk, ck, kk, _ = at.bootstrap_resample(X, n, c, key, k, seed=cfg.seed, round_=self.round)
            mk = self._fit(Xk, n, ck, kk)
            model = mk if model is None else model.concat(mk)
        base = float(self.global_model.export()["base"]) if self.global_model is not None else 0.0
        acq = dict(n_models=cfg.n_bootstrap, kind=cfg.acq, kappa=cfg.kappa, best=0.0,
                   model_base=[base] * cfg.n_bootstrap)
        if cfg.acq == "ei":   # incumbent: the lowest mean score over the measured configurations
            _, mu, _ = model.predict_acq(X, n, cfg.n_bootstrap, kind="mean", model_base=acq["model_base"])
            acq["best"] = float(mu.min())
        return model, acq

    def run(self, max_trials: int):
        while len(self.state.measured) < max_trials:
            before = len(self.state.measured)
            self.step()
            if len(self.state.measured) == before:      # space exhausted
                break
        return self.state.best_idx, self.state.best_cost
