#!/usr/bin/env python
"""bench_configs.py -- supplementary per-config measurements (BASELINE.json configs 1-5) on one B200.

bench.py times the headline step (config 2).  This script measures every config's own hot-path
call, each timed with CUDA events on the launching stream (3 warm-ups, median of reps):

  cfg1  matmul 512^3 (|S| = 151,250), 100-tree depth-6 GBT: SA 64 chains x 200 steps -> top-8
        (alpha = eps = 0), and exhaustive scoring of all 151,250 configs (features + GBT)
  cfg2a conv 28x28 128->128 K3 S1 (C6 shape), 500 trees d6: SA 4096 x 500 (as bench.py) and
        scoring of 2^20 candidates;  cfg2b the Table-1 C7 space, same work
  cfg3  the 12 ResNet-18 conv2d spaces (union |S| = 1.74e9), 1000-tree depth-8 GBT,
        65,536 chains (chain c -> workload c mod 12) x STEPS3 steps, per-workload top-128
  cfg4  MobileNet-v1 depthwise spaces: refit 100 trees d6 on 10^5 synthetic measured samples
        (features_extract + gbt_fit_hist, single rank)
  cfg5  scoring sweep (a n + c) mod |S_union| over the 12 ResNet spaces with a 2000-tree d8
        ensemble, N = 2^16 candidates per launch pair (features_extract + gbt_predict)

Prints one JSON object; `python bench_configs.py --only cfg1,cfg4` limits the set.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def timed(fn, reps=5, warm=3):
    import torch
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def sa_case(at, synth, wls, T, D, chains, steps, k, chain_w=None, reps=3):
    import torch
    sp = at.Space(wls)
    ens = synth.ensemble(T, D, seed=1805)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    temps = torch.from_numpy(synth.temperatures(steps, synth.energy_scale(T))).cuda()
    ci = torch.zeros(chains, dtype=torch.int64, device="cuda")
    cw = None if chain_w is None else torch.from_numpy(chain_w).cuda()
    state = {"init": True}

    def run():
        at.sa_explore(sp, g, ci, temps, seed=1805, round_=0, k_out=k, chain_workload=cw, init=state["init"])
        state["init"] = False

    ms = timed(run, reps=reps, warm=2)
    node_steps = chains * (steps + 1) * T * D
    return {"chains": chains, "steps": steps, "trees": T, "depth": D, "ms": round(ms, 3),
            "chain_steps_per_s": round(chains * (steps + 1) / (ms / 1e3), 1),
            "Gnode_steps_per_s": round(node_steps / (ms / 1e3) / 1e9, 2)}


def score_case(at, synth, wls, T, D, n, sweep=False, peaks=None):
    import numpy as np
    import torch
    sp = at.Space(wls)
    ens = synth.ensemble(T, D, seed=1805)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    if sweep:
        idx_h = synth.sweep_indices(sp.size(), 0, n)
    else:
        idx_h = synth.uniform_indices(sp.size(), n, seed=7)
    idx = torch.from_numpy(idx_h.view(np.int64)).cuda()
    ld = (n + 127) // 128 * 128
    X = torch.empty((468, ld), dtype=torch.float32, device="cuda")
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    tf = timed(lambda: sp.features(idx, out=X, ld=ld))
    tp = timed(lambda: g.predict(X, n=n, out=out), reps=3)
    hbm = (peaks or {}).get("hbm_gbs", 6547.2)
    fb, pb = n * (8 + 468 * 4), n * (468 * 4 + 4)
    return {"candidates": n, "trees": T, "depth": D, "features_ms": round(tf, 4), "predict_ms": round(tp, 4),
            "cand_per_s": round(n / ((tf + tp) / 1e3), 1),
            "features_GBps": round(fb / tf / 1e6, 1), "features_frac_hbm": round(fb / tf / 1e6 / hbm, 4),
            "predict_GBps": round(pb / tp / 1e6, 1), "predict_frac_hbm": round(pb / tp / 1e6 / hbm, 4),
            "predict_Gnode_steps_per_s": round(n * T * D / (tp / 1e3) / 1e9, 2)}


def sweep_case(at, synth, T, D, Ns, chunk=1 << 24, peaks=None):
    """Config 5 as a sweep over N: candidates (a n + c) mod |S_union| scored in chunks of
    <= 2^24 by features_extract -> gbt_predict (the features of 10^8 candidates would be 187 GB)."""
    import numpy as np
    import torch
    sp = at.Space(synth.ALL_RESNET)
    ens = synth.ensemble(T, D, seed=1805)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    cmax = min(chunk, max(Ns))
    X = torch.empty((468, cmax), dtype=torch.float32, device="cuda")
    rows = []
    for n in Ns:
        idx = torch.from_numpy(synth.sweep_indices(sp.size(), 0, n).view(np.int64)).cuda()
        out = torch.empty(n, dtype=torch.float32, device="cuda")

        def run():
            for c0 in range(0, n, chunk):
                c1 = min(n, c0 + chunk)
                sp.features(idx[c0:c1], out=X, ld=cmax)
                g.predict(X, n=c1 - c0, out=out[c0:c1])

        ms = timed(run, reps=1 if n >= 10 ** 7 else 3, warm=1)
        # fused: sa_explore with 0 steps scores its chain states (features in shared memory, never in
        # HBM) and keeps the distinct top-64 per workload
        offs = np.array(sp.offsets[:12], dtype=np.uint64)
        cw = torch.from_numpy((np.searchsorted(offs, idx.cpu().numpy().view(np.uint64), "right") - 1)
                              .astype(np.int16)).cuda()
        temps = torch.empty(0, dtype=torch.float32, device="cuda")
        fused = {}

        def run_fused():
            for c0 in range(0, n, chunk):
                c1 = min(n, c0 + chunk)
                fused["r"] = at.sa_explore(sp, g, idx[c0:c1], temps, seed=1805, round_=0, k_out=64,
                                           chain_workload=cw[c0:c1], init=False)

        msf = timed(run_fused, reps=1 if n >= 10 ** 7 else 3, warm=1)
        last = (n - 1) // chunk * chunk   # the last chunk's scores, both ways
        same = bool(torch.equal(fused["r"]["chain_energy"].view(torch.int32), out[last:].view(torch.int32)))
        rows.append({"candidates": n, "ms": round(ms, 3), "cand_per_s": round(n / (ms / 1e3), 1),
                     "Gnode_steps_per_s": round(n * T * D / (ms / 1e3) / 1e9, 2),
                     "fused_ms": round(msf, 3), "fused_cand_per_s": round(n / (msf / 1e3), 1),
                     "fused_scores_bit_identical": same})
        del idx, out, cw
        torch.cuda.empty_cache()
    return {"trees": T, "depth": D, "chunk": chunk,
            "path": "unfused: features_extract -> gbt_predict per chunk; fused: sa_explore with 0 steps per chunk "
                    "(+ distinct top-64 per workload)",
            "sweep": rows}


def main():
    import numpy as np
    import torch

    from paper_1805_08166_b200 import at, build, synth
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg1,cfg2a,cfg2b,cfg3,cfg4,cfg5")
    ap.add_argument("--steps3", type=int, default=100)
    args = ap.parse_args()
    build.build()
    torch.cuda.set_device(0)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    only = set(args.only.split(","))
    res = {"device": torch.cuda.get_device_name(0)}
    if "cfg1" in only:
        r = {"sa": sa_case(at, synth, [synth.MATMUL_512], 100, 6, 64, 200, 8, reps=5)}
        r["exhaustive_scoring"] = score_case(at, synth, [synth.MATMUL_512], 100, 6, 151250, peaks=peaks)
        res["cfg1"] = r
    for name, wl in (("cfg2a", synth.CFG2A), ("cfg2b", synth.CFG2B)):
        if name in only:
            res[name] = {"sa": sa_case(at, synth, [wl], 500, 6, 4096, 500, 128),
                         "scoring": score_case(at, synth, [wl], 500, 6, 1 << 20, peaks=peaks)}
    if "cfg3" in only:
        cw = (np.arange(65536) % 12).astype(np.int16)
        res["cfg3"] = {"sa": sa_case(at, synth, synth.ALL_RESNET, 1000, 8, 65536, args.steps3, 128, chain_w=cw,
                                     reps=1),
                       "note": f"{args.steps3} SA steps per launch (config: 500); throughput is per chain-step"}
    if "cfg4" in only:
        n = 100000
        sp = at.Space(synth.ALL_DW)
        key = synth.group_keys(n, 9, seed=4)
        sizes = np.array([sp.size(w) for w in range(9)], dtype=np.uint64)
        loc = synth.uniform_indices(1 << 62, n, seed=5) % sizes[key]
        idx = torch.from_numpy((loc + np.array(sp.offsets[:9], dtype=np.uint64)[key]).view(np.int64)).cuda()
        X = sp.features(idx)
        cost = torch.from_numpy(synth.labels(X[:, :n].T.cpu().numpy(), seed=6)).cuda()
        kg = torch.from_numpy(key.view(np.int16)).cuda()
        ms = timed(lambda: at.gbt_fit_hist(X, n, cost, kg, n_trees=100, depth=6), reps=3, warm=1)
        res["cfg4"] = {"samples": n, "trees": 100, "depth": 6, "refit_ms": round(ms, 2),
                       "ms_per_tree": round(ms / 100, 3)}
    if "cfg5" in only:
        res["cfg5"] = score_case(at, synth, synth.ALL_RESNET, 2000, 8, 1 << 16, sweep=True, peaks=peaks)
        res["cfg5_sweep"] = sweep_case(at, synth, 2000, 8, [10 ** 4, 10 ** 5, 10 ** 6, 10 ** 7, 10 ** 8], peaks=peaks)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
