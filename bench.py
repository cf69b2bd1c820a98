#!/usr/bin/env python
"""bench.py -- throughput of the AutoTVM hot path (arXiv 1805.08166) on B200.

One STEP = one exploration round of Algorithm 1 over the whole hot path (SURVEY.md
8(a) rows a2-a9) on config 3 of BASELINE.json, strong-scaled over the N GPUs:
  * sa_explore: 65,536 persistent SA chains in total (global chain c explores ResNet-18 workload
    C(c mod 12 + 1); rank r owns a contiguous slice of global ids) x 500 steps on the union of the
    12 Table-1 conv2d spaces (|S| = 1,740,983,040), energy = a 1000-tree depth-8 GBT; every
    chain-step decodes a proposal, extracts its 468 features, scores it and takes the Metropolis
    decision (a2-a6);
  * per workload the distinct top lambda b = 128 of the visited set, measured configs excluded
    (a7); with N > 1: ONE all-gather of the packed per-rank lists (NCCL over NVLink) + topk_merge;
  * select_topk for each of the 12 workloads (one select_topk_batch launch): b = 64, eps = 0.05,
    alpha = 0.1 (a8);
  * refit: features_extract of the measured database D (|D| = 12 x 128 synthetic measured configs,
    pairs within a workload) + gbt_fit_hist, 100 trees, depth 6, rank loss (a9), replicated on
    every rank (bit-identical, no communication: at this |D| a per-level histogram all-reduce
    costs more than it saves).  The refit is not fed back into the next step's SA energy, so every
    step carries the same 1000-tree work.
metric: candidate schedules scored per second = 65,536 x 501 / step time (the whole job, all
GPUs; SA steps/s = 65,536 x 500 / step time beside it).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment, bench.py starts N ranks itself (torchrun).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate schedules scored/sec (features+GBT) and SA steps/sec at 1/2/4/8 B200"
UNIT = "candidates/s"
# config 3 (headline)
CHAINS, SA_STEPS, T_TREES, DEPTH = 65536, 500, 1000, 8
NW = 12
K_POOL, B, EPS, ALPHA = 128, 64, 0.05, 0.1
D_PER_W = 128
D_SIZE = NW * D_PER_W
FIT_TREES, FIT_DEPTH = 100, 6
SEED = 1805
# config 2 (extra key)
C2_CHAINS, C2_STEPS, C2_TREES, C2_DEPTH, C2_D = 4096, 500, 500, 6, 1024
SWEEP_N = 1 << 20


def workload_desc(n_gpus):
    return {
        "workload": "config 3: the 12 ResNet-18 conv2d workloads of Table 1 batched (union |S|=1740983040), "
                    "1000-tree depth-8 GBT energy, 65536 SA chains x 500 steps (chain c -> workload c mod 12), "
                    "per-workload distinct top-128 -> diversity select b=64 eps=0.05 alpha=0.1 (12 workloads), "
                    "refit 100 trees d6 rank loss on |D|=1536 (128 per workload)",
        "chains_total": CHAINS, "chains_per_gpu": CHAINS // n_gpus, "sa_steps": SA_STEPS, "gbt_trees": T_TREES,
        "gbt_depth": DEPTH, "pool": K_POOL, "b": B, "workloads": NW,
        "refit": {"samples": D_SIZE, "trees": FIT_TREES, "depth": FIT_DEPTH, "placement": "replicated per rank"},
        "parallelism": f"dp{n_gpus} strong scaling: global chain ids split contiguously over ranks; one packed "
                       "NCCL all_gather of the per-rank top-k lists + topk_merge; select and refit replicated",
        "l2": "flushed between steps (256 MiB write outside the per-step events)",
        "global_batch": CHAINS,
    }


# ----------------------------------------------------------------------------- clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
            # nvidia-smi needs ~0.1-0.5 s before its first sample: wait for it so the timed region is sampled
            t0 = time.time()
            while time.time() - t0 < 5.0 and os.path.getsize(self.path) == 0:
                time.sleep(0.01)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.close()

    def summary(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if s > 300] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def _events(stream, fn, reps, warm=2):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


# ----------------------------------------------------------------------------- the config-3 round
class Config3:
    """Inputs of the headline step on this rank (all synthetic, seeded: DESIGN.md section 4)."""

    def __init__(self, rank, world, dev):
        import numpy as np
        import torch

        from paper_1805_08166_b200 import at, synth
        from paper_1805_08166_b200 import dist as D
        self.at, self.world = at, world
        self.grouped = torch.distributed.is_initialized()   # the exchange runs whenever a group exists
        self.space = at.Space(synth.ALL_RESNET)
        ens = synth.ensemble(T_TREES, DEPTH, seed=SEED)
        self.model = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
        self.temps = torch.from_numpy(synth.temperatures(SA_STEPS, synth.energy_scale(T_TREES))).to(dev)
        self.base, self.cnt = D.strong_slice(CHAINS, rank, world)
        self.chain_idx = torch.zeros(self.cnt, dtype=torch.int64, device=dev)
        self.cw = D.chain_workloads(self.base, self.cnt, NW, dev)
        # measured database D: 128 uniform configurations per workload, group key = workload
        key = (np.arange(D_SIZE) % NW).astype(np.uint16)
        sizes = np.array([self.space.size(w) for w in range(NW)], dtype=np.uint64)
        loc = synth.uniform_indices(1 << 62, D_SIZE, seed=SEED + 1) % sizes[key]
        d_idx = loc + np.array(self.space.offsets[:NW], dtype=np.uint64)[key]
        self.d_idx = torch.from_numpy(d_idx.view(np.int64)).to(dev)
        XD0 = self.space.features(self.d_idx)
        self.cost = torch.from_numpy(synth.labels(XD0[:, :D_SIZE].T.cpu().numpy(), seed=SEED + 2)).to(dev)
        self.gkey = torch.from_numpy(key.view(np.int16)).to(dev)
        self.measured = torch.sort(self.d_idx)[0]
        self.first = True
        self.last = None

    def step(self, r, chain_idx=None, measured=None, cost=None, d_idx=None):
        at, D = self.at, __import__("paper_1805_08166_b200.dist", fromlist=["x"])
        chain_idx = self.chain_idx if chain_idx is None else chain_idx
        meas = self.measured if measured is None else measured
        cost = self.cost if cost is None else cost
        d_idx = self.d_idx if d_idx is None else d_idx
        res = at.sa_explore(self.space, self.model, chain_idx, self.temps, seed=SEED, round_=r, k_out=K_POOL,
                            chain_workload=self.cw, measured=meas, init=self.first, chain_id_base=self.base)
        self.first = False
        oi, osc, on = res["out_idx"], res["out_score"], res["out_n"]
        if self.grouped:
            gi, gs, gn = D.gather_lists(oi, osc, on)
            oi, osc, on = at.topk_merge(self.space, gi, gs, gn, K_POOL, measured=meas)
        sel, _ = at.select_topk_batch(self.space, oi, osc, on, b=B, eps=EPS, alpha=ALPHA, seed=SEED, round_=r,
                                      measured=meas)   # the 12 workloads' selections in one launch
        sels = list(sel)
        XD = self.space.features(d_idx)
        fit = at.gbt_fit_hist(XD, D_SIZE, cost, self.gkey, n_trees=FIT_TREES, depth=FIT_DEPTH)
        self.last = (oi, osc, on, sels, fit)
        return sels

    def digest(self):
        """sha256 of the merged pools (idx, score bits, counts) and the 12 selections of the last step:
        identical at every rank count (global-id Philox streams, deterministic merge)."""
        import torch
        oi, osc, on, sels, _ = self.last
        h = hashlib.sha256()
        for t in (oi, osc.view(torch.int32), on, torch.stack(sels)):
            h.update(t.cpu().numpy().tobytes())
        return h.hexdigest()[:16], [int(x) for x in on.cpu().tolist()]


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1805_08166_b200 import at, build
    from paper_1805_08166_b200 import dist as D

    build.build()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    grouped = world > 1 or args.dist
    if grouped:
        # --dist at N = 1: a one-rank NCCL group, so the N > 1 code path (all-gather, merge, max-over-ranks,
        # the candidate split) runs and can be checked on one GPU
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    stream = torch.cuda.current_stream()
    peaks = _peaks()
    c3 = Config3(rank, world, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    for r in range(args.warmup):
        c3.step(r)
    torch.cuda.synchronize()

    # timed region: exactly K steps, per-step CUDA events on the launching stream
    at.prof_reset()
    at.prof_enable(True)
    launches0 = at.launch_count()
    evs = []
    if grouped:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c3.step(args.warmup + k)
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        if grouped:
            dist.barrier()
    launches = at.launch_count() - launches0
    at.prof_enable(False)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = D.max_over_ranks(sum(step_ms), dev)
    prof = {k: at.prof_query(k) for k in at.AT_K}
    launches = int(D.max_over_ranks(float(launches), dev))
    value = CHAINS * (SA_STEPS + 1) * args.steps / (total_ms / 1e3)
    digest, pool_n = c3.digest()
    clocks = clk.summary()

    roofline = sa_roofline(prof, sum(step_ms), c3.cnt, peaks)
    extra = {}
    if not grouped and not args.quick:
        extra["e2e"] = run_e2e(args, c3, dev, stream, world)
        extra["config2_round"] = config2_round(dev, stream)
        extra["configs"] = other_configs(dev, stream, peaks)
    elif not args.quick:
        extra["e2e"] = run_e2e(args, c3, dev, stream, world)
        extra["cfg5_split"] = cfg5_split(rank, world, dev, stream)
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_desc(world),
        "sa_steps_per_s": round(CHAINS * SA_STEPS * args.steps / (total_ms / 1e3), 1),
        "roofline": roofline, "e2e": extra.get("e2e"), "clocks": clocks, "gpu_launches": launches,
        "kernel_ms": {k: round(v[1], 3) for k, v in prof.items() if v[0]},
        "topk_sha": digest, "pool_counts": pool_n,
    }
    for k in ("config2_round", "configs", "cfg5_split"):
        if k in extra:
            out[k] = extra[k]
    if rank == 0 and not grouped and not (args.no_cpu_baseline or args.quick):
        out["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(out), file=_JSON_OUT, flush=True)
    if grouped:
        dist.barrier()
        dist.destroy_process_group()


def sa_roofline(prof, step_ms_sum, n_chains, peaks):
    """Roofline of the dominant kernel of the step, sa_kernel (its share is in step_share).  It is bound by
    the shared-memory pipe of the tree walk: each warp node-step is two 128-B L1/shared wavefronts (the
    node, then the feature) at one wavefront per clock per SM -> 148 x 16 node-steps per clock (DESIGN.md
    section 6); algorithmic work per launch = chains x (steps + 1) x trees x depth node-steps."""
    shares = {k: round(v[1] / max(step_ms_sum, 1e-9), 4) for k, v in prof.items() if v[0]}
    dom = max(shares, key=shares.get) if shares else "sa"
    sa_n, sa_ms = prof["sa"]
    node_steps = n_chains * (SA_STEPS + 1) * T_TREES * DEPTH
    sm_clk = (peaks.get("sm_max_mhz") or 1965.0) * 1e6
    lds_peak = 148 * 16 * sm_clk / 1e9
    sa_avg = sa_ms / max(sa_n, 1)
    achieved = node_steps / (sa_avg / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
    if os.path.exists(tpath):
        t = json.load(open(tpath)).get("sa_kernel_cfg3", {})
        if t:
            traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
    r = {"kernel": "sa_kernel", "dominant_class": dom, "bound": "alu", "achieved": round(achieved, 2),
         "peak": round(lds_peak, 1), "unit": "Gnode-steps/s", "frac": round(achieved / lds_peak, 4),
         "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/r02_ncu_traffic.json)",
         "peak_source": "derived: 148 SMs x 16 node-steps/clk (two 128-B L1/shared wavefronts per warp node-step) x "
                        "sm_max_mhz of MEASURED_PEAKS.json (no measured shared-memory peak exists)",
         "units_per_launch": f"{n_chains} chains x {SA_STEPS + 1} scored states x {T_TREES} trees x {DEPTH} levels",
         "avg_launch_ms": round(sa_avg, 4), "step_share": shares}
    wpath = os.path.join(ROOT, "profiles", "r01_walk_ceiling.json")
    if os.path.exists(wpath):
        wc = max(x.get("Gnode_steps_per_s", 0.0) for x in json.load(open(wpath))["results"] if "error" not in x)
        r["walk_ceiling_measured"] = round(wc, 1)
        r["frac_of_measured_ceiling"] = round(achieved / wc, 4)
    return r


def run_e2e(args, c3, dev, stream, world):
    """The same step through the public API with its inputs in pinned HOST memory: chain states, measured
    list, costs and the database indices copied in, the 12 selections and the final chain states copied
    out, all inside the timed region."""
    import torch
    h_chain = c3.chain_idx.cpu().pin_memory()
    h_meas = c3.measured.cpu().pin_memory()
    h_cost = c3.cost.cpu().pin_memory()
    h_didx = c3.d_idx.cpu().pin_memory()
    h_sel = torch.empty((NW, B), dtype=torch.int64).pin_memory()
    h_chain_out = torch.empty_like(h_chain).pin_memory()
    k = max(1, min(args.steps, 3))
    from paper_1805_08166_b200 import dist as D
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for r in range(k):
        c = h_chain.to(dev, non_blocking=True)
        m = h_meas.to(dev, non_blocking=True)
        co = h_cost.to(dev, non_blocking=True)
        di = h_didx.to(dev, non_blocking=True)
        sels = c3.step(1000 + r, chain_idx=c, measured=m, cost=co, d_idx=di)
        h_sel.copy_(torch.stack(sels)[:, :B], non_blocking=True)
        h_chain_out.copy_(c, non_blocking=True)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = D.max_over_ranks(t0.elapsed_time(t1), dev)
    h2d = h_chain.numel() * 8 + h_meas.numel() * 8 + h_cost.numel() * 4 + h_didx.numel() * 8
    d2h = NW * B * 8 + h_chain.numel() * 8
    return {"value": round(CHAINS * (SA_STEPS + 1) * k / (ms / 1e3), 1), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": k,
            "path": "paper_1805_08166_b200.at (C-ABI) with pinned host inputs copied in and results copied out"}


def cfg5_split(rank, world, dev, stream, n=10 ** 7, chunk=1 << 22):
    """Config 5 across the ranks: candidates (a n + c) mod |S_union| over the 12 ResNet spaces,
    a contiguous slice of the N = 10^7 per rank, features_extract -> gbt_predict with the 2000-tree depth-8
    ensemble, no communication; time = max over ranks, value = N / time."""
    import numpy as np
    import torch

    from paper_1805_08166_b200 import at, synth
    from paper_1805_08166_b200 import dist as D
    sp = at.Space(synth.ALL_RESNET)
    ens = synth.ensemble(2000, 8, seed=SEED)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    b, e = D.sample_slice(n, rank, world)
    idx = torch.from_numpy(synth.sweep_indices(sp.size(), b, e - b).view(np.int64)).to(dev)
    X = torch.empty((468, chunk), dtype=torch.float32, device=dev)
    s = torch.empty(e - b, dtype=torch.float32, device=dev)

    def run():
        for c0 in range(0, e - b, chunk):
            c1 = min(e - b, c0 + chunk)
            sp.features(idx[c0:c1], out=X, ld=chunk)
            g.predict(X, n=c1 - c0, out=s[c0:c1])

    run()
    torch.cuda.synchronize()
    if torch.distributed.is_initialized():
        torch.distributed.barrier()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    run()
    z.record(stream)
    torch.cuda.synchronize()
    ms = D.max_over_ranks(a.elapsed_time(z), dev)
    return {"candidates": n, "per_rank": e - b, "ms": round(ms, 2), "cand_per_s": round(n / (ms / 1e3), 1),
            "split": "contiguous candidate slices, no collective", "trees": 2000, "depth": 8}


# ----------------------------------------------------------------------------- extra keys (1 GPU)
def config2_round(dev, stream):
    """BASELINE config 2 as one Algorithm-1 round (the round-1 headline): 4096 chains x 500 steps on the
    conv 28x28 128->128 K3 S1 space, 500-tree depth-6 energy, top-128, select b=64, refit on |D|=1024."""
    import numpy as np
    import torch

    from paper_1805_08166_b200 import at, synth
    space = at.Space([synth.CFG2A])
    ens = synth.ensemble(C2_TREES, C2_DEPTH, seed=SEED)
    model = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    temps = torch.from_numpy(synth.temperatures(C2_STEPS, synth.energy_scale(C2_TREES))).to(dev)
    chain_idx = torch.zeros(C2_CHAINS, dtype=torch.int64, device=dev)
    d_idx = torch.from_numpy(synth.uniform_indices(space.size(), C2_D, seed=SEED + 1).view(np.int64)).to(dev)
    cost = torch.from_numpy(synth.labels(space.features(d_idx)[:, :C2_D].T.cpu().numpy(), seed=SEED + 2)).to(dev)
    gkey = torch.zeros(C2_D, dtype=torch.int16, device=dev)
    meas = torch.sort(d_idx)[0]
    st = {"first": True, "r": 0}

    def step():
        res = at.sa_explore(space, model, chain_idx, temps, seed=SEED, round_=st["r"], k_out=K_POOL, measured=meas,
                            init=st["first"])
        st["first"] = False
        at.select_topk(space, 0, res["out_idx"][0], res["out_score"][0], b=B, eps=EPS, alpha=ALPHA, seed=SEED,
                       round_=st["r"], measured=meas)
        at.gbt_fit_hist(space.features(d_idx), C2_D, cost, gkey, n_trees=FIT_TREES, depth=FIT_DEPTH)
        st["r"] += 1

    ms = _events(stream, step, reps=5, warm=3)
    return {"workload": "config 2 (conv 28x28 128->128 K3 S1, 500-tree d6, 4096 chains x 500 steps, top-128, "
                        "select b=64, refit 100 trees d6 on |D|=1024)", "ms_per_step": round(ms, 3),
            "value": round(C2_CHAINS * (C2_STEPS + 1) / (ms / 1e3), 1), "unit": UNIT}


def other_configs(dev, stream, peaks):
    """Configs 1, 4, 5 and the HBM-bound scoring stream, each timed with CUDA events (median)."""
    import numpy as np
    import torch

    from paper_1805_08166_b200 import at, synth
    hbm = peaks.get("hbm_gbs", 6547.2)
    out = {}

    def score(wls, T, D, idx_h, reps=5):
        sp = at.Space(wls)
        ens = synth.ensemble(T, D, seed=SEED)
        g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
        n = len(idx_h)
        idx = torch.from_numpy(idx_h.view(np.int64)).to(dev)
        ld = (n + 127) // 128 * 128
        X = torch.empty((468, ld), dtype=torch.float32, device=dev)
        sc = torch.empty(n, dtype=torch.float32, device=dev)
        tf = _events(stream, lambda: sp.features(idx, out=X, ld=ld), reps)
        tp = _events(stream, lambda: g.predict(X, n=n, out=sc), reps)
        fb, pb = n * (8 + 468 * 4), n * (468 * 4 + 4)
        return {"candidates": n, "trees": T, "depth": D, "cand_per_s": round(n / ((tf + tp) / 1e3), 1),
                "features_extract": {"ms": round(tf, 4), "GBps": round(fb / tf / 1e6, 1),
                                     "frac_hbm": round(fb / tf / 1e6 / hbm, 4)},
                "gbt_predict": {"ms": round(tp, 4), "GBps": round(pb / tp / 1e6, 1),
                                "frac_hbm": round(pb / tp / 1e6 / hbm, 4),
                                "Gnode_steps_per_s": round(n * T * D / tp / 1e6, 2)}}

    # config 1: exhaustive scoring of all 151,250 matmul-512 schedules (100 trees d6)
    out["cfg1_exhaustive_scoring"] = score([synth.MATMUL_512], 100, 6, np.arange(151250, dtype=np.uint64))
    # the feature stream at 2^20 candidates with the config-2 ensemble (HBM roofline of features_extract)
    sp2 = at.Space([synth.CFG2A])
    out["scoring_sweep_cfg2"] = score([synth.CFG2A], C2_TREES, C2_DEPTH, synth.sweep_indices(sp2.size(), 0, SWEEP_N))
    out["hbm_peak_GBps"] = hbm
    # config 4: refit 100 trees d6 on 10^5 samples over the 9 MobileNet depthwise spaces
    n = 100000
    sp4 = at.Space(synth.ALL_DW)
    key = synth.group_keys(n, 9, seed=4)
    sizes = np.array([sp4.size(w) for w in range(9)], dtype=np.uint64)
    loc = synth.uniform_indices(1 << 62, n, seed=5) % sizes[key]
    idx = torch.from_numpy((loc + np.array(sp4.offsets[:9], dtype=np.uint64)[key]).view(np.int64)).to(dev)
    X = sp4.features(idx)
    cost = torch.from_numpy(synth.labels(X[:, :n].T.cpu().numpy(), seed=6)).to(dev)
    kg = torch.from_numpy(key.view(np.int16)).to(dev)
    ms = _events(stream, lambda: at.gbt_fit_hist(X, n, cost, kg, n_trees=100, depth=6), reps=3, warm=1)
    out["cfg4_refit"] = {"samples": n, "trees": 100, "depth": 6, "ms": round(ms, 2), "ms_per_tree": round(ms / 100, 3)}
    # the multi-rank refit's per-rank compute: rank 0's work at R ranks (histograms over its 1/R sample slice,
    # everything else replicated) with the exchange replaced by a no-op -- the numbers exclude communication
    from paper_1805_08166_b200 import dist as D
    per_rank = {}
    for R in (2, 4, 8):
        hr = D.sample_slice(n, 0, R)
        per_rank[str(R)] = round(_events(stream, lambda: at.gbt_fit_hist(X, n, cost, kg, n_trees=100, depth=6,
                                                                         hist_range=hr, allreduce=lambda t: None),
                                         reps=2, warm=1), 2)
    out["cfg4_refit"]["per_rank_ms_no_exchange"] = per_rank
    del X
    # config 5: 10^7 candidates (a n + c) mod |S_union| x 2000-tree d8, in chunks of 2^24 (features -> GBT)
    sp5 = at.Space(synth.ALL_RESNET)
    ens = synth.ensemble(2000, 8, seed=SEED)
    g5 = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    n5, chunk = 10 ** 8, 1 << 24   # north_star's 10^8 sweep, 2^24-candidate chunks (31 GB feature buffer)
    idx5 = torch.from_numpy(synth.sweep_indices(sp5.size(), 0, n5).view(np.int64)).to(dev)
    X5 = torch.empty((468, chunk), dtype=torch.float32, device=dev)
    s5 = torch.empty(n5, dtype=torch.float32, device=dev)
    spans = [(c0, min(n5, c0 + chunk)) for c0 in range(0, n5, chunk)]

    def feats():
        for c0, c1 in spans:
            sp5.features(idx5[c0:c1], out=X5, ld=chunk)

    def preds():   # every chunk scored from the last chunk's features: the same work per call
        for c0, c1 in spans:
            g5.predict(X5, n=c1 - c0, out=s5[c0:c1])

    def run5():
        for c0, c1 in spans:
            sp5.features(idx5[c0:c1], out=X5, ld=chunk)
            g5.predict(X5, n=c1 - c0, out=s5[c0:c1])

    ms5 = _events(stream, run5, reps=1, warm=1)
    ms5f = _events(stream, feats, reps=1, warm=0)
    ms5p = _events(stream, preds, reps=1, warm=0)
    out["cfg5_sweep_1e8"] = {"candidates": n5, "trees": 2000, "depth": 8, "ms": round(ms5, 2),
                             "cand_per_s": round(n5 / (ms5 / 1e3), 1),
                             "features_extract_ms": round(ms5f, 2),
                             "gbt_predict_ms": round(ms5p, 2),
                             "gbt_predict_cand_per_s": round(n5 / (ms5p / 1e3), 1),
                             "gbt_predict_Gnode_steps_per_s": round(n5 * 16000 / (ms5p / 1e3) / 1e9, 1),
                             "Gnode_steps_per_s": round(n5 * 16000 / (ms5 / 1e3) / 1e9, 1)}
    del X5, idx5, s5
    return out


# ----------------------------------------------------------------------------- oracle (CPU)
def oracle_step(n_chains, r, state, threads=1):
    """One config-3 step through the CPU oracle on `n_chains` chains (global ids 0.., workload c mod 12):
    SA + per-workload top-k, then the 12 selections and the refit on |D| = 1536; returns timings."""
    import numpy as np

    import oracle as O
    from paper_1805_08166_b200 import synth
    if "osp" not in state:
        state["osp"] = O.OracleSpace([O.workload(**w) for w in synth.ALL_RESNET])
        state["ens"] = O.OracleGbt(**synth.ensemble(T_TREES, DEPTH, seed=SEED))
        state["temps"] = synth.temperatures(SA_STEPS, synth.energy_scale(T_TREES))
        osp = state["osp"]
        key = (np.arange(D_SIZE) % NW).astype(np.uint16)
        sizes = np.array([osp.size(w) for w in range(NW)], dtype=np.uint64)
        loc = synth.uniform_indices(1 << 62, D_SIZE, seed=SEED + 1) % sizes[key]
        state["d_idx"] = loc + np.array([osp.offset(w) for w in range(NW)], dtype=np.uint64)[key]
        state["key"] = key
        state["cost"] = synth.labels(osp.features(state["d_idx"]), seed=SEED + 2)
        state["chains"] = None
    osp = state["osp"]
    t0 = time.perf_counter()
    if threads <= 1:
        cw = (np.arange(n_chains) % NW).astype(np.uint16)
        res = osp.sa_explore(state["ens"], n_chains, SA_STEPS, SEED, r, state["temps"], chain_workload=cw,
                             chain_idx=state["chains"])
        vE, vI = res["visited_E"], res["visited_idx"]
        state["chains"] = res["chain_idx"]
    else:
        from concurrent.futures import ThreadPoolExecutor
        per = n_chains // threads
        with ThreadPoolExecutor(threads) as ex:
            futs = [ex.submit(osp.sa_explore, state["ens"], per, SA_STEPS, SEED, r, state["temps"],
                              chain_id_base=k * per, chain_workload=((np.arange(per) + k * per) % NW).astype(np.uint16))
                    for k in range(threads)]
            rs = [f.result() for f in futs]
        vE = np.concatenate([x["visited_E"] for x in rs])
        vI = np.concatenate([x["visited_idx"] for x in rs])
    pools = osp.topk(vE, vI, K_POOL, measured=state["d_idx"])
    t1 = time.perf_counter()
    for w, (pi, pe) in enumerate(pools):
        osp.select(w, pi, pe, B, EPS, ALPHA, SEED, r, measured=state["d_idx"])
    XD = osp.features(state["d_idx"])
    O.fit_hist(XD, state["cost"], state["key"], n_trees=FIT_TREES, depth=FIT_DEPTH)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def cpu_baseline(sample_chains=96):
    """The oracle as it stands on a bounded sample of the step: SA over `sample_chains` chains (8 per
    workload) x 500 steps + top-k, extrapolated linearly to 65,536 chains (chains are independent), plus
    the full 12 selections + refit; one thread, and beside it the SA chains split over every host core."""
    st = {}
    t_sa, t_rest = oracle_step(sample_chains, 0, st)
    est = t_sa * CHAINS / sample_chains + t_rest
    out = {"value": round(CHAINS * (SA_STEPS + 1) / est, 1), "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"SA {sample_chains} chains x {SA_STEPS} steps + top-k ({t_sa:.2f} s, extrapolated x"
                     f"{CHAINS / sample_chains:.0f} to 65536 chains) + 12 selections + refit 100 trees on "
                     f"|D|={D_SIZE} ({t_rest:.2f} s); single-threaded C oracle",
           "cpu": _cpu_model()}
    try:
        nproc = os.cpu_count() or 1
        n = nproc * 12
        t_sa2, _ = oracle_step(n, 1, {}, threads=nproc)
        est2 = t_sa2 * CHAINS / n + t_rest
        out["threads"] = {"value": round(CHAINS * (SA_STEPS + 1) / est2, 1), "unit": UNIT, "cores": nproc,
                          "sample": f"SA {n} chains on {nproc} threads + top-k ({t_sa2:.2f} s, extrapolated to 65536 "
                                    f"chains) + single-threaded selections + refit ({t_rest:.2f} s)"}
    except Exception as e:   # a host without threads support still reports the 1-thread baseline
        out["threads"] = {"error": str(e)[:200]}
    return out


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cores)"
    except Exception:
        pass
    return f"{os.cpu_count()} logical cores"


def run_reference(args):
    """--impl reference: the CPU oracle as it stands (there is no reference code to install: the reference
    is a paper), on this arm's config / metric / unit; each step a bounded sample of the config-3 step
    (24 chains x 500 steps extrapolated to 65,536 + 12 selections + refit).  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sample = 24
    st = {}
    for r in range(args.warmup):
        oracle_step(sample, r, st)
    times = []
    for k in range(args.steps):
        t_sa, t_rest = oracle_step(sample, args.warmup + k, st)
        times.append(t_sa * CHAINS / sample + t_rest)
    tot = sum(times)
    value = CHAINS * (SA_STEPS + 1) * args.steps / tot
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT,
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tot / args.steps * 1e3, 1), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": workload_desc(1),
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"per step: SA {sample} chains x {SA_STEPS} steps + top-k (extrapolated x"
                                   f"{CHAINS // sample} to 65536 chains) + 12 selections + refit 100 trees on "
                                   f"|D|={D_SIZE}; single-threaded C oracle", "cpu": _cpu_model()},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), file=_JSON_OUT, flush=True)


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _self_launch(args):
    """--gpus N > 1 outside torchrun: start N ranks on this node (127.0.0.1) and pass their output on."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


_JSON_OUT = sys.stdout


def _claim_stdout():
    """stdout carries exactly one JSON line: keep a private handle on it and point fd 1 at stderr, so
    anything else a library prints there (NCCL's version banner, warnings) cannot interleave."""
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true", help="N = 1: run the N > 1 code path in a one-rank NCCL group")
    ap.add_argument("--quick", action="store_true", help="timed steps only (no e2e / extra configs / cpu baseline): for ncu")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(_self_launch(args))
    _claim_stdout()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
