#!/usr/bin/env python
"""bench.py -- throughput of the AutoTVM hot path (arXiv 1805.08166) on B200.

One STEP = one exploration round of Algorithm 1 over the whole hot path
 on config 2 of BASELINE.json:
  * sa_explore: 4096 persistent SA chains per GPU x 500 steps on the conv2d space
    28x28, 128->128, K3, S1 (|S| = 221,184,000; the shape BASELINE labels "C7" is Table 1's
    C6, reading Q2), energy = a 500-tree depth-6 GBT; every chain-step decodes a proposal,
    extracts its 468 features, scores it and takes the Metropolis decision (a2-a6);
  * the distinct top lambda*b = 128 of the visited set, measured configs excluded (a7);
    with N > 1 GPUs: NCCL all-gather of the per-rank lists + topk_merge;
  * select_topk: b = 64, eps = 0.05, alpha = 0.1 (a8);
  * refit: features_extract of the measured database D (|D| = 1024 synthetic measured
    configs) + gbt_fit_hist, 100 trees, depth 6, rank loss, histogram all-reduce over
    ranks (a9).  The refit result is not fed back into the next step's SA so every step
    carries the same 500-tree work.
metric: candidate schedules scored per second = chains x (steps + 1) x N / step time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
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
CHAINS, SA_STEPS, T_TREES, DEPTH = 4096, 500, 500, 6
K_POOL, B, EPS, ALPHA = 128, 64, 0.05, 0.1
D_SIZE, FIT_TREES, FIT_DEPTH = 1024, 100, 6
SEED = 1805
SWEEP_N = 1 << 20
SHARD_MIN = 16384          # refit databases at least this large shard their histograms over ranks


def workload_desc(n_gpus):
    return {
        "workload": "config 2: conv2d 28x28 128->128 K3 S1 P1 (Table-1 C6 shape; BASELINE label 'C7'), "
                    "T_CONV |S|=221184000; 500-tree depth-6 GBT energy; 4096 SA chains/GPU x 500 steps; "
                    "distinct top-128 -> diversity select b=64 eps=0.05 alpha=0.1; refit 100 trees d6 rank loss "
                    "on |D|=1024",
        "chains_per_gpu": CHAINS, "sa_steps": SA_STEPS, "gbt_trees": T_TREES, "gbt_depth": DEPTH,
        "pool": K_POOL, "b": B, "refit": {"samples": D_SIZE, "trees": FIT_TREES, "depth": FIT_DEPTH},
        "parallelism": f"dp{n_gpus} (chains sharded by global id; top-k all-gather; refit of |D|=1024 "
                       "replicated per rank, histogram all-reduce only for |D| >= 16384)",
        "l2": "flushed between steps (256 MiB write outside the per-step events)",
        "global_batch": CHAINS * n_gpus,
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
            # nvidia-smi needs ~0.1-0.5 s before its first sample: wait for it, so the (short) timed
            # region that follows is actually sampled
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


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1805_08166_b200 import at, build, synth
    from paper_1805_08166_b200 import dist as D

    build.build()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()

    space = at.Space([synth.CFG2A])
    ens = synth.ensemble(T_TREES, DEPTH, seed=SEED)
    model = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    temps_h = synth.temperatures(SA_STEPS, synth.energy_scale(T_TREES))
    temps = torch.from_numpy(temps_h).to(dev)
    base, cnt = D.chain_slice(CHAINS, rank)
    chain_idx = torch.zeros(cnt, dtype=torch.int64, device=dev)
    # measured database D (synthetic measurement = random log-linear model of the features)
    d_idx_h = synth.uniform_indices(space.size(), D_SIZE, seed=SEED + 1)
    d_idx = torch.from_numpy(d_idx_h.view(np.int64)).to(dev)
    XD0 = space.features(d_idx)
    cost_h = synth.labels(XD0[:, :D_SIZE].T.cpu().numpy(), seed=SEED + 2)
    cost = torch.from_numpy(cost_h).to(dev)
    gkey = torch.zeros(D_SIZE, dtype=torch.int16, device=dev)
    measured = torch.sort(d_idx)[0]
    # the refit's histograms are sharded (slice + int64 all-reduce per level) only when the
    # database is large enough for the saved work to beat 7 collectives per tree; |D| = 1024 is
    # refit redundantly on every rank (bit-identical results, no communication)
    shard_refit = world > 1 and D_SIZE >= SHARD_MIN
    hb, he = D.sample_slice(D_SIZE, rank, world) if shard_refit else (0, D_SIZE)
    allreduce = D.make_allreduce() if shard_refit else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    state = {"first": True}

    def step(r, chain_buf, meas, dcost, didx):
        res = at.sa_explore(space, model, chain_buf, temps, seed=SEED, round_=r, k_out=K_POOL, measured=meas,
                            init=state["first"], chain_id_base=base)
        state["first"] = False
        oi, osc, on = res["out_idx"], res["out_score"], res["out_n"]
        if world > 1:
            gi, gs, gn = D.gather_lists(oi, osc, on)
            oi, osc, on = at.topk_merge(space, gi, gs, gn, K_POOL, measured=meas)
        sel, nsel = at.select_topk(space, 0, oi[0], osc[0], b=B, eps=EPS, alpha=ALPHA, seed=SEED, round_=r,
                                   measured=meas)
        XD = space.features(didx)
        fit = at.gbt_fit_hist(XD, D_SIZE, dcost, gkey, n_trees=FIT_TREES, depth=FIT_DEPTH,
                              hist_range=(hb, he) if shard_refit else None, allreduce=allreduce)
        return sel, nsel, fit

    # warm-up (untimed)
    for r in range(args.warmup):
        step(r, chain_idx, measured, cost, d_idx)
    torch.cuda.synchronize()

    # timed region: exactly K steps, per-step CUDA events on the launching stream
    at.prof_reset()
    at.prof_enable(True)
    launches0 = at.launch_count()
    evs = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(args.warmup + k, chain_idx, measured, cost, d_idx)
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = at.launch_count() - launches0
    at.prof_enable(False)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = D.max_over_ranks(sum(step_ms), dev)
    prof = {k: at.prof_query(k) for k in at.AT_K}
    launches = int(D.max_over_ranks(float(launches), dev))
    candidates = CHAINS * (SA_STEPS + 1) * world * args.steps
    value = candidates / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # ---- dominant kernel roofline (SA kernel: tree walk on the L1/shared data pipe)
    import json as _json
    peaks = _json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    sa_n, sa_ms = prof["sa"]
    node_steps = CHAINS * (SA_STEPS + 1) * T_TREES * DEPTH          # per launch
    sm_clk = (peaks.get("sm_max_mhz") or 1965.0) * 1e6
    lds_peak = 148 * 16 * sm_clk / 1e9                               # Gnode-steps/s
    sa_avg = sa_ms / max(sa_n, 1)
    achieved = node_steps / (sa_avg / 1e3) / 1e9
    shares = {k: round(v[1] / max(sum(step_ms), 1e-9), 4) for k, v in prof.items() if v[0]}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")
    if os.path.exists(tpath):
        t = json.load(open(tpath)).get("sa_kernel", {})
        if t:
            traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
    roofline = {"kernel": "sa_kernel", "bound": "alu", "achieved": round(achieved, 2), "peak": round(lds_peak, 1),
                "unit": "Gnode-steps/s", "frac": round(achieved / lds_peak, 4),
                "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/)", "peak_source": "148 SMs x 16 node-steps/clk (two 128-B L1/shared wavefronts per "
                                                 "warp node-step) x sm_max_mhz of MEASURED_PEAKS.json",
                "avg_launch_ms": round(sa_avg, 4), "step_share": shares}
    # the walk's measured ceiling: tools/micro/walk_ceiling.cu (the same node-step instruction pattern,
    # everything in shared memory, no barriers, up to 24 walks per warp) plateaus at this rate
    wpath = os.path.join(ROOT, "profiles", "r01_walk_ceiling.json")
    if os.path.exists(wpath):
        wc = max(r.get("Gnode_steps_per_s", 0.0) for r in json.load(open(wpath))["results"] if "error" not in r)
        roofline["walk_ceiling_measured"] = round(wc, 1)
        roofline["frac_of_measured_ceiling"] = round(achieved / wc, 4)

    # ---- scoring sweep: features_extract + gbt_predict on 2^20 candidates (HBM roofline of the feature stream)
    sweep = None if args.quick else scoring_sweep(space, model, dev, stream, peaks)

    # ---- e2e: same step through the public API with host buffers (pinned) and copies in the timed region
    e2e = None if args.quick else run_e2e(args, step, chain_idx, measured, cost, d_idx, dev, stream, world)

    clocks = clk.summary()
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_desc(world),
        "sa_steps_per_s": round(CHAINS * SA_STEPS * world * args.steps / (total_ms / 1e3), 1),
        "roofline": roofline, "scoring_sweep": sweep, "e2e": e2e, "clocks": clocks, "gpu_launches": launches,
        "kernel_ms": {k: round(v[1], 3) for k, v in prof.items() if v[0]},
    }
    if rank == 0 and world == 1 and not (args.no_cpu_baseline or args.quick):
        out["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def scoring_sweep(space, model, dev, stream, peaks):
    import numpy as np
    import torch

    from paper_1805_08166_b200 import at, synth
    n = SWEEP_N
    idx = torch.from_numpy(synth.sweep_indices(space.size(), 0, n).view(np.int64)).to(dev)
    X = torch.empty((468, n), dtype=torch.float32, device=dev)
    score = torch.empty(n, dtype=torch.float32, device=dev)
    for _ in range(3):
        space.features(idx, out=X, ld=n)
        model.predict(X, n=n, out=score)
    torch.cuda.synchronize()
    reps = 5
    ef = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    ep = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for r in range(reps):
        ef[r][0].record(stream)
        space.features(idx, out=X, ld=n)
        ef[r][1].record(stream)
        ep[r][0].record(stream)
        model.predict(X, n=n, out=score)
        ep[r][1].record(stream)
    torch.cuda.synchronize()
    tf = statistics.median(a.elapsed_time(b) for a, b in ef)
    tp = statistics.median(a.elapsed_time(b) for a, b in ep)
    hbm = peaks.get("hbm_gbs", 6547.2)
    fbytes = n * (8 + 468 * 4)
    pbytes = n * (468 * 4 + 4)
    return {
        "candidates": n, "cand_per_s": round(n / ((tf + tp) / 1e3), 1),
        "features_extract": {"ms": round(tf, 4), "GBps": round(fbytes / tf / 1e6, 1),
                             "frac_hbm": round(fbytes / tf / 1e6 / hbm, 4), "bytes_per_cand": 8 + 468 * 4},
        "gbt_predict": {"ms": round(tp, 4), "GBps": round(pbytes / tp / 1e6, 1),
                        "frac_hbm": round(pbytes / tp / 1e6 / hbm, 4), "bytes_per_cand": 468 * 4 + 4,
                        "Gnode_steps_per_s": round(n * T_TREES * DEPTH / tp / 1e6, 2)},
        "hbm_peak_GBps": hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
    }


def run_e2e(args, step, chain_idx, measured, cost, d_idx, dev, stream, world):
    import torch
    h_chain = chain_idx.cpu().pin_memory()
    h_meas = measured.cpu().pin_memory()
    h_cost = cost.cpu().pin_memory()
    h_didx = d_idx.cpu().pin_memory()
    h_sel = torch.empty(B, dtype=torch.int64).pin_memory()
    h_chain_out = torch.empty_like(h_chain).pin_memory()
    k = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for r in range(k):
        c = h_chain.to(dev, non_blocking=True)
        m = h_meas.to(dev, non_blocking=True)
        co = h_cost.to(dev, non_blocking=True)
        di = h_didx.to(dev, non_blocking=True)
        sel, nsel, fit = step(1000 + r, c, m, co, di)
        h_sel.copy_(sel[:B], non_blocking=True)
        h_chain_out.copy_(c, non_blocking=True)
    t1.record(stream)
    torch.cuda.synchronize()
    from paper_1805_08166_b200 import dist as D
    ms = D.max_over_ranks(t0.elapsed_time(t1), dev)
    h2d = h_chain.numel() * 8 + h_meas.numel() * 8 + h_cost.numel() * 4 + h_didx.numel() * 8
    d2h = B * 8 + h_chain.numel() * 8
    return {"value": round(CHAINS * (SA_STEPS + 1) * world * k / (ms / 1e3), 1), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": k,
            "path": "paper_1805_08166_b200.at (C-ABI) with pinned host inputs copied in and results copied out"}


# ----------------------------------------------------------------------------- oracle (CPU)
def oracle_step(n_chains, r, state):
    """One step of the same workload through the CPU oracle on `n_chains` chains; returns timings."""
    import numpy as np

    import oracle as O
    from paper_1805_08166_b200 import synth
    if "osp" not in state:
        state["osp"] = O.OracleSpace([O.workload(**synth.CFG2A)])
        state["ens"] = O.OracleGbt(**synth.ensemble(T_TREES, DEPTH, seed=SEED))
        state["temps"] = synth.temperatures(SA_STEPS, synth.energy_scale(T_TREES))
        d_idx = synth.uniform_indices(state["osp"].size(), D_SIZE, seed=SEED + 1)
        state["d_idx"] = d_idx
        state["cost"] = synth.labels(state["osp"].features(d_idx), seed=SEED + 2)
        state["chains"] = None
    osp = state["osp"]
    t0 = time.perf_counter()
    res = osp.sa_explore(state["ens"], n_chains, SA_STEPS, SEED, r, state["temps"], chain_idx=state["chains"])
    (pi, pe), = osp.topk(res["visited_E"], res["visited_idx"], K_POOL, measured=state["d_idx"])
    t1 = time.perf_counter()
    osp.select(0, pi, pe, B, EPS, ALPHA, SEED, r, measured=state["d_idx"])
    XD = osp.features(state["d_idx"])
    O.fit_hist(XD, state["cost"], np.zeros(D_SIZE, np.uint16), n_trees=FIT_TREES, depth=FIT_DEPTH)
    t2 = time.perf_counter()
    state["chains"] = res["chain_idx"]
    return t1 - t0, t2 - t1


def cpu_baseline(sample_chains=256):
    """The oracle as it stands, one thread, on a bounded sample of the step: SA over `sample_chains`
    chains x 500 steps + top-k, then the full select + refit; the SA part is extrapolated linearly to
    4096 chains (chains are independent) to express a full-step rate in the metric's unit.  Beside it
    (SURVEY 8(d)): the same oracle with its SA chains split over every host core (one thread per
    chain slice, the ctypes calls release the GIL), select + refit still single-threaded."""
    st = {}
    t_sa, t_rest = oracle_step(sample_chains, 0, st)
    est = t_sa * CHAINS / sample_chains + t_rest
    out = {"value": round(CHAINS * (SA_STEPS + 1) / est, 1), "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"SA {sample_chains} chains x {SA_STEPS} steps + top-k ({t_sa:.2f} s, extrapolated x"
                     f"{CHAINS // sample_chains} to 4096 chains) + select + refit 100 trees on |D|=1024 "
                     f"({t_rest:.2f} s); single-threaded C oracle",
           "cpu": _cpu_model()}
    try:
        out["threads"] = _cpu_baseline_threads(st, t_rest)
    except Exception as e:   # a host without threads support still reports the 1-thread baseline
        out["threads"] = {"error": str(e)[:200]}
    return out


def _cpu_baseline_threads(st, t_rest, per_thread=32):
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np
    nproc = os.cpu_count() or 1
    osp, ens, temps = st["osp"], st["ens"], st["temps"]
    n = nproc * per_thread
    t0 = time.perf_counter()
    with ThreadPoolExecutor(nproc) as ex:
        futs = [ex.submit(osp.sa_explore, ens, per_thread, SA_STEPS, SEED, 1, temps, chain_id_base=k * per_thread)
                for k in range(nproc)]
        res = [f.result() for f in futs]
    osp.topk(np.concatenate([r["visited_E"] for r in res]), np.concatenate([r["visited_idx"] for r in res]), K_POOL,
             measured=st["d_idx"])
    t_sa = time.perf_counter() - t0
    est = t_sa * CHAINS / n + t_rest
    return {"value": round(CHAINS * (SA_STEPS + 1) / est, 1), "unit": UNIT, "cores": nproc,
            "sample": f"SA {n} chains on {nproc} threads + top-k ({t_sa:.2f} s, extrapolated to 4096 chains) + "
                      f"single-threaded select + refit ({t_rest:.2f} s)"}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cores)"
    except Exception:
        pass
    return f"{os.cpu_count()} logical cores"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sample = 32
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
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_desc(1),
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"per step: SA {sample} chains x {SA_STEPS} steps + top-k (extrapolated x"
                                   f"{CHAINS // sample} to 4096 chains) + select + refit 100 trees on |D|=1024; "
                                   "single-threaded C oracle", "cpu": _cpu_model()},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="timed steps only (no sweep / e2e / cpu baseline): for ncu")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
