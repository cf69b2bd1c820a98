"""ctypes wrapper around liboracle.so -- the plain CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product package paper_1805_08166_b200 never
imports it; the C sources share no code with the CUDA path (see oracle.h).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
NFEAT = 468

CFLAGS = ["-O2", "-std=gnu11", "-Wall", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math"]


def build(force: bool = False) -> Path:
    src = HERE / "oracle.c"
    hdr = HERE / "oracle.h"
    if force or not LIB.exists() or LIB.stat().st_mtime < max(src.stat().st_mtime, hdr.stat().st_mtime):
        tmp = LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", *CFLAGS, "-o", str(tmp), str(src), "-lm"])
        os.replace(tmp, LIB)
    return LIB


class Workload(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("kind", "n", "m", "k", "h", "w", "ic", "oc", "ksize", "stride", "pad")]


class Space(C.Structure):
    _fields_ = [
        ("wl", Workload), ("tmpl", C.c_int), ("n_axes", C.c_int),
        ("axis_ext", C.c_int64 * 6), ("axis_levels", C.c_int * 6),
        ("n_knobs", C.c_int), ("knob_kind", C.c_int * 9), ("knob_axis", C.c_int * 9),
        ("radix", C.c_int * 9), ("fact", C.POINTER(C.c_int) * 9),
        ("place", C.c_uint64 * 9), ("size", C.c_uint64), ("unroll_vals", C.c_int * 5),
        ("n_dims", C.c_int * 3), ("shape", (C.c_int64 * 4) * 3), ("rowstride", (C.c_int64 * 4) * 3),
        ("n_terms", (C.c_int * 4) * 3), ("term_axis", ((C.c_int * 2) * 4) * 3),
        ("term_mult", ((C.c_int64 * 2) * 4) * 3),
    ]


class SpaceSet(C.Structure):
    _fields_ = [("n", C.c_int), ("sp", Space * 16), ("offset", C.c_uint64 * 17)]


class Nest(C.Structure):
    _fields_ = [("n", C.c_int), ("axis", C.c_int * 18), ("level", C.c_int * 18),
                ("ext", C.c_int64 * 18), ("ann", C.c_int * 18), ("coef", C.c_int64 * 18)]


class LoopCtx(C.Structure):
    _fields_ = [("length", C.c_int64), ("top_down", C.c_int64), ("bottom_up", C.c_int64),
                ("ann", C.c_int), ("touch", C.c_uint64 * 3), ("reuse", C.c_float * 3),
                ("stride", C.c_int64 * 3)]


class Gbt(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("depth", C.c_int32),
                ("feat", C.POINTER(C.c_uint16)), ("thresh", C.POINTER(C.c_float)),
                ("leaf", C.POINTER(C.c_float)), ("base", C.c_float)]


class FitOpts(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("depth", C.c_int32), ("max_bins", C.c_int32),
                ("group_size", C.c_int32), ("eta", C.c_float), ("lambda_", C.c_float),
                ("min_child_weight", C.c_float), ("seed", C.c_uint64), ("objective", C.c_int32),
                ("base_margin", C.POINTER(C.c_float))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(LIB))
        _lib.or_exp_det.restype = C.c_float
        _lib.or_exp_det.argtypes = [C.c_float]
        _lib.or_mulhi64.restype = C.c_uint64
        _lib.or_mulhi64.argtypes = [C.c_uint64, C.c_uint64]
        _lib.or_count_factorizations.restype = C.c_uint64
        _lib.or_count_factorizations.argtypes = [C.c_int64, C.c_int]
        _lib.or_touch.restype = C.c_uint64
        _lib.or_touch_bruteforce.restype = C.c_uint64
        _lib.or_encode.restype = C.c_uint64
        _lib.or_gbt_score.restype = C.c_float
        _lib.or_expected_improvement.restype = C.c_float
        _lib.or_expected_improvement.argtypes = [C.c_float, C.c_float, C.c_float]
        _lib.or_acquisition.restype = C.c_float
        _lib.or_rank_loss.restype = C.c_double
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def workload(kind, **kw) -> Workload:
    w = Workload()
    w.kind = {"matmul": 0, "conv2d": 1, "depthwise": 2}.get(kind, kind)
    for k, v in kw.items():
        setattr(w, k, int(v))
    return w


class OracleSpace:
    """A union schedule space over one or more workloads (or_space_set)."""

    def __init__(self, workloads):
        self.workloads = list(workloads)
        arr = (Workload * len(self.workloads))(*self.workloads)
        self.s = SpaceSet()
        rc = lib().or_space_set_create(arr, len(self.workloads), C.byref(self.s))
        if rc != 0:
            raise ValueError("oracle: bad workload")

    def __del__(self):
        try:
            lib().or_space_set_free(C.byref(self.s))
        except Exception:
            pass

    @property
    def n(self):
        return self.s.n

    def size(self, w=None):
        if w is None:
            return int(self.s.offset[self.s.n])
        return int(self.s.sp[w].size)

    def offset(self, w):
        return int(self.s.offset[w])

    def radices(self, w=0):
        sp = self.s.sp[w]
        return [int(sp.radix[j]) for j in range(sp.n_knobs)]

    def factors(self, w, j):
        sp = self.s.sp[w]
        L = sp.axis_levels[sp.knob_axis[j]]
        return [tuple(sp.fact[j][r * L + l] for l in range(L)) for r in range(sp.radix[j])]

    def decode(self, idx, w=0):
        ch = (C.c_int * 9)()
        lib().or_decode(C.byref(self.s.sp[w]), C.c_uint64(idx), ch)
        return [int(ch[j]) for j in range(self.s.sp[w].n_knobs)]

    def encode(self, choices, w=0):
        ch = (C.c_int * 9)(*choices)
        return int(lib().or_encode(C.byref(self.s.sp[w]), ch))

    def lower(self, choices, w=0) -> Nest:
        ch = (C.c_int * 9)(*choices)
        ns = Nest()
        lib().or_lower(C.byref(self.s.sp[w]), ch, C.byref(ns))
        return ns

    def context(self, choices, w=0):
        ns = self.lower(choices, w)
        rows = (LoopCtx * 18)()
        lib().or_context(C.byref(self.s.sp[w]), C.byref(ns), rows)
        return ns, [rows[k] for k in range(ns.n)]

    def touch(self, ns, b, k, w=0, brute=False):
        f = lib().or_touch_bruteforce if brute else lib().or_touch
        return int(f(C.byref(self.s.sp[w]), C.byref(ns), C.c_int(b), C.c_int(k)))

    def features(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        out = np.zeros((len(idx), NFEAT), dtype=np.float32)
        rc = lib().or_features(C.byref(self.s), _p(idx, C.c_uint64), C.c_int64(len(idx)), _p(out, C.c_float))
        if rc != 0:
            raise ValueError("oracle: index out of range")
        return out

    # -- SA / top-k / select -------------------------------------------------
    def features_knobs(self, idx):
        """Configuration features (Q44): [n][32] fp32."""
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        out = np.zeros((len(idx), 32), np.float32)
        rc = lib().or_features_knobs(C.byref(self.s), _p(idx, C.c_uint64), C.c_int64(len(idx)), _p(out, C.c_float))
        if rc != 0:
            raise ValueError(f"oracle features_knobs rc={rc}")
        return out

    def sa_explore(self, ens, n_chains, n_steps, seed, round_, temps, chain_id_base=0,
                   chain_workload=None, chain_idx=None, acq=None):
        """acq: optional (kind, kappa, best) -- `ens` is then a list of K models and the energy is
        their acquisition."""
        if acq is not None:
            arr = (Gbt * len(ens))(*[m.c() for m in ens])
            g = arr
        else:
            g = ens.c()
        init = chain_idx is None
        cidx = np.zeros(n_chains, np.uint64) if init else np.array(chain_idx, dtype=np.uint64)
        cE = np.zeros(n_chains, np.float32)
        nw = (n_steps + 31) // 32
        acc = np.zeros((n_chains, nw), np.uint32)
        vE = np.zeros((n_chains, n_steps + 1), np.float32)
        vI = np.zeros((n_chains, n_steps + 1), np.uint64)
        temps = np.ascontiguousarray(temps, dtype=np.float32)
        cw = None if chain_workload is None else np.ascontiguousarray(chain_workload, dtype=np.uint16)
        head = (C.byref(self.s), C.byref(g)) if acq is None else \
            (C.byref(self.s), g, C.c_int(len(ens)), C.c_int(ACQ[acq[0]]), C.c_float(acq[1]), C.c_float(acq[2]))
        fn = lib().or_sa_explore if acq is None else lib().or_sa_explore_acq
        rc = fn(
            *head, C.c_int32(n_chains), C.c_int32(n_steps), C.c_uint64(seed),
            C.c_uint32(round_), C.c_uint32(chain_id_base), _p(temps, C.c_float),
            None if cw is None else _p(cw, C.c_uint16), C.c_int(1 if init else 0),
            _p(cidx, C.c_uint64), _p(cE, C.c_float), _p(acc, C.c_uint32), _p(vE, C.c_float), _p(vI, C.c_uint64))
        if rc != 0:
            raise ValueError(f"oracle sa_explore rc={rc}")
        return dict(chain_idx=cidx, chain_energy=cE, accept_bits=acc, visited_E=vE, visited_idx=vI)

    def topk(self, E, idx, K, measured=()):
        E = np.ascontiguousarray(E, dtype=np.float32).ravel()
        idx = np.ascontiguousarray(idx, dtype=np.uint64).ravel()
        meas = np.ascontiguousarray(np.sort(np.asarray(measured, dtype=np.uint64)))
        oi = np.zeros((self.n, K), np.uint64)
        oE = np.zeros((self.n, K), np.float32)
        on = np.zeros(self.n, np.int32)
        lib().or_topk_distinct(C.byref(self.s), _p(E, C.c_float), _p(idx, C.c_uint64), C.c_int64(len(E)),
                               _p(meas, C.c_uint64), C.c_int64(len(meas)), C.c_int32(K),
                               _p(oi, C.c_uint64), _p(oE, C.c_float), _p(on, C.c_int32))
        return [(oi[w, :on[w]].copy(), oE[w, :on[w]].copy()) for w in range(self.n)]

    def select(self, w, pool_idx, pool_E, b, eps, alpha, seed, round_, measured=()):
        pi = np.ascontiguousarray(pool_idx, dtype=np.uint64)
        pe = np.ascontiguousarray(pool_E, dtype=np.float32)
        meas = np.ascontiguousarray(np.sort(np.asarray(measured, dtype=np.uint64)))
        out = np.zeros(max(b, 1), np.uint64)
        on = C.c_int32(0)
        rc = lib().or_select(C.byref(self.s), C.c_int(w), _p(pi, C.c_uint64), _p(pe, C.c_float),
                             C.c_int64(len(pi)), _p(meas, C.c_uint64), C.c_int64(len(meas)), C.c_int32(b),
                             C.c_float(eps), C.c_float(alpha), C.c_uint64(seed), C.c_uint32(round_),
                             _p(out, C.c_uint64), C.byref(on))
        if rc != 0:
            raise ValueError("oracle select failed")
        return out[:on.value].copy()


class OracleGbt:
    """Heap-layout ensemble (feat u16 [T][2^D-1], thresh f32 [T][2^D-1], leaf f32 [T][2^D])."""

    def __init__(self, feat, thresh, leaf, base=0.0):
        self.feat = np.ascontiguousarray(feat, dtype=np.uint16)
        self.thresh = np.ascontiguousarray(thresh, dtype=np.float32)
        self.leaf = np.ascontiguousarray(leaf, dtype=np.float32)
        self.base = float(np.float32(base))
        self.n_trees = self.leaf.shape[0]
        self.depth = int(round(np.log2(self.leaf.shape[1])))

    def c(self) -> Gbt:
        g = Gbt()
        g.n_trees, g.depth = self.n_trees, self.depth
        g.feat = _p(self.feat, C.c_uint16)
        g.thresh = _p(self.thresh, C.c_float)
        g.leaf = _p(self.leaf, C.c_float)
        g.base = self.base
        return g

    def predict(self, X, slots=False):
        X = np.ascontiguousarray(X, dtype=np.float32)
        n, F = X.shape
        score = np.zeros(n, np.float32)
        sl = np.zeros((self.n_trees, n), np.uint8) if slots else None
        g = self.c()
        lib().or_gbt_predict(C.byref(g), _p(X, C.c_float), C.c_int64(n), C.c_int(F), _p(score, C.c_float),
                             None if sl is None else _p(sl, C.c_uint8))
        return (score, sl) if slots else score


def gbt_concat(a, b):
    """Eq. 4: the global model's trees then the local model's, as one OracleGbt."""
    D = max(a.depth, b.depth)
    T = a.n_trees + b.n_trees
    feat = np.zeros((T, (1 << D) - 1), np.uint16)
    thr = np.zeros((T, (1 << D) - 1), np.float32)
    leaf = np.zeros((T, 1 << D), np.float32)
    base = C.c_float()
    ga, gb = a.c(), b.c()
    lib().or_gbt_concat(C.byref(ga), C.byref(gb), _p(feat, C.c_uint16), _p(thr, C.c_float), _p(leaf, C.c_float),
                        C.byref(base))
    return OracleGbt(feat, thr, leaf, base.value)


ACQ = {"mean": 0, "ucb": 1, "ei": 2}


def bootstrap_indices(n, model, seed=1805, round_=0):
    """Q40: model `model`'s bootstrap multiset (n draws with replacement, Philox tag BOOT)."""
    idx = np.zeros(n, np.int64)
    lib().or_bootstrap_indices(C.c_int64(n), C.c_int32(model), C.c_uint64(seed), C.c_uint32(round_), _p(idx, C.c_int64))
    return idx


def expected_improvement(mu, sd, best):
    return float(np.float32(lib().or_expected_improvement(C.c_float(mu), C.c_float(sd), C.c_float(best))))


def acquisition(kind, f, kappa=1.0, best=0.0):
    f = np.ascontiguousarray(f, dtype=np.float32)
    m, s = C.c_float(), C.c_float()
    v = lib().or_acquisition(C.c_int(ACQ[kind]), C.c_int(len(f)), _p(f, C.c_float), C.c_float(kappa), C.c_float(best),
                             C.byref(m), C.byref(s))
    return float(np.float32(v)), float(np.float32(m.value)), float(np.float32(s.value))


def predict_acq(models, X, kind="ucb", kappa=1.0, best=0.0):
    """Acquisition over K models: (score, mean, std) per row of X [n][F]."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, F = X.shape
    arr = (Gbt * len(models))(*[m.c() for m in models])
    score, mean, std = np.zeros(n, np.float32), np.zeros(n, np.float32), np.zeros(n, np.float32)
    rc = lib().or_gbt_predict_acq(arr, C.c_int(len(models)), _p(X, C.c_float), C.c_int64(n), C.c_int(F),
                                  C.c_int(ACQ[kind]), C.c_float(kappa), C.c_float(best), _p(score, C.c_float),
                                  _p(mean, C.c_float), _p(std, C.c_float))
    if rc != 0:
        raise ValueError(f"oracle predict_acq rc={rc}")
    return score, mean, std


def reg_gradients(cost, pred):
    cost = np.ascontiguousarray(cost, dtype=np.float32)
    pred = np.ascontiguousarray(pred, dtype=np.float32)
    n = cost.shape[0]
    g = np.zeros(n, np.int64)
    h = np.zeros(n, np.int64)
    lib().or_reg_gradients(_p(cost, C.c_float), _p(pred, C.c_float), C.c_int64(n), _p(g, C.c_int64), _p(h, C.c_int64))
    return g, h


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return [int(o[i]) for i in range(4)]


def exp_det(a):
    return float(np.float32(lib().or_exp_det(C.c_float(a))))


def exp_det_array(a):
    a = np.asarray(a, dtype=np.float32)
    return np.array([lib().or_exp_det(C.c_float(float(v))) for v in a.ravel()], dtype=np.float32).reshape(a.shape)


def exp_det_range(first_bits, n):
    """exp_det of the n fp32 values with bit patterns first_bits, first_bits + 1, ... (C loop)."""
    out = np.empty(n, np.float32)
    lib().or_exp_det_range(C.c_uint32(first_bits), C.c_int64(n), _p(out, C.c_float))
    return out


def mulhi64(a, b):
    return int(lib().or_mulhi64(C.c_uint64(a), C.c_uint64(b)))


def count_factorizations(n, L):
    return int(lib().or_count_factorizations(C.c_int64(n), C.c_int(L)))


def fit_cuts(X, max_bins=256):
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, F = X.shape
    cuts = np.zeros((F, max_bins - 1), np.float32)
    nc = np.zeros(F, np.int32)
    lib().or_fit_cuts(_p(X, C.c_float), C.c_int64(n), C.c_int(F), C.c_int(max_bins), _p(cuts, C.c_float),
                      _p(nc, C.c_int32))
    return cuts, nc


def group_positions(gkey, seed, tree):
    gk = np.ascontiguousarray(gkey, dtype=np.uint16)
    pos = np.zeros(len(gk), np.int64)
    lib().or_group_positions(_p(gk, C.c_uint16), C.c_int64(len(gk)), C.c_uint64(seed), C.c_int32(tree),
                             _p(pos, C.c_int64))
    return pos


def pair_gradients(cost, pred, gkey, seed, tree, group_size=64):
    cost = np.ascontiguousarray(cost, dtype=np.float32)
    pred = np.ascontiguousarray(pred, dtype=np.float32)
    gk = np.ascontiguousarray(gkey, dtype=np.uint16)
    g = np.zeros(len(cost), np.int64)
    h = np.zeros(len(cost), np.int64)
    lib().or_pair_gradients(_p(cost, C.c_float), _p(pred, C.c_float), _p(gk, C.c_uint16), C.c_int64(len(cost)),
                            C.c_uint64(seed), C.c_int32(tree), C.c_int32(group_size), _p(g, C.c_int64),
                            _p(h, C.c_int64))
    return g, h


def rank_loss(cost, pred):
    cost = np.ascontiguousarray(cost, dtype=np.float32)
    pred = np.ascontiguousarray(pred, dtype=np.float32)
    return float(lib().or_rank_loss(_p(cost, C.c_float), _p(pred, C.c_float), C.c_int64(len(cost))))


def fit_hist(X, cost, gkey, n_trees=100, depth=6, max_bins=256, group_size=64, eta=0.1, lam=1.0,
             min_child_weight=1.0, seed=1805, want_hist0=False, objective="rank", base_margin=None):
    """objective "rank" (Eq. 2) or "reg" (sum (f - c)^2); base_margin [n]:
    initial predictions (transfer learning, Eq. 4)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, F = X.shape
    cost = np.ascontiguousarray(cost, dtype=np.float32)
    gk = np.ascontiguousarray(gkey, dtype=np.uint16)
    bm = None if base_margin is None else np.ascontiguousarray(base_margin, dtype=np.float32)
    o = FitOpts(n_trees, depth, max_bins, group_size, eta, lam, min_child_weight, seed,
                {"rank": 0, "reg": 1}[objective], None if bm is None else _p(bm, C.c_float))
    ni, nl = (1 << depth) - 1, 1 << depth
    feat = np.zeros((n_trees, ni), np.uint16)
    thr = np.zeros((n_trees, ni), np.float32)
    leaf = np.zeros((n_trees, nl), np.float32)
    pred = np.zeros(n, np.float32)
    h0 = np.zeros((F, max_bins, 2), np.int64) if want_hist0 else None
    rc = lib().or_fit_hist(_p(X, C.c_float), C.c_int64(n), C.c_int(F), _p(cost, C.c_float), _p(gk, C.c_uint16),
                           C.byref(o), _p(feat, C.c_uint16), _p(thr, C.c_float), _p(leaf, C.c_float),
                           _p(pred, C.c_float), None if h0 is None else _p(h0, C.c_int64))
    if rc != 0:
        raise ValueError(f"oracle fit rc={rc}")
    out = dict(feat=feat, thresh=thr, leaf=leaf, pred=pred)
    if want_hist0:
        out["hist0"] = h0
    return out
