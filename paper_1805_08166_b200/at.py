"""Thin ctypes binding of libautotvm_b200.so (include/at_b200.h).

Argument marshalling only: torch tensors supply device memory and the current CUDA
stream; every step of the path runs in the library's sm_100a kernels.  There is no
CPU fallback: if the shared library or a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
# tools may point this at an instrumented build (AT_LIB=...; e.g. the -DAT_CHECKS variant) before the first call
LIB_PATH = Path(os.environ.get("AT_LIB", str(PKG / "libautotvm_b200.so")))
NFEAT = 468

AT_K = dict(features=0, predict=1, sa=2, topk=3, select=4, fit_prep=5, fit_grad=6, fit_hist=7, fit_split=8,
            fit_update=9, fit_graph=10)


class ATError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"at_b200 error {code}: {msg}")
        self.code = code


class Workload(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("kind", "n", "m", "k", "h", "w", "ic", "oc", "ksize", "stride", "pad")]


class SaOpts(C.Structure):
    _fields_ = [("n_chains", C.c_int32), ("n_steps", C.c_int32), ("k_out", C.c_int32), ("init", C.c_int32),
                ("seed", C.c_uint64), ("round", C.c_uint32), ("chain_id_base", C.c_uint32),
                ("d_temps", C.c_void_p), ("d_accept_bits", C.c_void_p), ("d_visited_E", C.c_void_p),
                ("d_visited_idx", C.c_void_p), ("acq", C.c_void_p)]


class SelectOpts(C.Structure):
    _fields_ = [("b", C.c_int32), ("eps", C.c_float), ("alpha", C.c_float), ("seed", C.c_uint64),
                ("round", C.c_uint32)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


class FitOpts(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("depth", C.c_int32), ("max_bins", C.c_int32), ("group_size", C.c_int32),
                ("eta", C.c_float), ("lambda_", C.c_float), ("min_child_weight", C.c_float), ("seed", C.c_uint64),
                ("allreduce", ALLREDUCE_FN), ("ctx", C.c_void_p), ("d_pred_out", C.c_void_p),
                ("d_hist0_out", C.c_void_p), ("objective", C.c_int32), ("d_base_margin", C.c_void_p)]

OBJECTIVES = {"rank": 0, "reg": 1}
KNOB_FEATURES = 32   # AT_KNOB_FEATURES
ACQ = {"mean": 0, "ucb": 1, "ei": 2}   # P:208-215 acquisition over bootstrap models


class AcqOpts(C.Structure):
    _fields_ = [("n_models", C.c_int32), ("kind", C.c_int32), ("kappa", C.c_float), ("best", C.c_float),
                ("model_base", C.c_float * 8)]   # Eq. 2 / sum (f - c)^2


_lib = None


def lib() -> C.CDLL:
    """Load the CUDA library (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ATError(-6, f"{LIB_PATH} missing: run `python -m paper_1805_08166_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        L.at_last_error.restype = C.c_char_p
        L.at_launch_count.restype = C.c_int64
        L.space_create.argtypes = [C.POINTER(Workload), i32, C.POINTER(vp)]
        L.space_info.argtypes = [vp, vp, vp, vp, vp, vp]
        L.space_destroy.argtypes = [vp]
        L.space_check.argtypes = [vp, vp]
        L.features_extract.argtypes = [vp, vp, i64, vp, i64, vp]
        L.features_knobs.argtypes = [vp, vp, i64, vp, i64, vp]
        L.gbt_create.argtypes = [i32, i32, i32, vp, vp, vp, C.c_float, C.POINTER(vp)]
        L.gbt_info.argtypes = [vp, vp, vp, vp]
        L.gbt_export.argtypes = [vp, vp, vp, vp, vp]
        L.gbt_destroy.argtypes = [vp]
        L.gbt_concat.argtypes = [vp, vp, C.POINTER(vp)]
        L.gbt_predict_acq.argtypes = [vp, vp, i64, i64, C.POINTER(AcqOpts), vp, vp, vp, vp]
        L.bootstrap_resample.argtypes = [vp, i64, i64, i32, vp, vp, i32, C.c_uint64, C.c_uint32, vp, i64, vp, vp, vp, vp]
        L.gbt_predict.argtypes = [vp, vp, i64, i64, vp, vp, vp]
        L.sa_explore.argtypes = [vp, vp, vp, vp, vp, vp, i64, C.POINTER(SaOpts), vp, vp, vp, vp]
        L.topk_merge.argtypes = [vp, vp, vp, vp, i32, i32, vp, i64, i32, vp, vp, vp, vp]
        L.select_topk.argtypes = [vp, i32, vp, vp, i64, vp, i64, C.POINTER(SelectOpts), vp, vp, vp]
        L.select_topk_batch.argtypes = [vp, i32, i32, vp, vp, i64, vp, i64, vp, i64, C.POINTER(SelectOpts), vp, vp, vp]
        L.gbt_fit_hist.argtypes = [vp, i64, i64, i32, vp, vp, i64, i64, C.POINTER(FitOpts), C.POINTER(vp), vp]
        L.at_exp_det_eval.argtypes = [C.c_uint32, i64, vp, vp]
        L.at_prof_enable.argtypes = [C.c_int]
        L.at_prof_query.argtypes = [i32, vp, vp]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise ATError(rc, lib().at_last_error().decode())


def _stream(stream=None):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ATError(-1, "expected a CUDA tensor")
    if not t.is_contiguous():
        raise ATError(-1, "expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def _u64(t):
    import torch
    assert t.dtype in (torch.int64, torch.uint64), t.dtype
    return _ptr(t)


def workload(kind=0, **kw) -> Workload:
    w = Workload()
    w.kind = {"matmul": 0, "conv2d": 1, "depthwise": 2}.get(kind, kind)
    for k, v in kw.items():
        setattr(w, k, int(v))
    return w


class Space:
    """S_e over one or more workloads (space_create)."""

    def __init__(self, workloads):
        ws = [w if isinstance(w, Workload) else workload(**w) for w in workloads]
        arr = (Workload * len(ws))(*ws)
        h = C.c_void_p()
        _check(lib().space_create(arr, len(ws), C.byref(h)))
        self.h = h
        self.n_workloads = len(ws)
        tot = C.c_uint64()
        offs = (C.c_uint64 * (len(ws) + 1))()
        rad = (C.c_int32 * (9 * len(ws)))()
        _check(lib().space_info(h, C.byref(tot), None, None, offs, rad))
        self.size_total = int(tot.value)
        self.offsets = [int(x) for x in offs]
        self.radices = [[int(rad[w * 9 + j]) for j in range(9) if rad[w * 9 + j]] for w in range(len(ws))]

    def size(self, w=None):
        return self.size_total if w is None else self.offsets[w + 1] - self.offsets[w]

    def close(self):
        if getattr(self, "h", None):
            lib().space_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, stream=None):
        """Synchronize the stream and raise AT_ERANGE if an earlier call met an out-of-range index."""
        _check(lib().space_check(self.h, _stream(stream)))

    def features(self, idx, out=None, ld=None, stream=None):
        """idx: int64 CUDA tensor of global indices -> SoA [468][ld] float32."""
        import torch
        n = idx.numel()
        if ld is None:
            ld = max(4, (n + 127) // 128 * 128)
        if out is None:
            out = torch.empty((NFEAT, ld), dtype=torch.float32, device=idx.device)
        _check(lib().features_extract(self.h, _u64(idx), n, _ptr(out), ld, _stream(stream)))
        return out

    def knob_features(self, idx, out=None, ld=None, stream=None):
        """Configuration features: idx int64 CUDA tensor -> SoA [32][ld] float32."""
        import torch
        n = idx.numel()
        if ld is None:
            ld = max(4, (n + 127) // 128 * 128)
        if out is None:
            out = torch.empty((KNOB_FEATURES, ld), dtype=torch.float32, device=idx.device)
        _check(lib().features_knobs(self.h, _u64(idx), n, _ptr(out), ld, _stream(stream)))
        return out


class Gbt:
    """GBT ensemble handle (gbt_create / fit output)."""

    def __init__(self, feat=None, thresh=None, leaf=None, base=0.0, n_features=NFEAT, handle=None):
        if handle is not None:
            self.h = handle
        else:
            feat = np.ascontiguousarray(feat, dtype=np.uint16)
            thresh = np.ascontiguousarray(thresh, dtype=np.float32)
            leaf = np.ascontiguousarray(leaf, dtype=np.float32)
            T, nl = leaf.shape
            D = int(round(np.log2(nl)))
            h = C.c_void_p()
            _check(lib().gbt_create(T, D, n_features, feat.ctypes.data_as(C.c_void_p),
                                    thresh.ctypes.data_as(C.c_void_p), leaf.ctypes.data_as(C.c_void_p),
                                    C.c_float(float(base)), C.byref(h)))
            self.h = h
        T, D, F = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().gbt_info(self.h, C.byref(T), C.byref(D), C.byref(F)))
        self.n_trees, self.depth, self.n_features = T.value, D.value, F.value

    def close(self):
        if getattr(self, "h", None):
            lib().gbt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def predict_acq(self, X, n, n_models, kind="ucb", kappa=1.0, best=0.0, model_base=None, stream=None):
        """K = n_models equal concatenated models: (energy, mean, std) per candidate."""
        import torch
        ld = X.shape[1]
        out = [torch.empty(n, dtype=torch.float32, device=X.device) for _ in range(3)]
        mb = (C.c_float * 8)(*([0.0] * 8 if model_base is None else list(model_base) + [0.0] * (8 - len(model_base))))
        o = AcqOpts(n_models, ACQ[kind], kappa, best, mb)
        _check(lib().gbt_predict_acq(self.h, _ptr(X), n, ld, C.byref(o), _ptr(out[0]), _ptr(out[1]), _ptr(out[2]),
                                     _stream(stream)))
        return tuple(out)

    def concat(self, other: "Gbt") -> "Gbt":
        """Eq. 4: self's trees then other's as one ensemble (gbt_concat)."""
        h = C.c_void_p()
        _check(lib().gbt_concat(self.h, other.h, C.byref(h)))
        return Gbt(handle=h)

    def export(self):
        T, D = self.n_trees, self.depth
        feat = np.zeros((T, (1 << D) - 1), np.uint16)
        thr = np.zeros((T, (1 << D) - 1), np.float32)
        leaf = np.zeros((T, 1 << D), np.float32)
        base = C.c_float()
        _check(lib().gbt_export(self.h, feat.ctypes.data_as(C.c_void_p), thr.ctypes.data_as(C.c_void_p),
                                leaf.ctypes.data_as(C.c_void_p), C.byref(base)))
        return dict(feat=feat, thresh=thr, leaf=leaf, base=np.float32(base.value))

    def predict(self, X, n=None, out=None, slots=False, stream=None):
        """X: SoA [F][ld] float32 CUDA tensor -> scores [n] (and leaf slots u8 [T][n])."""
        import torch
        ld = X.shape[1]
        n = ld if n is None else n
        if out is None:
            out = torch.empty(n, dtype=torch.float32, device=X.device)
        sl = torch.empty((self.n_trees, n), dtype=torch.uint8, device=X.device) if slots else None
        _check(lib().gbt_predict(self.h, _ptr(X), n, ld, _ptr(out), _ptr(sl), _stream(stream)))
        return (out, sl) if slots else out


def sa_explore(space: Space, gbt: Gbt, chain_idx, temps, *, seed, round_, k_out, chain_workload=None,
               measured=None, init=False, chain_id_base=0, accept_bits=None, visited=False, acq=None, stream=None):
    """Run the SA kernel; returns dict(out_idx [nw][k], out_score, out_n [nw], chain_energy, ...).
    acq: optional dict(n_models, kind, kappa, best, model_base): the energy is then the acquisition
    over the n_models models concatenated in `gbt`."""
    import torch
    dev = chain_idx.device
    n_chains = chain_idx.numel()
    n_steps = temps.numel()
    o = SaOpts()
    o.n_chains, o.n_steps, o.k_out, o.init = n_chains, n_steps, k_out, 1 if init else 0
    o.seed, o.round, o.chain_id_base = seed, round_, chain_id_base
    o.d_temps = temps.data_ptr()
    if acq is not None:
        mb = list(acq.get("model_base", [])) + [0.0] * 8
        ao = AcqOpts(acq["n_models"], ACQ[acq.get("kind", "ucb")], acq.get("kappa", 1.0), acq.get("best", 0.0),
                     (C.c_float * 8)(*mb[:8]))
        o.acq = C.cast(C.pointer(ao), C.c_void_p)
    res = {}
    if accept_bits is True:
        accept_bits = torch.zeros((n_chains, (n_steps + 31) // 32), dtype=torch.int32, device=dev)
    if accept_bits is not None:
        o.d_accept_bits = accept_bits.data_ptr()
        res["accept_bits"] = accept_bits
    if visited:
        vE = torch.empty((n_chains, n_steps + 1), dtype=torch.float32, device=dev)
        vI = torch.empty((n_chains, n_steps + 1), dtype=torch.int64, device=dev)
        o.d_visited_E, o.d_visited_idx = vE.data_ptr(), vI.data_ptr()
        res["visited_E"], res["visited_idx"] = vE, vI
    nw = space.n_workloads
    out_idx = torch.empty((nw, k_out), dtype=torch.int64, device=dev)
    out_sc = torch.empty((nw, k_out), dtype=torch.float32, device=dev)
    out_n = torch.empty(nw, dtype=torch.int32, device=dev)
    energy = torch.empty(n_chains, dtype=torch.float32, device=dev)
    nm = 0 if measured is None else measured.numel()
    _check(lib().sa_explore(space.h, gbt.h, _u64(chain_idx), _ptr(energy),
                            _ptr(chain_workload) if chain_workload is not None else None,
                            _ptr(measured) if nm else None, nm, C.byref(o), _ptr(out_idx), _ptr(out_sc),
                            _ptr(out_n), _stream(stream)))
    res.update(out_idx=out_idx, out_score=out_sc, out_n=out_n, chain_energy=energy, chain_idx=chain_idx)
    return res


def topk_merge(space: Space, in_idx, in_score, in_n, k_out, measured=None, stream=None):
    """in_*: [n_lists][n_workloads][k_in] (all-gathered per-rank lists) -> distinct top k_out per workload."""
    import torch
    n_lists, nw, k_in = in_idx.shape
    dev = in_idx.device
    out_idx = torch.empty((nw, k_out), dtype=torch.int64, device=dev)
    out_sc = torch.empty((nw, k_out), dtype=torch.float32, device=dev)
    out_n = torch.empty(nw, dtype=torch.int32, device=dev)
    nm = 0 if measured is None else measured.numel()
    _check(lib().topk_merge(space.h, _u64(in_idx), _ptr(in_score), _ptr(in_n), n_lists, k_in,
                            _ptr(measured) if nm else None, nm, k_out, _ptr(out_idx), _ptr(out_sc), _ptr(out_n),
                            _stream(stream)))
    return out_idx, out_sc, out_n


def select_topk(space: Space, workload_id, pool_idx, pool_score, *, b, eps, alpha, seed, round_,
                measured=None, stream=None):
    import torch
    dev = pool_idx.device
    o = SelectOpts(b, eps, alpha, seed, round_)
    out = torch.empty(max(b, 1), dtype=torch.int64, device=dev)
    out_n = torch.empty(1, dtype=torch.int32, device=dev)
    nm = 0 if measured is None else measured.numel()
    _check(lib().select_topk(space.h, workload_id, _u64(pool_idx), _ptr(pool_score), pool_idx.numel(),
                             _ptr(measured) if nm else None, nm, C.byref(o), _ptr(out), _ptr(out_n),
                             _stream(stream)))
    return out, out_n


def select_topk_batch(space: Space, pool_idx, pool_score, pool_n=None, *, b, eps, alpha, seed, round_, w0=0,
                      measured=None, stream=None):
    """Every workload's selection in one launch: pool_idx / pool_score [n_w][k] (e.g. sa_explore's out_idx /
    out_score), pool_n [n_w] int32 device counts (or None: all k) -> (out [n_w][b], out_n [n_w])."""
    import torch
    n_w, k = pool_idx.shape
    dev = pool_idx.device
    o = SelectOpts(b, eps, alpha, seed, round_)
    out = torch.empty((n_w, max(b, 1)), dtype=torch.int64, device=dev)
    out_n = torch.empty(n_w, dtype=torch.int32, device=dev)
    nm = 0 if measured is None else measured.numel()
    _check(lib().select_topk_batch(space.h, w0, n_w, _u64(pool_idx), _ptr(pool_score), k,
                                   _ptr(pool_n) if pool_n is not None else None, k, _ptr(measured) if nm else None, nm,
                                   C.byref(o), _ptr(out), _ptr(out_n), _stream(stream)))
    return out, out_n


def gbt_fit_hist(X, n, cost, group_key, *, n_trees=100, depth=6, max_bins=256, group_size=64, eta=0.1, lam=1.0,
                 min_child_weight=1.0, seed=1805, hist_range=None, allreduce=None, pred_out=None, hist0_out=None,
                 objective="rank", base_margin=None, stream=None) -> Gbt:
    """Histogram GBT refit under the rank loss (objective "rank") or the regression loss ("reg").
    X: SoA [F][ld] CUDA tensor of all n samples; base_margin: optional [n] CUDA float tensor of
    initial predictions (transfer learning: f_global(x_i), Eq. 4).

    allreduce: optional python callable(tensor_view_int64) summing in place across ranks;
    it receives a torch view of the library's device buffer.
    """
    import torch
    F, ld = X.shape
    hb, he = (0, n) if hist_range is None else hist_range
    keep = []
    if allreduce is not None:
        def _cb(ptr, count, ctx, strm):
            try:
                buf = _view_i64(ptr, count, X.device)
                # stream-ordered: the collective runs after the histogram kernels the library enqueued on
                # its stream, and the library's next kernels on that stream run after it
                st = torch.cuda.ExternalStream(strm, device=X.device) if strm else torch.cuda.default_stream(X.device)
                with torch.cuda.stream(st):
                    allreduce(buf)
                return 0
            except Exception as e:  # noqa: BLE001 - reported through the status code
                print("allreduce callback failed:", e, flush=True)
                return -4
        cb = ALLREDUCE_FN(_cb)
        keep.append(cb)
    else:
        cb = ALLREDUCE_FN()
    o = FitOpts(n_trees, depth, max_bins, group_size, eta, lam, min_child_weight, seed, cb, None,
                pred_out.data_ptr() if pred_out is not None else None,
                hist0_out.data_ptr() if hist0_out is not None else None, OBJECTIVES[objective],
                base_margin.data_ptr() if base_margin is not None else None)
    h = C.c_void_p()
    _check(lib().gbt_fit_hist(_ptr(X), n, ld, F, _ptr(cost), _ptr(group_key), hb, he, C.byref(o), C.byref(h),
                              _stream(stream)))
    return Gbt(handle=h)


def bootstrap_resample(X, n, cost, group_key, model, *, seed=1805, round_=0, stream=None):
    """Q40: model `model`'s bootstrap multiset of the n samples -> (X_out [F][n'], cost, keys, idx)."""
    import torch
    F, ld = X.shape
    ldo = (n + 3) // 4 * 4
    Xo = torch.zeros((F, ldo), dtype=torch.float32, device=X.device)
    co = torch.empty(n, dtype=torch.float32, device=X.device)
    ko = torch.empty(n, dtype=torch.int16, device=X.device)
    io = torch.empty(n, dtype=torch.int64, device=X.device)
    _check(lib().bootstrap_resample(_ptr(X), n, ld, F, _ptr(cost), _ptr(group_key), model, seed, round_, _ptr(Xo), ldo,
                                    _ptr(co), _ptr(ko), _ptr(io), _stream(stream)))
    return Xo, co, ko, io


class _CudaArray:
    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<i8", "data": (ptr, False), "version": 3}


def _view_i64(ptr, count, device):
    import torch
    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArray(ptr, count), device=device)


def exp_det_eval(first_bits, n, out=None, stream=None):
    """Device exp_det (reading Q22) of the fp32 values with bits first_bits + i, i < n."""
    import torch
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device="cuda")
    _check(lib().at_exp_det_eval(first_bits, n, _ptr(out), _stream(stream)))
    return out


def launch_count() -> int:
    return int(lib().at_launch_count())


def prof_enable(on=True):
    _check(lib().at_prof_enable(1 if on else 0))


def prof_reset():
    _check(lib().at_prof_reset())


def prof_query(kernel: str):
    n = C.c_int64()
    ms = C.c_double()
    _check(lib().at_prof_query(AT_K[kernel], C.byref(n), C.byref(ms)))
    return int(n.value), float(ms.value)
