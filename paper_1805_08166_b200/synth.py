"""Seeded synthetic inputs shared by tests and bench.py.

This module holds NONE of the method's arithmetic (no decoding, lowering,
features, tree walks, annealing or fitting): it only draws seeded numbers with
numpy and lists the paper's workload shapes.  Both the CUDA path and the CPU
oracle consume its outputs; neither is imported here.

Input recipe:
  * workloads: matmul 512^3, ResNet-18 conv2d C1..C12 (Table 1, P:276-296,
    pad = K // 2), MobileNet-v1 depthwise 3x3 layers (reading Q30);
  * ensembles: complete depth-D trees; internal-node feature uniform over the 466
    non-padding columns, threshold 2^(e/2), e uniform in [0, 42) (spans the
    1 .. 2^20.5 range of the integer-derived features), leaves uniform in
    [-0.1, 0.1) (reading Q38);
  * candidates: uniform flat indices, or the bijection n -> (a n + c) mod |S|
    with a = 2654435761, c = 1805 (config 5, reading Q29);
  * temperatures: geometric T0 -> 0.05 T0 over the steps (reading Q21);
  * labels: a random positive log-linear model of given feature columns times
    lognormal(0, 0.1) noise (stand-in for hardware measurement f).
"""
from __future__ import annotations

import numpy as np

NFEAT = 468
NFEAT_USED = 466          # columns 466, 467 are zero padding (Appendix A)
SEED = 1805

# ---- workloads ---------------------------------------------------------------
MATMUL_512 = dict(kind=0, n=512, m=512, k=512)

# Table 1: (H=W, IC, OC, K, S)
RESNET18 = {
    "C1": (224, 3, 64, 7, 2), "C2": (56, 64, 64, 3, 1), "C3": (56, 64, 64, 1, 1),
    "C4": (56, 64, 128, 3, 2), "C5": (56, 64, 128, 1, 2), "C6": (28, 128, 128, 3, 1),
    "C7": (28, 128, 256, 3, 2), "C8": (28, 128, 256, 1, 2), "C9": (14, 256, 256, 3, 1),
    "C10": (14, 256, 512, 3, 2), "C11": (14, 256, 512, 1, 2), "C12": (7, 512, 512, 3, 1),
}

# MobileNet-v1 224^2 width 1.0 depthwise 3x3 layers (H, C, S), reading Q30
MOBILENET_DW = [(112, 32, 1), (112, 64, 2), (56, 128, 1), (56, 128, 2), (28, 256, 1),
                (28, 256, 2), (14, 512, 1), (14, 512, 2), (7, 1024, 1)]


def conv(h, ic, oc, k, s):
    return dict(kind=1, h=h, w=h, ic=ic, oc=oc, ksize=k, stride=s, pad=k // 2)


def dw(h, c, s, k=3):
    return dict(kind=2, h=h, w=h, ic=c, oc=c, ksize=k, stride=s, pad=k // 2)


def resnet(name):
    return conv(*RESNET18[name])


# config 2: BASELINE.json labels it "C7 (28x28, 128->128, 3x3)"; that shape is Table 1's C6.
CFG2A = conv(28, 128, 128, 3, 1)     # literal shape (reading Q2)
CFG2B = resnet("C7")                 # Table-1 C7
ALL_RESNET = [resnet(f"C{i}") for i in range(1, 13)]
ALL_DW = [dw(*t) for t in MOBILENET_DW]

# tiny pin workloads
MATMUL_8 = dict(kind=0, n=8, m=8, k=8)
CONV_TINY = dict(kind=1, h=4, w=4, ic=2, oc=2, ksize=3, stride=1, pad=1)


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


# ---- ensembles -----------------------------------------------------------------
def ensemble(n_trees: int, depth: int, seed: int = SEED, n_feat_used: int = NFEAT_USED, base: float = 0.0):
    """Complete random trees in heap layout: feat u16 [T][2^D-1], thresh f32, leaf f32 [T][2^D]."""
    g = rng(seed)
    ni, nl = (1 << depth) - 1, 1 << depth
    feat = g.integers(0, n_feat_used, size=(n_trees, ni), dtype=np.int64).astype(np.uint16)
    e = g.integers(0, 42, size=(n_trees, ni))
    thresh = np.power(2.0, e / 2.0).astype(np.float32)
    leaf = ((g.random((n_trees, nl)) - 0.5) * 0.2).astype(np.float32)
    return dict(feat=feat, thresh=thresh, leaf=leaf, base=np.float32(base))


def hand_ensemble():
    """Depth-2, two-tree ensemble with a pass-through tree (SURVEY 8(c) GBT pin)."""
    inf = np.float32(np.inf)
    feat = np.array([[0, 1, 1], [1, 0, 0]], np.uint16)
    thresh = np.array([[2.5, 0.5, 1.5], [1.0, inf, inf]], np.float32)
    leaf = np.array([[1, 2, 3, 4], [0.25, 0.25, -0.5, -0.5]], np.float32)
    return dict(feat=feat, thresh=thresh, leaf=leaf, base=np.float32(0.0))


# ---- candidates / chains ---------------------------------------------------------
def uniform_indices(size: int, n: int, seed: int = SEED, offset: int = 0) -> np.ndarray:
    g = rng(seed)
    return (g.integers(0, size, size=n, dtype=np.uint64) + np.uint64(offset)).astype(np.uint64)


def sweep_indices(size: int, start: int, n: int, a: int = 2654435761, c: int = 1805) -> np.ndarray:
    """Config-5 candidate stream n -> (a n + c) mod |S| (a bijection when gcd(a, |S|) = 1)."""
    k = np.arange(start, start + n, dtype=np.uint64)
    return ((k * np.uint64(a) + np.uint64(c)) % np.uint64(size)).astype(np.uint64)


def temperatures(n_steps: int, t0: float, ratio: float = 0.05) -> np.ndarray:
    """Geometric schedule T0 -> ratio*T0, computed in fp64 and rounded to fp32."""
    if n_steps <= 1:
        return np.full(max(n_steps, 0), t0, dtype=np.float32)
    s = np.arange(n_steps, dtype=np.float64)
    return (t0 * np.power(ratio, s / (n_steps - 1))).astype(np.float32)


def energy_sigma(E) -> float:
    """Reading Q21's T0: the population standard deviation of the chains' initial energies, fp64,
    sequential in chain order (1.0 if it is 0, e.g. a constant model)."""
    e = [float(x) for x in np.asarray(E, dtype=np.float32)]
    if not e:
        return 1.0
    mu = 0.0
    for x in e:
        mu += x
    mu /= len(e)
    var = 0.0
    for x in e:
        var += (x - mu) * (x - mu)
    sd = (var / len(e)) ** 0.5
    return sd if sd > 0.0 else 1.0


def energy_scale(n_trees: int) -> float:
    """Std of a sum of n_trees U(-0.1, 0.1) leaves: the T0 used with synthetic ensembles."""
    return float(0.2 / np.sqrt(12.0) * np.sqrt(n_trees))


def labels(X: np.ndarray, seed: int = SEED, n_terms: int = 12) -> np.ndarray:
    """Synthetic positive costs from a random log-linear model of given feature columns.

    X is [n][468] (row-major) or anything exposing the same column values; the
    model is c = exp(sum_j a_j log2(1 + X[:, col_j]) / n_terms) * lognormal(0, 0.1).
    """
    g = rng(seed)
    n = X.shape[0]
    cols = g.integers(0, NFEAT_USED, size=n_terms)
    a = g.normal(0.0, 1.0, size=n_terms)
    z = np.zeros(n, dtype=np.float64)
    for c, w in zip(cols, a):
        z += w * np.log2(1.0 + np.abs(X[:, c].astype(np.float64)))
    noise = g.normal(0.0, 0.1, size=n)
    return np.exp(z / n_terms + noise).astype(np.float32)


def group_keys(n: int, n_workloads: int, seed: int = SEED) -> np.ndarray:
    return rng(seed + 17).integers(0, n_workloads, size=n).astype(np.uint16)
