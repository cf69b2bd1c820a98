"""GPU parity: the sm_100a library (through the C-ABI) against the CPU oracle.

Every comparison is element by element on the same seeded inputs (paper_1805_08166_b200.synth):
bit-exact for indices, features, leaf slots, accept bits, top-k, selections, histograms and
fitted trees; scores within 1e-6 relative (north_star) -- and in practice bit-exact.
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_1805_08166_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def at():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1805_08166_b200 import at as _at
    from paper_1805_08166_b200 import build
    build.build()
    return _at


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def u64(a):
    return dev(np.asarray(a, dtype=np.uint64).view(np.int64))


def host_u64(t):
    return t.cpu().numpy().view(np.uint64)


def gpu_features(at, space, idx):
    X = space.features(u64(idx))
    return X[:, :len(idx)].cpu().numpy().T.copy()


def assert_bits_equal(a, b, what):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    bad = np.argwhere(a.view(np.uint32) != b.view(np.uint32)) if a.dtype == np.float32 else np.argwhere(a != b)
    assert len(bad) == 0, f"{what}: {len(bad)} mismatches, first {bad[:5].tolist()} gpu={a[tuple(bad[0])]} oracle={b[tuple(bad[0])]}"


# ------------------------------------------------------------------ space
@pytest.mark.parametrize("wls", [[synth.MATMUL_512], [synth.CFG2A], [synth.CFG2B], synth.ALL_RESNET, synth.ALL_DW,
                                 [synth.MATMUL_8, synth.CONV_TINY, synth.ALL_DW[8]]])
def test_space_matches_oracle(at, wls):
    g = at.Space(wls)
    o = O.OracleSpace([O.workload(**w) for w in wls])
    assert g.size_total == o.size()
    assert g.offsets == [o.offset(w) for w in range(len(wls))] + [o.size()]
    for w in range(len(wls)):
        assert g.radices[w] == o.radices(w)


# ------------------------------------------------------------------ features
def test_features_all_of_config1_space(at):
    """Config 1: every one of the 151,250 matmul-512 schedules, bit-exact."""
    sp = at.Space([synth.MATMUL_512])
    osp = O.OracleSpace([O.workload(**synth.MATMUL_512)])
    idx = np.arange(osp.size(), dtype=np.uint64)
    assert_bits_equal(gpu_features(at, sp, idx), osp.features(idx), "features cfg1")


@pytest.mark.parametrize("name,wls,n", [
    ("cfg2a", [synth.CFG2A], 3001), ("cfg2b", [synth.CFG2B], 2999), ("C1", [synth.resnet("C1")], 1500),
    ("resnet-union", synth.ALL_RESNET, 6007), ("dw-union", synth.ALL_DW, 4099),
    ("mixed", [synth.MATMUL_8, synth.CONV_TINY, synth.ALL_DW[3]], 1777)])
def test_features_random_candidates(at, name, wls, n):
    sp = at.Space(wls)
    osp = O.OracleSpace([O.workload(**w) for w in wls])
    idx = synth.uniform_indices(osp.size(), n, seed=hash(name) % 1000)
    idx[:3] = [0, osp.size() - 1, osp.offset(len(wls) - 1)]
    assert_bits_equal(gpu_features(at, sp, idx), osp.features(idx), f"features {name}")


def test_features_edge_cases(at):
    sp = at.Space([synth.CFG2A])
    out = torch.full((468, 128), 7.0, device="cuda")
    sp.features(u64(np.zeros(0, np.uint64)), out=out, ld=128)          # n = 0 is a no-op
    assert torch.all(out == 7.0)
    one = gpu_features(at, sp, np.array([12345], np.uint64))
    osp = O.OracleSpace([O.workload(**synth.CFG2A)])
    assert_bits_equal(one, osp.features(np.array([12345], np.uint64)), "n=1")
    with pytest.raises(at.ATError):
        sp.features(u64(np.zeros(10, np.uint64)), out=torch.empty((468, 8), device="cuda"), ld=8)


# ------------------------------------------------------------------ GBT
def test_hand_ensemble(at):
    e = synth.hand_ensemble()
    g = at.Gbt(e["feat"], e["thresh"], e["leaf"], n_features=2)
    X = dev(np.array([[1, 2.5, 3], [0, 1.5, 0.7]], np.float32))
    s, sl = g.predict(X, slots=True)
    assert s.cpu().tolist() == [1.25, 3.5, 3.25]
    assert sl.cpu().numpy().T.tolist() == [[0, 0], [3, 2], [2, 0]]
    ex = g.export()
    for k in ("feat", "thresh", "leaf"):
        assert np.array_equal(ex[k], e[k])


@pytest.mark.parametrize("T,D,n", [(100, 6, 2048), (37, 3, 1000), (500, 6, 777), (1000, 8, 300), (33, 1, 65),
                                   (2000, 8, 4099), (150, 7, 1000)])
def test_gbt_predict_scores_and_slots(at, T, D, n):
    """Depth >= 7 ensembles that stream go through the rank form (u16 feature ranks, 4-B nodes)."""
    ens = synth.ensemble(T, D, seed=T * 10 + D)
    osp = O.OracleSpace([O.workload(**w) for w in synth.ALL_RESNET])
    idx = synth.uniform_indices(osp.size(), n, seed=T)
    Xo = osp.features(idx)
    sp = at.Space(synth.ALL_RESNET)
    Xg = sp.features(u64(idx))
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"], base=0.125)
    s, sl = g.predict(Xg, n=n, slots=True)
    es, esl = O.OracleGbt(ens["feat"], ens["thresh"], ens["leaf"], base=0.125).predict(Xo, slots=True)
    assert_bits_equal(sl.cpu().numpy(), esl, "leaf slots")
    s = s.cpu().numpy()
    assert np.all(np.abs(s - es) <= 1e-6 * np.maximum(np.abs(es), 1e-30) + 0.0)
    assert_bits_equal(s, es, "scores (canonical order => bit-exact)")


@pytest.mark.parametrize("T,D", [(400, 8), (300, 7)])
def test_predict_rank_form_edge_values(at, T, D):
    """Rank form vs the fp32 walk (AT_PREDICT_RANK=0) on feature values equal to thresholds, -0.0 /
    +0.0, +-inf and NaN, with +inf pass-through and -inf / 0.0 thresholds: same scores, same slots."""
    rng = np.random.default_rng(T)
    ens = synth.ensemble(T, D, seed=T + D)
    th = ens["thresh"]
    th[:, 0] = np.float32(np.inf)                          # roots: pass-through
    th[rng.random(th.shape) < 0.02] = np.float32(-np.inf)
    th[rng.random(th.shape) < 0.02] = np.float32(0.0)
    th[rng.random(th.shape) < 0.02] = np.float32(-0.0)
    n = 3000
    X = np.power(2.0, rng.integers(0, 42, size=(468, n)) / 2.0).astype(np.float32)   # many exact threshold values
    m = rng.random(X.shape)
    X[m < 0.01] = np.float32(-0.0)
    X[(m >= 0.01) & (m < 0.02)] = np.float32(0.0)
    X[(m >= 0.02) & (m < 0.025)] = np.float32(np.inf)
    X[(m >= 0.025) & (m < 0.03)] = np.float32(-np.inf)
    X[(m >= 0.03) & (m < 0.035)] = np.float32(np.nan)
    Xg = dev(np.ascontiguousarray(X))
    g = at.Gbt(ens["feat"], th, ens["leaf"], base=0.5)
    outs = []
    for env in ("1", "0"):
        os.environ["AT_PREDICT_RANK"] = env
        try:
            s, sl = g.predict(Xg, n=n, slots=True)
            outs.append((s.cpu().numpy(), sl.cpu().numpy()))
        finally:
            os.environ.pop("AT_PREDICT_RANK", None)
    assert_bits_equal(outs[0][1], outs[1][1], "leaf slots")
    assert_bits_equal(outs[0][0], outs[1][0], "scores")
    fin = np.all(np.isfinite(X), axis=0)   # the oracle on the finite-feature candidates
    es, esl = O.OracleGbt(ens["feat"], th, ens["leaf"], base=0.5).predict(np.ascontiguousarray(X[:, fin].T), slots=True)
    assert_bits_equal(outs[0][0][fin], es, "scores vs oracle")


@pytest.mark.parametrize("rk_grp", ["2", "4"])
def test_predict_rank_streamed_pass_edge_values(at, rk_grp):
    """The streamed rank pass (no leaf slots asked for: the predict_kernel<..., ONLY = 2> variant, 2 or 4
    candidate groups) on the edge values of the test above plus one feature with 256 distinct thresholds
    (ranks up to 256) and NaN features (rank 0xFFFF, which must go right): scores equal the fp32 walk's
    and, on finite candidates, the oracle's."""
    rng = np.random.default_rng(77)
    T, D = 300, 8
    ens = synth.ensemble(T, D, seed=78)
    th, feat = ens["thresh"], ens["feat"]
    feat[:, 1:40] = 3                                                   # feature 3: 256 distinct thresholds
    th[:, 1:40] = rng.choice(np.arange(256, dtype=np.float32) * 0.5, size=(T, 39))
    th[rng.random(th.shape) < 0.02] = np.float32(np.inf)
    th[rng.random(th.shape) < 0.02] = np.float32(-np.inf)
    th[rng.random(th.shape) < 0.02] = np.float32(-0.0)
    n = 5000
    X = np.power(2.0, rng.integers(0, 42, size=(468, n)) / 2.0).astype(np.float32)
    X[3] = rng.integers(-2, 260, size=n).astype(np.float32) * 0.5      # every rank of feature 3
    m = rng.random(X.shape)
    X[m < 0.01] = np.float32(-0.0)
    X[(m >= 0.01) & (m < 0.02)] = np.float32(np.inf)
    X[(m >= 0.02) & (m < 0.03)] = np.float32(-np.inf)
    X[(m >= 0.03) & (m < 0.04)] = np.float32(np.nan)
    Xg = dev(np.ascontiguousarray(X))
    g = at.Gbt(feat, th, ens["leaf"], base=0.25)
    outs = []
    for env in ("1", "0"):
        os.environ.update(AT_PREDICT_RANK=env, AT_RK_GRP=rk_grp)
        try:
            outs.append(g.predict(Xg, n=n).cpu().numpy())
        finally:
            os.environ.pop("AT_PREDICT_RANK", None)
            os.environ.pop("AT_RK_GRP", None)
    assert_bits_equal(outs[0], outs[1], "scores (rank pass vs fp32 walk)")
    fin = np.all(np.isfinite(X), axis=0)
    es = O.OracleGbt(feat, th, ens["leaf"], base=0.25).predict(np.ascontiguousarray(X[:, fin].T))
    assert_bits_equal(outs[0][fin], es, "scores vs oracle")


def test_predict_rank_form_odd_feature_count(at):
    """F = 7 (the last rank pair has one feature), depth 8, 200 streamed trees; rank vs fp32 vs oracle."""
    rng = np.random.default_rng(5)
    T, D, F, n = 200, 8, 7, 1500
    ni, nl = (1 << D) - 1, 1 << D
    feat = rng.integers(0, F, size=(T, ni)).astype(np.uint16)
    thr = rng.integers(0, 50, size=(T, ni)).astype(np.float32)
    leaf = ((rng.random((T, nl)) - 0.5) * 0.2).astype(np.float32)
    X = rng.integers(0, 50, size=(F, n)).astype(np.float32)
    g = at.Gbt(feat, thr, leaf, n_features=F)
    Xg = dev(np.ascontiguousarray(X))
    outs = []
    for env in ("1", "0"):
        os.environ["AT_PREDICT_RANK"] = env
        try:
            s, sl = g.predict(Xg, n=n, slots=True)
            outs.append((s.cpu().numpy(), sl.cpu().numpy()))
        finally:
            os.environ.pop("AT_PREDICT_RANK", None)
    assert_bits_equal(outs[0][1], outs[1][1], "leaf slots")
    assert_bits_equal(outs[0][0], outs[1][0], "scores")
    es = O.OracleGbt(feat, thr, leaf).predict(np.ascontiguousarray(X.T))
    assert_bits_equal(outs[0][0], es, "scores vs oracle")


def test_predict_rank_form_of_a_fitted_model(at):
    """A device-only handle (gbt_fit_hist output, depth 8) gets its rank tables built lazily on the
    first deep predict; scores and slots equal the fp32 walk's and the oracle's."""
    n = 2500
    osp, idx, X, c, key = fit_inputs(n, synth.ALL_RESNET[:3], seed=41)
    sp = at.Space(synth.ALL_RESNET[:3])
    Xg = sp.features(u64(idx))
    gm = at.gbt_fit_hist(Xg, n, dev(c), dev(key.view(np.int16)), n_trees=120, depth=8)
    ex = gm.export()
    cand = synth.uniform_indices(osp.size(), 3000, seed=42)
    Xc = sp.features(u64(cand))
    outs = []
    for env in ("1", "0"):
        os.environ["AT_PREDICT_RANK"] = env
        try:
            s, sl = gm.predict(Xc, n=3000, slots=True)
            outs.append((s.cpu().numpy(), sl.cpu().numpy()))
        finally:
            os.environ.pop("AT_PREDICT_RANK", None)
    assert_bits_equal(outs[0][1], outs[1][1], "leaf slots")
    assert_bits_equal(outs[0][0], outs[1][0], "scores")
    es = O.OracleGbt(ex["feat"], ex["thresh"], ex["leaf"]).predict(osp.features(cand))
    assert_bits_equal(outs[0][0], es, "scores vs oracle")


def test_scores_config1_exhaustive_top8(at):
    """Config 1 pin: exhaustive scoring of all 151,250 configs; GPU top-8 == oracle top-8."""
    ens = synth.ensemble(100, 6, seed=1805)
    osp = O.OracleSpace([O.workload(**synth.MATMUL_512)])
    idx = np.arange(osp.size(), dtype=np.uint64)
    Xo = osp.features(idx)
    es = O.OracleGbt(**ens).predict(Xo)
    sp = at.Space([synth.MATMUL_512])
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    s = g.predict(sp.features(u64(idx)), n=len(idx)).cpu().numpy()
    assert_bits_equal(s, es, "cfg1 scores")
    o8 = np.lexsort((idx, es))[:8]
    g8 = np.lexsort((idx, s))[:8]
    assert np.array_equal(idx[o8], idx[g8])


# ------------------------------------------------------------------ SA + top-k
def run_both(at, wls, ens, n_chains, n_steps, seed, round_, temps, K, chain_workload=None, chain_idx=None,
             measured=(), chain_id_base=0):
    osp = O.OracleSpace([O.workload(**w) for w in wls])
    oe = O.OracleGbt(**ens)
    r = osp.sa_explore(oe, n_chains, n_steps, seed, round_, temps, chain_id_base=chain_id_base,
                       chain_workload=chain_workload, chain_idx=chain_idx)
    otop = osp.topk(r["visited_E"], r["visited_idx"], K, measured=measured)
    sp = at.Space(wls)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"], base=ens["base"])
    init = chain_idx is None
    cidx = u64(np.zeros(n_chains, np.uint64) if init else chain_idx)
    cw = None if chain_workload is None else dev(np.asarray(chain_workload, np.uint16).view(np.int16))
    meas = u64(np.sort(np.asarray(measured, np.uint64))) if len(measured) else None
    res = at.sa_explore(sp, g, cidx, dev(temps), seed=seed, round_=round_, k_out=K, chain_workload=cw,
                        measured=meas, init=init, chain_id_base=chain_id_base, accept_bits=True, visited=True)
    torch.cuda.synchronize()
    return r, otop, res


def compare_sa(r, otop, res):
    assert_bits_equal(host_u64(res["visited_idx"]), r["visited_idx"], "visited idx")
    assert_bits_equal(res["visited_E"].cpu().numpy(), r["visited_E"], "visited E")
    assert_bits_equal(res["accept_bits"].cpu().numpy().view(np.uint32), r["accept_bits"], "accept bits")
    assert_bits_equal(host_u64(res["chain_idx"]), r["chain_idx"], "final states")
    assert_bits_equal(res["chain_energy"].cpu().numpy(), r["chain_energy"], "final energies")
    on = res["out_n"].cpu().numpy()
    for w, (oi, oE) in enumerate(otop):
        assert on[w] == len(oi)
        assert_bits_equal(host_u64(res["out_idx"][w, :on[w]]), oi, f"top-k idx w{w}")
        assert_bits_equal(res["out_score"][w, :on[w]].cpu().numpy(), oE, f"top-k E w{w}")


def test_sa_tiny_space_exhaustive(at):
    """Chains started at every config of the matmul-8^3 space: top-k == exhaustive ranking."""
    ens = synth.ensemble(40, 6, seed=4)
    N = 2000
    temps = synth.temperatures(5, 0.3)
    r, otop, res = run_both(at, [synth.MATMUL_8], ens, N, 5, 5, 0, temps, 64, chain_idx=np.arange(N, dtype=np.uint64))
    compare_sa(r, otop, res)


@pytest.mark.parametrize("T,D,steps,chains", [(500, 6, 40, 70), (100, 6, 33, 96), (60, 8, 20, 33)])
def test_sa_conv_parity(at, T, D, steps, chains):
    ens = synth.ensemble(T, D, seed=T + D)
    temps = synth.temperatures(steps, synth.energy_scale(T))
    r, otop, res = run_both(at, [synth.CFG2A], ens, chains, steps, 1805, 3, temps, 128)
    compare_sa(r, otop, res)


def test_sa_union_with_measured_and_persistence(at):
    ens = synth.ensemble(120, 6, seed=77)
    n_chains, steps = 48, 24
    cw = (np.arange(n_chains) % 12).astype(np.uint16)
    temps = synth.temperatures(steps, synth.energy_scale(120))
    r, otop, res = run_both(at, synth.ALL_RESNET, ens, n_chains, steps, 9, 0, temps, 16, chain_workload=cw)
    compare_sa(r, otop, res)
    # round 1 from the persisted states, excluding some measured configs
    meas = np.concatenate([otop[w][0][:3] for w in range(12)])
    r2, otop2, res2 = run_both(at, synth.ALL_RESNET, ens, n_chains, steps, 9, 1, temps, 16, chain_workload=cw,
                               chain_idx=r["chain_idx"], measured=meas)
    compare_sa(r2, otop2, res2)


def test_sa_edge_temperatures_and_zero_steps(at):
    ens = synth.ensemble(50, 5, seed=3)
    for temps in (np.full(20, np.inf, np.float32), np.zeros(20, np.float32), np.zeros(0, np.float32)):
        r, otop, res = run_both(at, [synth.CFG2B], ens, 40, len(temps), 2, 0, temps, 32)
        compare_sa(r, otop, res)


def test_sa_full_config2_sampled_chains(at):
    """Config 2 at its benchmark size (4096 chains x 500 steps, 500 trees): chains sampled one by one."""
    ens = synth.ensemble(500, 6, seed=1805)
    steps = 500
    temps = synth.temperatures(steps, synth.energy_scale(500))
    sp = at.Space([synth.CFG2A])
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    res = at.sa_explore(sp, g, u64(np.zeros(4096, np.uint64)), dev(temps), seed=1805, round_=0, k_out=128,
                        init=True, accept_bits=True, visited=True)
    torch.cuda.synchronize()
    osp = O.OracleSpace([O.workload(**synth.CFG2A)])
    oe = O.OracleGbt(**ens)
    for c in (0, 1, 2047, 4095):
        r = osp.sa_explore(oe, 1, steps, 1805, 0, temps, chain_id_base=c)
        assert_bits_equal(res["accept_bits"][c:c + 1].cpu().numpy().view(np.uint32), r["accept_bits"], f"chain {c}")
        assert_bits_equal(host_u64(res["visited_idx"][c:c + 1]), r["visited_idx"], f"chain {c} idx")
    # the returned top-k is the distinct top-k of the visited set (checked with numpy on the GPU's visited set,
    # whose entries are themselves oracle-checked above on samples)
    vE = res["visited_E"].cpu().numpy().ravel()
    vI = host_u64(res["visited_idx"]).ravel()
    o = np.lexsort((vI, vE))
    _, first = np.unique(vI[o], return_index=True)
    keep = o[np.sort(first)][:128]
    assert np.array_equal(host_u64(res["out_idx"][0]), vI[keep])


def test_topk_merge_matches_oracle(at):
    wls = [synth.CFG2A, synth.CFG2B]
    osp = O.OracleSpace([O.workload(**w) for w in wls])
    rng = np.random.default_rng(0)
    L, K = 5, 40
    idx = np.zeros((L, 2, K), np.uint64)
    sc = np.zeros((L, 2, K), np.float32)
    cnt = rng.integers(0, K + 1, size=(L, 2)).astype(np.int32)
    pool = {w: synth.uniform_indices(osp.size(w), 90, seed=w) + np.uint64(osp.offset(w)) for w in range(2)}
    score_of = {int(i): np.float32(rng.integers(0, 20) / 8) for w in range(2) for i in pool[w]}   # many ties
    for l in range(L):
        for w in range(2):
            pick = rng.choice(pool[w], size=K, replace=False)
            idx[l, w] = pick
            sc[l, w] = [score_of[int(i)] for i in pick]
    meas = np.sort(pool[0][:7])
    allE, allI = [], []
    for l in range(L):
        for w in range(2):
            allE += list(sc[l, w, :cnt[l, w]])
            allI += list(idx[l, w, :cnt[l, w]])
    otop = osp.topk(np.array(allE, np.float32), np.array(allI, np.uint64), 30, measured=meas)
    sp = at.Space(wls)
    gi, gs, gn = at.topk_merge(sp, u64(idx), dev(sc), dev(cnt), 30, measured=u64(meas))
    for w in range(2):
        n = int(gn[w])
        assert n == len(otop[w][0])
        assert_bits_equal(host_u64(gi[w, :n]), otop[w][0], "merge idx")
        assert_bits_equal(gs[w, :n].cpu().numpy(), otop[w][1], "merge E")


# ------------------------------------------------------------------ select
@pytest.mark.parametrize("b,eps,alpha,n_pool", [(64, 0.05, 0.1, 128), (64, 0.0, 0.0, 128), (8, 0.0, 0.0, 8),
                                                (64, 0.05, 1.0, 40), (16, 0.5, 0.3, 100), (64, 0.05, 0.1, 1000)])
def test_select_matches_oracle(at, b, eps, alpha, n_pool):
    wls = synth.ALL_RESNET
    osp = O.OracleSpace([O.workload(**w) for w in wls])
    w = 6
    pool = synth.uniform_indices(osp.size(w), n_pool, seed=n_pool) + np.uint64(osp.offset(w))
    E = (np.random.default_rng(b).integers(0, 50, n_pool) / 16).astype(np.float32)   # ties on purpose
    o = np.lexsort((pool, E))
    pool, E = pool[o], E[o]
    meas = np.sort(np.concatenate([synth.uniform_indices(osp.size(w), 30, seed=5) + np.uint64(osp.offset(w)),
                                   np.array([1, 2, 3], np.uint64)]))
    ref = osp.select(w, pool, E, b, eps, alpha, seed=11, round_=2, measured=meas)
    sp = at.Space(wls)
    out, n = at.select_topk(sp, w, u64(pool), dev(E), b=b, eps=eps, alpha=alpha, seed=11, round_=2,
                            measured=u64(meas))
    assert int(n) == len(ref)
    assert_bits_equal(host_u64(out[:int(n)]), ref, "selection")


def test_select_exhausted_space(at):
    wl = dict(kind=0, n=1, m=1, k=2)
    osp = O.OracleSpace([O.workload(**wl)])
    meas = np.array([0, 1, 2, 3], np.uint64)
    pool = np.array([4, 5], np.uint64)
    E = np.array([0.1, 0.2], np.float32)
    ref = osp.select(0, pool, E, 20, 0.5, 0.0, 1, 0, measured=meas)
    sp = at.Space([wl])
    out, n = at.select_topk(sp, 0, u64(pool), dev(E), b=20, eps=0.5, alpha=0.0, seed=1, round_=0, measured=u64(meas))
    assert_bits_equal(host_u64(out[:int(n)]), ref, "exhausted")


# ------------------------------------------------------------------ refit
def fit_inputs(n, wls, seed):
    osp = O.OracleSpace([O.workload(**w) for w in wls])
    key = synth.group_keys(n, len(wls), seed=seed)
    idx = np.array([osp.offset(int(k)) + int(v) for k, v in
                    zip(key, synth.uniform_indices(1 << 62, n, seed=seed) % np.array([osp.size(int(k)) for k in key],
                                                                                     dtype=np.uint64))], np.uint64)
    X = osp.features(idx)
    return osp, idx, X, synth.labels(X, seed=seed), key


@pytest.mark.parametrize("n,wls,trees,depth", [(1500, [synth.CFG2A, synth.CFG2B], 6, 4),
                                               (700, synth.ALL_DW[:3], 4, 6),
                                               (3000, [synth.MATMUL_512], 3, 5)])
@pytest.mark.parametrize("path", ["subtraction", "level-by-level"])
def test_fit_matches_oracle(at, n, wls, trees, depth, path):
    """hist0_out (the parity hook for tree 0's root histogram) routes around the fused forest."""
    osp, idx, X, c, key = fit_inputs(n, wls, seed=n)
    ref = O.fit_hist(X, c, key, n_trees=trees, depth=depth, want_hist0=True)
    sp = at.Space(wls)
    Xg = sp.features(u64(idx))
    pred = torch.empty(n, dtype=torch.float32, device="cuda")
    h0 = torch.empty((468, 256, 2), dtype=torch.int64, device="cuda")
    os.environ.update(FIT_PATHS[path])
    try:
        g = at.gbt_fit_hist(Xg, n, dev(c), dev(key.view(np.int16)), n_trees=trees, depth=depth, pred_out=pred,
                            hist0_out=h0)
    finally:
        for k in FIT_PATHS[path]:
            os.environ.pop(k, None)
    ex = g.export()
    assert_bits_equal(h0.cpu().numpy(), ref["hist0"], "root histogram of tree 0")
    assert_bits_equal(ex["feat"], ref["feat"], "split features")
    assert_bits_equal(ex["thresh"], ref["thresh"], "thresholds")
    assert_bits_equal(ex["leaf"], ref["leaf"], "leaves")
    assert_bits_equal(pred.cpu().numpy(), ref["pred"], "fit predictions")


def test_fit_many_unique_values_uses_quantile_cuts(at):
    n = 2000
    rng = np.random.default_rng(3)
    X = np.zeros((n, 468), np.float32)
    X[:, :40] = rng.random((n, 40)).astype(np.float32) * 1000        # > 256 unique values
    X[:, 40:80] = rng.integers(0, 5, (n, 40)).astype(np.float32)
    c = (X[:, 0] + 3 * X[:, 41] + rng.random(n)).astype(np.float32)
    key = np.zeros(n, np.uint16)
    ref = O.fit_hist(X, c, key, n_trees=3, depth=4)
    Xg = dev(np.ascontiguousarray(np.pad(X, ((0, 48), (0, 0))).T))
    g = __import__("paper_1805_08166_b200").at.gbt_fit_hist(Xg, n, dev(c), dev(key.view(np.int16)), n_trees=3, depth=4)
    ex = g.export()
    for k in ("feat", "thresh", "leaf"):
        assert_bits_equal(ex[k], ref[k], k)


def test_fit_rank_invariance_two_emulated_ranks(at):
    """Histogram slices + all-reduce: 2 ranks emulated with 2 host threads and 2 streams on one GPU
    (host-side barrier, no kernel waits on another) give the bit-identical ensemble."""
    import threading
    n = 1200
    osp, idx, X, c, key = fit_inputs(n, [synth.CFG2A], seed=9)
    sp = at.Space([synth.CFG2A])
    Xg = sp.features(u64(idx))
    cg, kg = dev(c), dev(key.view(np.int16))
    single = at.gbt_fit_hist(Xg, n, cg, kg, n_trees=4, depth=5).export()
    torch.cuda.synchronize()
    bar = threading.Barrier(2)
    bufs = [None, None]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    out = [None, None]

    def make_ar(r):
        def ar(t):
            streams[r].synchronize()
            bufs[r] = t
            bar.wait()
            if r == 0:
                s = bufs[0] + bufs[1]
                bufs[0].copy_(s)
                bufs[1].copy_(s)
                torch.cuda.synchronize()
            bar.wait()
        return ar

    def run(r):
        with torch.cuda.stream(streams[r]):
            rng = (0, n // 2) if r == 0 else (n // 2, n)
            out[r] = at.gbt_fit_hist(Xg, n, cg, kg, n_trees=4, depth=5, hist_range=rng, allreduce=make_ar(r),
                                     stream=streams[r])
            streams[r].synchronize()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    for r in range(2):
        ex = out[r].export()
        for k in ("feat", "thresh", "leaf"):
            assert_bits_equal(ex[k], single[k], f"rank {r} {k}")


def _emulated_ranks(at, R, Xg, n, cg, kg, **kw):
    """R ranks as R host threads + R streams on one GPU: each fits over its sample slice; the all-reduce is a
    host barrier + a device sum (no kernel ever waits on another rank's kernel)."""
    import threading
    from paper_1805_08166_b200 import dist as D
    bar = threading.Barrier(R)
    bufs = [None] * R
    streams = [torch.cuda.Stream() for _ in range(R)]
    out = [None] * R
    err = []

    def make_ar(r):
        def ar(t):
            torch.cuda.current_stream().synchronize()
            bufs[r] = t
            bar.wait()
            if r == 0:
                s = bufs[0].clone()
                for q in range(1, R):
                    s += bufs[q]
                for q in range(R):
                    bufs[q].copy_(s)
                torch.cuda.synchronize()
            bar.wait()
        return ar

    def run(r):
        try:
            with torch.cuda.stream(streams[r]):
                out[r] = at.gbt_fit_hist(Xg, n, cg, kg, hist_range=D.sample_slice(n, r, R), allreduce=make_ar(r),
                                         stream=streams[r], **kw)
                streams[r].synchronize()
        except Exception as e:   # noqa: BLE001
            err.append(e)
            bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(R)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not err, err
    return out


@pytest.mark.parametrize("n,R,trees,depth,nw", [(100000, 2, 3, 6, 9), (5000, 3, 4, 5, 3), (20000, 8, 2, 7, 9)])
def test_fit_subtraction_path_rank_invariance(at, n, R, trees, depth, nw):
    """Eq. 2: the multi-rank subtraction path -- every rank builds the smaller
    children's histograms over its own sample slice, one int64 all-reduce per level -- gives the
    bit-identical ensemble of the single-rank fit (emulated ranks, n > 2048)."""
    wls = synth.ALL_DW[:nw]
    sp = at.Space(wls)
    key = synth.group_keys(n, nw, seed=n)
    sizes = np.array([sp.size(w) for w in range(nw)], dtype=np.uint64)
    loc = synth.uniform_indices(1 << 62, n, seed=n + 1) % sizes[key]
    idx = loc + np.array(sp.offsets[:nw], dtype=np.uint64)[key]
    Xg = sp.features(u64(idx))
    c = synth.labels(Xg[:, :n].T.cpu().numpy(), seed=n + 2)
    cg, kg = dev(c), dev(key.view(np.int16))
    single = at.gbt_fit_hist(Xg, n, cg, kg, n_trees=trees, depth=depth).export()
    torch.cuda.synchronize()
    out = _emulated_ranks(at, R, Xg, n, cg, kg, n_trees=trees, depth=depth)
    for r in range(R):
        ex = out[r].export()
        for k in ("feat", "thresh", "leaf"):
            assert_bits_equal(ex[k], single[k], f"rank {r} {k}")


FIT_PATHS = {"fused": {"AT_FIT_FUSED": "1"},                          # single launch (n <= 2048)
             "subtraction": {"AT_FIT_FUSED": "0"},                   # default above 2048
             "level-by-level": {"AT_FIT_FUSED": "0", "AT_FIT_SUB": "0"}}


def _fit_paths(at, Xg, n, c, key, paths=tuple(FIT_PATHS), **kw):
    """The fit through each single-rank path (env-selected), predictions included."""
    out = {}
    for name in paths:
        os.environ.update(FIT_PATHS[name])
        try:
            pred = torch.empty(n, dtype=torch.float32, device="cuda")
            ex = at.gbt_fit_hist(Xg, n, dev(c), dev(key.view(np.int16)), pred_out=pred, **kw).export()
            ex["pred"] = pred.cpu().numpy()
            out[name] = ex
        finally:
            for k in FIT_PATHS[name]:
                os.environ.pop(k, None)
    return out


def _check_paths(outs, ref, keys=("feat", "thresh", "leaf", "pred")):
    for name, ex in outs.items():
        for k in keys:
            assert_bits_equal(ex[k], ref[k], f"{name} {k}")


@pytest.mark.parametrize("n,wls,trees,depth,gs", [(1024, [synth.CFG2A], 5, 6, 64),     # bench's |D|
                                                  (2048, synth.ALL_RESNET[:4], 3, 8, 64),
                                                  (333, synth.ALL_DW[:5], 4, 3, 2),
                                                  (1000, [synth.MATMUL_512], 3, 5, 1024),
                                                  (1, [synth.CFG2A], 2, 4, 64),
                                                  (37, [synth.CFG2A, synth.CFG2B], 3, 1, 8),
                                                  (1536, synth.ALL_RESNET, 3, 6, 64),       # config 3's |D|: 192 threads
                                                  (1100, synth.ALL_DW[:3], 2, 5, 64),       # 160 threads
                                                  (1700, synth.ALL_RESNET[:6], 2, 6, 128)])  # 224 threads
def test_fit_fused_forest_matches_oracle(at, n, wls, trees, depth, gs):
    osp, idx, X, c, key = fit_inputs(n, wls, seed=n + depth)
    ref = O.fit_hist(X, c, key, n_trees=trees, depth=depth, group_size=gs)
    sp = at.Space(wls)
    Xg = sp.features(u64(idx))
    _check_paths(_fit_paths(at, Xg, n, c, key, n_trees=trees, depth=depth, group_size=gs), ref)


def test_fit_fused_forest_many_features_and_ties(at):
    """F = 1500 random features (more than one cooperative block per feature, so per-feature order
    state round-trips through global memory), duplicated columns (exact gain ties broken by the lower
    feature), constant columns, equal costs inside groups."""
    n, F = 900, 1500
    rng = np.random.default_rng(21)
    X = rng.integers(0, 40, (n, F)).astype(np.float32)
    X[:, 700:800] = X[:, 100:200]                   # duplicates of earlier features
    X[:, 800:850] = 3.0                             # constant
    X[:, 850:900] = rng.random((n, 50)).astype(np.float32) * 1e4
    c = np.round(X[:, 100] + 2 * X[:, 150] + rng.integers(0, 3, n), 0).astype(np.float32)
    key = (np.arange(n) % 7).astype(np.uint16)
    ref = O.fit_hist(X, c, key, n_trees=3, depth=5)
    Xg = dev(np.ascontiguousarray(X.T))
    _check_paths(_fit_paths(at, Xg, n, c, key, n_trees=3, depth=5), ref)


@pytest.mark.parametrize("n,wls,trees,depth", [(20000, synth.ALL_DW, 3, 6),
                                               (9000, synth.ALL_RESNET[:4], 2, 8),
                                               (2049, [synth.CFG2A], 3, 3)])
def test_fit_subtraction_path_matches_oracle(at, n, wls, trees, depth):
    """Histogram subtraction over node-contiguous positions (the single-rank path above 2048
    samples) and the plain level-by-level path against the oracle."""
    osp, idx, X, c, key = fit_inputs(n, wls, seed=n + 11)
    ref = O.fit_hist(X, c, key, n_trees=trees, depth=depth)
    Xg = at.Space(wls).features(u64(idx))
    _check_paths(_fit_paths(at, Xg, n, c, key, paths=("subtraction", "level-by-level"), n_trees=trees, depth=depth), ref)


def test_fit_subtraction_many_feature_ranges(at):
    """F = 1500 features with up to 256 bins each: the cells of the splittable features span many
    shared-memory ranges (one histogram block per range); quantile cuts, duplicated and constant
    columns, zero-gradient groups (equal costs)."""
    n, F = 5000, 1500
    rng = np.random.default_rng(33)
    X = rng.integers(0, 200, (n, F)).astype(np.float32)
    X[:, 1000:1100] = rng.random((n, 100)).astype(np.float32) * 1e4     # > 256 unique: quantile cuts
    X[:, 1100:1200] = X[:, 200:300]                                      # duplicates
    X[:, 1200:1250] = 7.0                                                # constant
    c = np.round(X[:, 5] + 2 * X[:, 1010] / 100 + rng.integers(0, 3, n), 0).astype(np.float32)
    c[:64] = 1.0                                                         # one group of equal costs
    key = (np.arange(n) % 3).astype(np.uint16)
    ref = O.fit_hist(X, c, key, n_trees=2, depth=6, want_hist0=False)
    Xg = dev(np.ascontiguousarray(X.T))
    _check_paths(_fit_paths(at, Xg, n, c, key, paths=("subtraction", "level-by-level"), n_trees=2, depth=6), ref)


@pytest.mark.parametrize("F,kind", [(1, "quantile"), (1, "constant"), (33, "mixed"), (2, "binary")])
def test_fit_subtraction_few_features(at, F, kind):
    """Edge layouts of the device-computed subtraction path (one feature range, a single stripe of 1-2
    features, one column past a stripe, a lone constant feature) against the oracle, n = 2500, depth 7."""
    n = 2500
    rng = np.random.default_rng(F * 7 + len(kind))
    if kind == "quantile":
        X = (rng.random((n, F)) * 1e3).astype(np.float32)           # > 256 unique values: 255 cuts
    elif kind == "constant":
        X = np.full((n, F), 4.0, np.float32)
    elif kind == "binary":
        X = rng.integers(0, 2, (n, F)).astype(np.float32)
    else:
        X = rng.integers(0, 300, (n, F)).astype(np.float32)
        X[:, 5] = 1.0
    c = (1.0 + rng.random(n) + (X[:, 0] if kind != "constant" else 0) / 500).astype(np.float32)
    key = (np.arange(n) % 3).astype(np.uint16)
    ref = O.fit_hist(X, c, key, n_trees=2, depth=7)
    Xg = dev(np.ascontiguousarray(X.T))
    _check_paths(_fit_paths(at, Xg, n, c, key, paths=("subtraction",), n_trees=2, depth=7), ref)


def test_fit_subtraction_no_splittable_feature(at):
    """Every feature constant (no cut anywhere) on the subtraction path: its device layout lets feature 0
    (one bin) stand in, so the root totals still come from a histogram and every node is a pass-through
    (threshold +inf, leaves = the Newton step of the totals), as the oracle builds it."""
    n = 3000
    rng = np.random.default_rng(5)
    X = np.full((n, 468), 2.0, np.float32)
    c = (1.0 + rng.random(n)).astype(np.float32)
    key = (np.arange(n) % 4).astype(np.uint16)
    ref = O.fit_hist(X, c, key, n_trees=2, depth=4)
    Xg = dev(np.ascontiguousarray(X.T))
    _check_paths(_fit_paths(at, Xg, n, c, key, paths=("subtraction", "level-by-level"), n_trees=2, depth=4), ref)


def test_fit_subtraction_large_gradients(at):
    """Regression on costs of order 10^4: |g| = 2 |f - c| 2^32 reaches 2^46, so the 64-bit histogram sums
    need their carries (low word -> high word) at every level."""
    n = 3000
    osp, idx, X, c, key = fit_inputs(n, [synth.CFG2A, synth.CFG2B], seed=77)
    c = (c / c.max() * 2.0e4 + 3000.0).astype(np.float32)
    ref = O.fit_hist(X, c, key, n_trees=3, depth=5, objective="reg")
    Xg = at.Space([synth.CFG2A, synth.CFG2B]).features(u64(idx))
    _check_paths(_fit_paths(at, Xg, n, c, key, paths=("subtraction", "level-by-level"), n_trees=3, depth=5,
                            objective="reg"), ref)


# ------------------------------------------------------------------ §8(f): regression objective, transfer (Eq. 4)
@pytest.mark.parametrize("n,wls,trees,depth,margin", [(1024, [synth.CFG2A], 4, 6, False),
                                                      (333, synth.ALL_DW[:5], 3, 4, True),
                                                      (2048, synth.ALL_RESNET[:4], 2, 8, False),
                                                      (37, [synth.CFG2B], 3, 2, True)])
def test_fit_regression_matches_oracle(at, n, wls, trees, depth, margin):
    """P:175 regression objective (g = 2 (f - c), h = 2), optionally on top of a base margin, in both
    the fused single-launch forest and the level-by-level path."""
    osp, idx, X, c, key = fit_inputs(n, wls, seed=3 * n + depth)
    m = np.random.default_rng(n).normal(0, 0.5, n).astype(np.float32) if margin else None
    ref = O.fit_hist(X, c, key, n_trees=trees, depth=depth, objective="reg", base_margin=m)
    Xg = at.Space(wls).features(u64(idx))
    kw = dict(n_trees=trees, depth=depth, objective="reg")
    if margin:
        kw["base_margin"] = dev(m)
    _check_paths(_fit_paths(at, Xg, n, c, key, **kw), ref)


@pytest.mark.parametrize("n,trees,depth", [(1024, 5, 6), (3000, 3, 5)])
def test_fit_rank_with_base_margin_matches_oracle(at, n, trees, depth):
    """Rank loss (Eq. 2) fitted on top of per-sample initial predictions (both paths)."""
    osp, idx, X, c, key = fit_inputs(n, [synth.CFG2A, synth.CFG2B], seed=n + 7)
    m = np.random.default_rng(n + 1).normal(0, 1.0, n).astype(np.float32)
    ref = O.fit_hist(X, c, key, n_trees=trees, depth=depth, base_margin=m)
    Xg = at.Space([synth.CFG2A, synth.CFG2B]).features(u64(idx))
    _check_paths(_fit_paths(at, Xg, n, c, key, n_trees=trees, depth=depth, base_margin=dev(m)), ref)


def test_gbt_concat_matches_oracle(at):
    """gbt_concat (Eq. 4): a depth-8 and a depth-5 ensemble become one depth-8 ensemble whose
    arrays and scores equal the oracle's concatenation bit for bit."""
    a, b = synth.ensemble(70, 8, seed=11), synth.ensemble(45, 5, seed=12)
    ga, gb = at.Gbt(a["feat"], a["thresh"], a["leaf"], base=0.25), at.Gbt(b["feat"], b["thresh"], b["leaf"], base=-1.5)
    cat = ga.concat(gb).export()
    ref = O.gbt_concat(O.OracleGbt(a["feat"], a["thresh"], a["leaf"], base=0.25),
                       O.OracleGbt(b["feat"], b["thresh"], b["leaf"], base=-1.5))
    for k in ("feat", "thresh", "leaf"):
        assert_bits_equal(cat[k], getattr(ref, k), k)
    assert np.float32(cat["base"]) == np.float32(ref.base)
    sp = at.Space([synth.CFG2A])
    idx = synth.uniform_indices(sp.size(), 3000, seed=13)
    X = sp.features(u64(idx))
    got = at.Gbt(cat["feat"], cat["thresh"], cat["leaf"], base=cat["base"]).predict(X, 3000)
    assert_bits_equal(got.cpu().numpy(), ref.predict(X[:, :3000].cpu().numpy().T.copy()), "concat scores")


def test_transfer_learning_pipeline_matches_oracle(at):
    """Eq. 4 end to end: a global model on history of C1-C6, its scores on the target's samples as
    the margin of the local fit, then f_global + f_local as one ensemble scoring new candidates."""
    hist_wls, tgt = synth.ALL_RESNET[:6], synth.CFG2B
    _, hidx, HX, hc, hkey = fit_inputs(1500, hist_wls, seed=41)
    gref = O.fit_hist(HX, hc, hkey, n_trees=8, depth=6)
    gg = at.gbt_fit_hist(at.Space(hist_wls).features(u64(hidx)), 1500, dev(hc), dev(hkey.view(np.int16)),
                         n_trees=8, depth=6)
    ge = gg.export()
    for k in ("feat", "thresh", "leaf"):
        assert_bits_equal(ge[k], gref[k], f"global {k}")
    osp, tidx, TX, tc, tkey = fit_inputs(400, [tgt], seed=42)
    tsp = at.Space([tgt])
    TXg = tsp.features(u64(tidx))
    margin_g = gg.predict(TXg, 400)
    og = O.OracleGbt(gref["feat"], gref["thresh"], gref["leaf"])
    margin_o = og.predict(TX)
    assert_bits_equal(margin_g.cpu().numpy(), margin_o, "global scores on the target samples")
    lref = O.fit_hist(TX, tc, tkey, n_trees=6, depth=4, base_margin=margin_o)
    lg = at.gbt_fit_hist(TXg, 400, dev(tc), dev(tkey.view(np.int16)), n_trees=6, depth=4, base_margin=margin_g)
    le = lg.export()
    for k in ("feat", "thresh", "leaf"):
        assert_bits_equal(le[k], lref[k], f"local {k}")
    cat_o = O.gbt_concat(og, O.OracleGbt(lref["feat"], lref["thresh"], lref["leaf"]))
    cidx = synth.uniform_indices(osp.size(), 2000, seed=43)
    got = gg.concat(lg).predict(tsp.features(u64(cidx)), 2000)
    assert_bits_equal(got.cpu().numpy(), cat_o.predict(osp.features(cidx)), "transfer model scores")


# ------------------------------------------------------------------ §8(f): bootstrap uncertainty, EI / UCB
def test_bootstrap_resample_matches_oracle(at):
    """Q40 multisets: the drawn indices and the gathered features / costs / keys."""
    osp, idx, X, c, key = fit_inputs(777, [synth.CFG2A, synth.CFG2B], seed=5)
    Xg = at.Space([synth.CFG2A, synth.CFG2B]).features(u64(idx))
    for k in range(3):
        Xo, co, ko, io = at.bootstrap_resample(Xg, 777, dev(c), dev(key.view(np.int16)), k, seed=31, round_=2)
        ref = O.bootstrap_indices(777, k, seed=31, round_=2)
        assert_bits_equal(io.cpu().numpy(), ref, f"model {k} indices")
        assert_bits_equal(Xo[:, :777].cpu().numpy().T.copy(), X[ref], "gathered features")
        assert_bits_equal(co.cpu().numpy(), c[ref], "gathered costs")
        assert_bits_equal(ko.cpu().numpy().view(np.uint16), key[ref], "gathered keys")


@pytest.mark.parametrize("kind", ["mean", "ucb", "ei"])
def test_predict_acq_matches_oracle(at, kind):
    """K = 5 models of 37 trees (not a multiple of 32) and mixed depths, concatenated: every model's
    canonical score, then mean / std / acquisition, bit for bit against the oracle."""
    depths = [6, 4, 6, 5, 6]
    ens = [synth.ensemble(37, d, seed=60 + k) for k, d in enumerate(depths)]
    bases = [0.0, 0.5, -0.25, 1.0, 0.0]
    gs = [at.Gbt(e["feat"], e["thresh"], e["leaf"], base=b) for e, b in zip(ens, bases)]
    cat = gs[0]
    for g in gs[1:]:
        cat = cat.concat(g)
    sp = at.Space([synth.CFG2A])
    idx = synth.uniform_indices(sp.size(), 2500, seed=61)
    Xg = sp.features(u64(idx))
    sc, mu, sd = cat.predict_acq(Xg, 2500, 5, kind=kind, kappa=1.5, best=-0.3, model_base=bases)
    om = [O.OracleGbt(e["feat"], e["thresh"], e["leaf"], base=b) for e, b in zip(ens, bases)]
    X = Xg[:, :2500].cpu().numpy().T.copy()
    rs, rm, rsd = O.predict_acq(om, X, kind=kind, kappa=1.5, best=-0.3)
    assert_bits_equal(mu.cpu().numpy(), rm, "mean")
    assert_bits_equal(sd.cpu().numpy(), rsd, "std")
    assert_bits_equal(sc.cpu().numpy(), rs, kind)
    assert np.all(rsd > 0)


def test_bootstrap_ensemble_pipeline_matches_oracle(at):
    """P:211 end to end: 5 bootstrap multisets of D, one rank-loss model per multiset, the models
    concatenated, UCB over them on new candidates -- each stage against the oracle."""
    osp, idx, X, c, key = fit_inputs(600, [synth.CFG2B], seed=71)
    Xg = osp_g = at.Space([synth.CFG2B]).features(u64(idx))
    models, oms = [], []
    for k in range(5):
        Xo, co, ko, io = at.bootstrap_resample(Xg, 600, dev(c), dev(key.view(np.int16)), k, seed=72)
        r = O.bootstrap_indices(600, k, seed=72)
        ref = O.fit_hist(X[r], c[r], key[r], n_trees=6, depth=5)
        g = at.gbt_fit_hist(Xo, 600, co, ko, n_trees=6, depth=5)
        ex = g.export()
        for f in ("feat", "thresh", "leaf"):
            assert_bits_equal(ex[f], ref[f], f"model {k} {f}")
        models.append(g)
        oms.append(O.OracleGbt(ref["feat"], ref["thresh"], ref["leaf"]))
    cat = models[0]
    for g in models[1:]:
        cat = cat.concat(g)
    cidx = synth.uniform_indices(osp.size(), 1500, seed=73)
    sc, mu, sd = cat.predict_acq(at.Space([synth.CFG2B]).features(u64(cidx)), 1500, 5, kind="ucb", kappa=1.0)
    rs, rm, rsd = O.predict_acq(oms, osp.features(cidx), kind="ucb", kappa=1.0)
    assert_bits_equal(sc.cpu().numpy(), rs, "ucb")
    assert_bits_equal(sd.cpu().numpy(), rsd, "std")


@pytest.mark.parametrize("kind,K,T,D", [("ucb", 3, 40, 6), ("ei", 5, 33, 5), ("mean", 2, 64, 8)])
def test_sa_acquisition_energy_matches_oracle(at, kind, K, T, D):
    """SA whose energy is the acquisition over K bootstrap-style models: proposals,
    energies, accept bits, final states and top-k bit for bit against the oracle."""
    ens = [synth.ensemble(T, D, seed=90 + k) for k in range(K)]
    bases = [0.1 * k for k in range(K)]
    steps, chains = 25, 70
    temps = synth.temperatures(steps, synth.energy_scale(T))
    osp = O.OracleSpace([O.workload(**synth.CFG2B)])
    om = [O.OracleGbt(e["feat"], e["thresh"], e["leaf"], base=b) for e, b in zip(ens, bases)]
    r = osp.sa_explore(om, chains, steps, 1805, 4, temps, acq=(kind, 0.7, -0.2))
    otop = osp.topk(r["visited_E"], r["visited_idx"], 64)
    gs = [at.Gbt(e["feat"], e["thresh"], e["leaf"], base=b) for e, b in zip(ens, bases)]
    cat = gs[0]
    for g in gs[1:]:
        cat = cat.concat(g)
    res = at.sa_explore(at.Space([synth.CFG2B]), cat, u64(np.zeros(chains, np.uint64)), dev(temps), seed=1805,
                        round_=4, k_out=64, init=True, accept_bits=True, visited=True,
                        acq=dict(n_models=K, kind=kind, kappa=0.7, best=-0.2, model_base=bases))
    torch.cuda.synchronize()
    compare_sa(r, otop, res)


@pytest.mark.parametrize("wls", [[synth.MATMUL_512], synth.ALL_RESNET, synth.ALL_DW,
                                 [synth.MATMUL_8, synth.CONV_TINY, synth.ALL_DW[8]]])
def test_knob_features_match_oracle(at, wls):
    """Configuration features (Q44) bit for bit, and a model over them (fitted on the
    knob representation, n_features = 32) scores identically on both sides."""
    osp = O.OracleSpace([O.workload(**w) for w in wls])
    idx = synth.uniform_indices(osp.size(), 3001, seed=17)
    sp = at.Space(wls)
    Xg = sp.knob_features(u64(idx))
    ref = osp.features_knobs(idx)
    assert_bits_equal(Xg[:, :3001].cpu().numpy().T.copy(), ref, "knob features")
    c = synth.labels(osp.features(idx), seed=5)   # costs from the loop-context view, model on the knob view
    key = np.zeros(3001, np.uint16)
    fref = O.fit_hist(ref, c, key, n_trees=4, depth=5)
    g = at.gbt_fit_hist(Xg, 3001, dev(c), dev(key.view(np.int16)), n_trees=4, depth=5)
    ex = g.export()
    for k in ("feat", "thresh", "leaf"):
        assert_bits_equal(ex[k], fref[k], f"knob-feature model {k}")
    s = g.predict(Xg, 3001).cpu().numpy()
    assert_bits_equal(s, O.OracleGbt(fref["feat"], fref["thresh"], fref["leaf"]).predict(ref), "scores")


def test_fit_errors(at):
    """S:306 / header: n = 0 -> AT_EEMPTY at once.  A non-finite cost: a single-rank fit (fused launch or
    device-laid-out subtraction path, no host sync) returns a model whose every later use reports
    AT_EINVAL; the level-by-level path (AT_FIT_SUB=0, reads its sizes back) reports AT_EINVAL itself."""
    with pytest.raises(at.ATError) as e:
        at.gbt_fit_hist(torch.zeros((468, 4), device="cuda"), 0, torch.zeros(4, device="cuda"),
                        torch.zeros(4, dtype=torch.int16, device="cuda"))
    assert e.value.code == -7
    c = torch.tensor([1.0, float("nan"), 2.0, 3.0], device="cuda")
    X = torch.zeros((468, 4), device="cuda")
    m = at.gbt_fit_hist(X, 4, c, torch.zeros(4, dtype=torch.int16, device="cuda"))
    for use in (lambda: m.export(), lambda: m.predict(X, n=4)):
        with pytest.raises(at.ATError) as e:
            use()
        assert e.value.code == -1
    n = 3000
    cb = torch.ones(n, device="cuda")
    cb[7] = float("inf")
    Xb = torch.rand((468, n), device="cuda")
    m = at.gbt_fit_hist(Xb, n, cb, torch.zeros(n, dtype=torch.int16, device="cuda"))
    for use in (lambda: m.export(), lambda: m.predict(Xb, n=n)):
        with pytest.raises(at.ATError) as e:
            use()
        assert e.value.code == -1
    os.environ["AT_FIT_SUB"] = "0"
    try:
        with pytest.raises(at.ATError) as e:
            at.gbt_fit_hist(Xb, n, cb, torch.zeros(n, dtype=torch.int16, device="cuda"))
        assert e.value.code == -1
    finally:
        del os.environ["AT_FIT_SUB"]


@pytest.mark.parametrize("n_fit", [800, 4000])
def test_fit_does_not_block_the_host(at, n_fit):
    """8(b) "every call is stream-ordered and asynchronous": a single-rank fit enqueued behind a long kernel
    returns to the host before that kernel finishes (the fused path, n = 800, and the subtraction path,
    n = 4000, size their launches on the device), and its model is the oracle's."""
    import time
    sp = at.Space(synth.ALL_RESNET)
    ens = synth.ensemble(1000, 8, seed=1805)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    n_ch = 65536
    temps = torch.from_numpy(synth.temperatures(40, synth.energy_scale(1000))).cuda()
    cw = dev((np.arange(n_ch) % 12).astype(np.int16))
    osp, idx, Xo, c, key = fit_inputs(n_fit, [synth.CFG2A], seed=21)
    Xg = at.Space([synth.CFG2A]).features(u64(idx))
    cg, kg = dev(c), dev(key.view(np.int16))
    at.gbt_fit_hist(Xg, n_fit, cg, kg, n_trees=2, depth=3)   # warm (workspace, attributes)
    torch.cuda.synchronize()
    at.sa_explore(sp, g, torch.zeros(n_ch, dtype=torch.int64, device="cuda"), temps, seed=1, round_=0, k_out=8,
                  chain_workload=cw, init=True)            # ~15 ms of device work
    t0 = time.perf_counter()
    m = at.gbt_fit_hist(Xg, n_fit, cg, kg, n_trees=5, depth=5)
    dt = time.perf_counter() - t0
    busy = not torch.cuda.current_stream().query()
    torch.cuda.synchronize()
    assert busy, f"the stream drained during the fit call ({dt * 1e3:.2f} ms)"
    ref = O.fit_hist(Xo, c, key, n_trees=5, depth=5)
    ex = m.export()
    for k in ("feat", "thresh", "leaf"):
        assert_bits_equal(ex[k], ref[k], f"model {k}")


# ------------------------------------------------------------------ full-size configurations, sampled
def test_config3_full_chain_count_sampled(at):
    """Config 3 launch shape: 65,536 chains over the 12 ResNet spaces, 1000-tree depth-8 energy
    (fewer steps to keep the test short); chains sampled and replayed one by one by the oracle."""
    ens = synth.ensemble(1000, 8, seed=1805)
    steps, n = 6, 65536
    temps = synth.temperatures(steps, synth.energy_scale(1000))
    cw = (np.arange(n) % 12).astype(np.uint16)
    sp = at.Space(synth.ALL_RESNET)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    res = at.sa_explore(sp, g, u64(np.zeros(n, np.uint64)), dev(temps), seed=1805, round_=0, k_out=128,
                        chain_workload=dev(cw.view(np.int16)), init=True, accept_bits=True, visited=True)
    torch.cuda.synchronize()
    osp = O.OracleSpace([O.workload(**w) for w in synth.ALL_RESNET])
    oe = O.OracleGbt(**ens)
    for c in (0, 11, 12345, 40000, 65535):
        r = osp.sa_explore(oe, 1, steps, 1805, 0, temps, chain_id_base=c, chain_workload=cw[c:c + 1])
        assert_bits_equal(host_u64(res["visited_idx"][c:c + 1]), r["visited_idx"], f"chain {c} idx")
        assert_bits_equal(res["visited_E"][c:c + 1].cpu().numpy(), r["visited_E"], f"chain {c} E")
        assert_bits_equal(res["accept_bits"][c:c + 1].cpu().numpy().view(np.uint32), r["accept_bits"], f"chain {c}")
    # per-workload top-k == distinct top-k of the (sample-verified) visited set
    vE = res["visited_E"].cpu().numpy()
    vI = host_u64(res["visited_idx"])
    on = res["out_n"].cpu().numpy()
    for w in (0, 5, 11):
        E, I = vE[cw == w].ravel(), vI[cw == w].ravel()
        o = np.lexsort((I, E))
        _, first = np.unique(I[o], return_index=True)
        keep = o[np.sort(first)][:128]
        assert on[w] == 128
        assert np.array_equal(host_u64(res["out_idx"][w]), I[keep])


def test_config4_refit_full_sample_count(at):
    """Config 4: 10^5 synthetic measured samples over the 9 MobileNet depthwise spaces (first trees
    only -- the oracle is O(n F) per level); trees, leaves and the root histogram bit-exact."""
    n = 100000
    osp = O.OracleSpace([O.workload(**w) for w in synth.ALL_DW])
    key = synth.group_keys(n, 9, seed=4)
    sizes = np.array([osp.size(w) for w in range(9)], dtype=np.uint64)
    loc = synth.uniform_indices(1 << 62, n, seed=5) % sizes[key]
    idx = loc + np.array([osp.offset(w) for w in range(9)], dtype=np.uint64)[key]
    Xo = osp.features(idx)
    c = synth.labels(Xo, seed=6)
    ref = O.fit_hist(Xo, c, key, n_trees=2, depth=6, want_hist0=True)
    sp = at.Space(synth.ALL_DW)
    Xg = sp.features(u64(idx))
    assert_bits_equal(Xg[:, :n].cpu().numpy().T, Xo, "features")
    h0 = torch.empty((468, 256, 2), dtype=torch.int64, device="cuda")
    pred = torch.empty(n, dtype=torch.float32, device="cuda")
    for path in ("subtraction", "level-by-level"):
        os.environ.update(FIT_PATHS[path])
        try:
            gm = at.gbt_fit_hist(Xg, n, dev(c), dev(key.view(np.int16)), n_trees=2, depth=6, hist0_out=h0,
                                 pred_out=pred)
        finally:
            for k in FIT_PATHS[path]:
                os.environ.pop(k, None)
        ex = gm.export()
        assert_bits_equal(h0.cpu().numpy(), ref["hist0"], f"{path} root histogram")
        for k in ("feat", "thresh", "leaf"):
            assert_bits_equal(ex[k], ref[k], f"{path} {k}")
        assert_bits_equal(pred.cpu().numpy(), ref["pred"], f"{path} fit predictions")


def test_config5_sweep_sampled(at):
    """Config 5: the (a n + c) mod |S| sweep over the 12 ResNet spaces with a 2000-tree depth-8
    ensemble; scores and leaf slots of sampled candidates against the oracle."""
    ens = synth.ensemble(2000, 8, seed=1805)
    sp = at.Space(synth.ALL_RESNET)
    n = 1 << 14
    idx = synth.sweep_indices(sp.size(), 10 ** 7, n)
    assert len(np.unique(idx)) == n
    X = sp.features(u64(idx))
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    s, sl = g.predict(X, n=n, slots=True)
    osp = O.OracleSpace([O.workload(**w) for w in synth.ALL_RESNET])
    pick = np.random.default_rng(0).choice(n, 48, replace=False)
    Xo = osp.features(idx[pick])
    es, esl = O.OracleGbt(**ens).predict(Xo, slots=True)
    assert_bits_equal(X[:, pick].cpu().numpy().T, Xo, "sampled features")
    assert_bits_equal(s.cpu().numpy()[pick], es, "sampled scores")
    assert_bits_equal(sl.cpu().numpy()[:, pick], esl, "sampled leaf slots")


# ------------------------------------------------------------------ exp_det, boundary errors
def test_exp_det_all_2_32_inputs_bit_identical(at):
    """Reading Q22 (Metropolis acceptance, Alg. 1; Eq. 2's sigmoid): the device
    exp_det equals the oracle's on every one of the 2^32 fp32 inputs (NaN outputs compared as NaN,
    their payload is not part of the contract)."""
    chunk = 1 << 27
    out = torch.empty(chunk, dtype=torch.float32, device="cuda")
    bad = 0
    for first in range(0, 1 << 32, chunk):
        at.exp_det_eval(first, chunk, out=out)
        g = out.cpu().numpy()
        o = O.exp_det_range(first, chunk)
        gb, ob = g.view(np.uint32), o.view(np.uint32)
        diff = gb != ob
        if diff.any():
            diff &= ~(np.isnan(g) & np.isnan(o))
            bad += int(diff.sum())
            assert bad == 0, f"exp_det differs at bits {first + int(np.flatnonzero(diff)[0]):#010x}"


def test_out_of_range_indices_report_erange(at):
    """SPEC S:138-142 ("errors: out-of-range index"), include/at_b200.h conventions: an index >= |S|
    in features_extract, a persistent chain state outside its workload or a chain workload >= n_w in
    sa_explore, a pool entry outside `workload` in select_topk -> the next call on the space (or
    space_check) returns AT_ERANGE; valid calls afterwards are unaffected."""
    sp = at.Space([synth.MATMUL_512, synth.MATMUL_8])
    n = sp.size()
    idx = u64(np.array([0, n - 1, n, 5], np.uint64))
    sp.features(idx)
    with pytest.raises(at.ATError) as e:
        sp.check()
    assert e.value.code == -2
    sp.features(idx[:2])
    sp.check()                                        # cleared, and the valid call is clean
    sp.features(idx)
    torch.cuda.synchronize()
    with pytest.raises(at.ATError) as e:              # reported by the NEXT call, which launches nothing
        sp.features(idx[:2])
    assert e.value.code == -2
    ens = synth.ensemble(8, 3, seed=1)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    temps = torch.full((4,), 0.1, dtype=torch.float32, device="cuda")
    # chain state of workload 1 claimed for workload 0
    bad_state = u64(np.array([sp.offsets[1] + 3, 7], np.uint64))
    cw = dev(np.array([0, 0], np.int16))
    at.sa_explore(sp, g, bad_state, temps, seed=1, round_=0, k_out=4, chain_workload=cw)
    with pytest.raises(at.ATError) as e:
        sp.check()
    assert e.value.code == -2
    # chain workload >= n_w
    at.sa_explore(sp, g, u64(np.array([1, 2], np.uint64)), temps, seed=1, round_=0, k_out=4,
                  chain_workload=dev(np.array([0, 5], np.int16)))
    with pytest.raises(at.ATError) as e:
        sp.check()
    assert e.value.code == -2
    # select pool entry of another workload
    pool = u64(np.array([1, 2, sp.offsets[1] + 1], np.uint64))
    at.select_topk(sp, 0, pool, dev(np.array([0.1, 0.2, 0.3], np.float32)), b=2, eps=0.0, alpha=0.1, seed=1,
                   round_=0)
    with pytest.raises(at.ATError) as e:
        sp.check()
    assert e.value.code == -2
    at.select_topk(sp, 0, pool[:2].contiguous(), dev(np.array([0.1, 0.2], np.float32)), b=2, eps=0.0, alpha=0.1,
                   seed=1, round_=0)
    sp.check()


def test_topk_drops_measured_over_several_rounds(at):
    """Alg. 1 P:152 / Q23: the distinct top-K excludes measured configurations even when the K best
    keys hold many measured ones (the tile's measured-drop loop runs several rounds)."""
    sp = at.Space([synth.MATMUL_8])
    osp = O.OracleSpace([O.workload(**synth.MATMUL_8)])
    ens = synth.ensemble(20, 5, seed=9)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    N = osp.size()
    allidx = np.arange(N, dtype=np.uint64)
    E = O.OracleGbt(**ens).predict(osp.features(allidx))
    order = allidx[np.lexsort((allidx, E))]
    for n_meas in (40, 200, 700):
        meas = np.sort(order[:n_meas])   # the whole head of the ranking is measured
        r = at.sa_explore(sp, g, u64(allidx), torch.empty(0, dtype=torch.float32, device="cuda"), seed=1,
                          round_=0, k_out=64, measured=u64(meas), init=False)
        k = int(r["out_n"][0])
        assert k == 64
        assert np.array_equal(host_u64(r["out_idx"][0][:k]), order[n_meas:n_meas + 64]), n_meas


def test_select_batch_equals_single_calls_and_oracle(at):
    """select_topk_batch (one launch, one block per workload, pools with device counts) == select_topk per
    workload == the oracle, on the 12-workload union with measured exclusions and a short pool."""
    sp = at.Space(synth.ALL_RESNET)
    osp = O.OracleSpace([O.workload(**w) for w in synth.ALL_RESNET])
    k = 40
    rng = np.random.default_rng(5)
    idx = np.zeros((12, k), np.uint64)
    sc = np.zeros((12, k), np.float32)
    for w in range(12):
        i = synth.uniform_indices(osp.size(w), k, seed=100 + w, offset=osp.offset(w))
        e = rng.random(k).astype(np.float32)
        o = np.lexsort((i, e))
        idx[w], sc[w] = i[o], e[o]
    cnt = np.full(12, k, np.int32)
    cnt[3] = 7                                              # a short pool
    meas = np.sort(np.concatenate([idx[w, :2] for w in range(0, 12, 2)]))
    out, on = at.select_topk_batch(sp, u64(idx), dev(sc), dev(cnt), b=16, eps=0.25, alpha=0.1, seed=9, round_=3,
                                   measured=u64(meas))
    for w in range(12):
        n = int(on[w])
        single, sn = at.select_topk(sp, w, u64(idx[w, :cnt[w]]), dev(sc[w, :cnt[w]]), b=16, eps=0.25, alpha=0.1,
                                    seed=9, round_=3, measured=u64(meas))
        assert n == int(sn) == 16
        assert np.array_equal(host_u64(out[w][:n]), host_u64(single[:n]))
        ref = osp.select(w, idx[w, :cnt[w]], sc[w, :cnt[w]], 16, 0.25, 0.1, 9, 3, measured=meas)
        assert np.array_equal(host_u64(out[w][:n]), ref), w


def test_topk_fast_path_and_its_fallback(at):
    """Alg. 1 P:152 / Q23 through the top-k threshold fast path: (1) a long run on the 2,000-config matmul
    space, where 4096 greedy chains pile onto a few local minima -- the candidates below the threshold
    are mostly duplicates, so the fast path must hand the workload to the exact tile reduction; (2) a
    12-workload union with measured configurations, settled by the fast path.  Both == the oracle."""
    sp = at.Space([synth.MATMUL_8])
    osp = O.OracleSpace([O.workload(**synth.MATMUL_8)])
    ens = synth.ensemble(30, 5, seed=12)
    n, steps = 4096, 40
    temps = np.zeros(steps, np.float32)
    r = at.sa_explore(sp, at.Gbt(ens["feat"], ens["thresh"], ens["leaf"]), torch.zeros(n, dtype=torch.int64, device="cuda"),
                      dev(temps), seed=4, round_=0, k_out=64, init=True, visited=True)
    (oi, oE), = osp.topk(r["visited_E"].cpu().numpy().ravel(), host_u64(r["visited_idx"]).ravel(), 64)
    k = int(r["out_n"][0])
    assert k == len(oi)
    assert np.array_equal(host_u64(r["out_idx"][0][:k]), oi)
    assert_bits_equal(r["out_score"][0][:k].cpu().numpy(), oE, "scores")
    # union with measured configurations
    ens2 = synth.ensemble(60, 6, seed=13)
    n2, st2 = 3000, 30
    cw = (np.arange(n2) % 12).astype(np.uint16)
    sp2 = at.Space(synth.ALL_RESNET)
    osp2 = O.OracleSpace([O.workload(**w) for w in synth.ALL_RESNET])
    t2 = synth.temperatures(st2, synth.energy_scale(60))
    g2 = at.Gbt(ens2["feat"], ens2["thresh"], ens2["leaf"])
    r0 = at.sa_explore(sp2, g2, torch.zeros(n2, dtype=torch.int64, device="cuda"), dev(t2), seed=6, round_=0, k_out=32,
                       chain_workload=dev(cw.view(np.int16)), init=True)
    meas = np.sort(np.concatenate([host_u64(r0["out_idx"][w][:10]) for w in range(12)]))
    r2 = at.sa_explore(sp2, g2, torch.zeros(n2, dtype=torch.int64, device="cuda"), dev(t2), seed=6, round_=0, k_out=32,
                       chain_workload=dev(cw.view(np.int16)), init=True, measured=u64(meas), visited=True)
    tops = osp2.topk(r2["visited_E"].cpu().numpy().ravel(), host_u64(r2["visited_idx"]).ravel(), 32, measured=meas)
    for w, (oi2, oE2) in enumerate(tops):
        k2 = int(r2["out_n"][w])
        assert k2 == len(oi2)
        assert np.array_equal(host_u64(r2["out_idx"][w][:k2]), oi2), w


@pytest.mark.parametrize("b,want", [(20, 1), (64, 4), (100, 5)])
def test_select_epsilon_count_matches_oracle(at, b, want):
    """Q26: ceil(eps b) with eps b formed in fp32 (eps = 0.05): GPU selection == oracle selection."""
    sp = at.Space([synth.CFG2B])
    osp = O.OracleSpace([O.workload(**synth.CFG2B)])
    idx = synth.uniform_indices(osp.size(), 2 * b, seed=b)
    E = np.random.default_rng(b).random(2 * b).astype(np.float32)
    o = np.lexsort((idx, E))
    out, n = at.select_topk(sp, 0, u64(idx[o]), dev(E[o]), b=b, eps=0.05, alpha=0.1, seed=3, round_=2)
    ref = osp.select(0, idx[o], E[o], b, 0.05, 0.1, 3, 2)
    assert int(n) == b and np.array_equal(host_u64(out[:b]), ref)


def test_rank_split_pack_gather_merge_equals_single_rank(at):
    """The bench's multi-GPU exchange without NCCL: config-3 chains split contiguously over R emulated
    ranks (each its own sa_explore with its global chain-id base), every rank's per-workload top-k packed
    into one int64 buffer (dist.pack_lists), the R buffers stacked as all_gather_into_tensor lays them out,
    unpacked and merged by topk_merge == one sa_explore over all chains; then select_topk_batch on the
    merged pools == on the single-rank pools ("a batch of parallel Markov chains")."""
    from paper_1805_08166_b200 import dist as D
    sp = at.Space(synth.ALL_RESNET)
    ens = synth.ensemble(200, 8, seed=44)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    n, steps, K = 6000, 12, 32
    temps = dev(synth.temperatures(steps, synth.energy_scale(200)))
    meas = u64(np.sort(synth.uniform_indices(sp.size(), 300, seed=5)))
    cw_all = D.chain_workloads(0, n, 12, "cuda")
    one = at.sa_explore(sp, g, torch.zeros(n, dtype=torch.int64, device="cuda"), temps, seed=3, round_=1, k_out=K,
                        chain_workload=cw_all, measured=meas, init=True)
    for R in (2, 3, 8):
        bufs = []
        for r in range(R):
            base, cnt = D.strong_slice(n, r, R)
            res = at.sa_explore(sp, g, torch.zeros(cnt, dtype=torch.int64, device="cuda"), temps, seed=3, round_=1,
                                k_out=K, chain_workload=D.chain_workloads(base, cnt, 12, "cuda"), measured=meas,
                                init=True, chain_id_base=base)
            bufs.append(D.pack_lists(res["out_idx"], res["out_score"], res["out_n"]))
        gi, gs, gn = D.unpack_lists(torch.stack(bufs), 12, K)
        mi, ms, mn = at.topk_merge(sp, gi, gs, gn, K, measured=meas)
        assert torch.equal(mn, one["out_n"]), R
        for w in range(12):
            k = int(mn[w])
            assert torch.equal(mi[w][:k], one["out_idx"][w][:k]), (R, w)
            assert torch.equal(ms[w][:k].view(torch.int32), one["out_score"][w][:k].view(torch.int32)), (R, w)
        s1, n1 = at.select_topk_batch(sp, mi, ms, mn, b=16, eps=0.05, alpha=0.1, seed=3, round_=1, measured=meas)
        s0, n0 = at.select_topk_batch(sp, one["out_idx"], one["out_score"], one["out_n"], b=16, eps=0.05, alpha=0.1,
                                      seed=3, round_=1, measured=meas)
        assert torch.equal(n1, n0) and torch.equal(s1, s0), R


# ------------------------------------------------------------------ Algorithm 1 end to end
def test_algorithm1_rounds_match_oracle(at):
    """Three rounds of Algorithm 1 (SA -> select -> measure -> refit, persistent chains) through the
    C-ABI and through the oracle: identical selections, costs and final models every round."""
    from paper_1805_08166_b200.tune import TuneConfig, Tuner
    wl = dict(kind=0, n=64, m=128, k=32)
    cfg = TuneConfig(n_chains=40, n_steps=25, b=16, lam=2, eps=0.125, alpha=0.1, n_trees=6, depth=4, seed=77)
    osp = O.OracleSpace([O.workload(**wl)])

    def measure(idx):   # stand-in for hardware run time: a fixed function of the schedule
        return synth.labels(osp.features(np.asarray(idx, dtype=np.uint64)), seed=99)

    ens0 = synth.ensemble(30, 5, seed=3)
    tuner = Tuner(wl, at.Gbt(ens0["feat"], ens0["thresh"], ens0["leaf"]), measure, cfg)
    # oracle replay of the same loop
    model = O.OracleGbt(**ens0)
    chains, measured, costs = None, [], []
    for r in range(3):
        sel_gpu = tuner.step()
        e0 = osp.sa_explore(model, cfg.n_chains, 0, cfg.seed, r, np.zeros(0, np.float32), chain_idx=chains)
        temps = synth.temperatures(cfg.n_steps, synth.energy_sigma(e0["chain_energy"]), cfg.t_ratio)   # Q21
        res = osp.sa_explore(model, cfg.n_chains, cfg.n_steps, cfg.seed, r, temps, chain_idx=chains)
        chains = res["chain_idx"]
        (pi, pe), = osp.topk(res["visited_E"], res["visited_idx"], cfg.lam * cfg.b, measured=measured)
        sel = osp.select(0, pi, pe, cfg.b, cfg.eps, cfg.alpha, cfg.seed, r, measured=measured)
        assert np.array_equal(sel_gpu, sel), f"round {r}"
        measured += sel.tolist()
        costs += measure(sel).tolist()
        X = osp.features(np.array(measured, dtype=np.uint64))
        fit = O.fit_hist(X, np.array(costs, np.float32), np.zeros(len(measured), np.uint16), n_trees=cfg.n_trees,
                         depth=cfg.depth, seed=cfg.seed + r)
        model = O.OracleGbt(fit["feat"], fit["thresh"], fit["leaf"])
        ex = tuner.model.export()
        for k in ("feat", "thresh", "leaf"):
            assert_bits_equal(ex[k], fit[k], f"round {r} model {k}")
        assert np.array_equal(host_u64(tuner.state.chain_idx), chains), f"round {r} chains"
    assert len(set(tuner.state.measured)) == len(tuner.state.measured) == 3 * cfg.b      # never re-measured
    assert tuner.state.best_cost == min(costs)


@pytest.mark.parametrize("objective,K,acq", [("reg", 3, "ei"), ("rank", 2, "ucb")])
def test_algorithm1_with_transfer_and_bootstrap_matches_oracle(at, objective, K, acq):
    """Algorithm 1 with the §8(f) options together: a global model (Eq. 4) under every local fit,
    K bootstrap models and an EI / UCB SA energy, regression or rank loss;
    two rounds replayed by the oracle: identical selections and models."""
    from paper_1805_08166_b200.tune import TuneConfig, Tuner
    wl = dict(kind=0, n=64, m=128, k=32)
    cfg = TuneConfig(n_chains=36, n_steps=20, b=12, lam=2, eps=0.125, alpha=0.1, n_trees=5, depth=4, seed=55,
                     objective=objective, n_bootstrap=K, acq=acq, kappa=0.8)
    osp = O.OracleSpace([O.workload(**wl)])

    def measure(idx):
        return synth.labels(osp.features(np.asarray(idx, dtype=np.uint64)), seed=98)

    eg = synth.ensemble(20, 5, seed=6)
    gglob = at.Gbt(eg["feat"], eg["thresh"], eg["leaf"], base=0.125)
    oglob = O.OracleGbt(eg["feat"], eg["thresh"], eg["leaf"], base=0.125)
    tuner = Tuner(wl, gglob, measure, cfg, global_model=gglob)
    model, oacq, chains, measured, costs = oglob, None, None, [], []
    for r in range(2):
        sel_gpu = tuner.step()
        e0 = osp.sa_explore(model, cfg.n_chains, 0, cfg.seed, r, np.zeros(0, np.float32), chain_idx=chains, acq=oacq)
        temps = synth.temperatures(cfg.n_steps, synth.energy_sigma(e0["chain_energy"]), cfg.t_ratio)   # Q21
        res = osp.sa_explore(model, cfg.n_chains, cfg.n_steps, cfg.seed, r, temps, chain_idx=chains, acq=oacq)
        chains = res["chain_idx"]
        (pi, pe), = osp.topk(res["visited_E"], res["visited_idx"], cfg.lam * cfg.b, measured=measured)
        sel = osp.select(0, pi, pe, cfg.b, cfg.eps, cfg.alpha, cfg.seed, r, measured=measured)
        assert np.array_equal(sel_gpu, sel), f"round {r}"
        measured += sel.tolist()
        costs += measure(sel).tolist()
        X = osp.features(np.array(measured, dtype=np.uint64))
        c = np.array(costs, np.float32)
        models = []
        for k in range(K):
            ri = O.bootstrap_indices(len(measured), k, seed=cfg.seed, round_=r)
            Xk = X[ri]
            fit = O.fit_hist(Xk, c[ri], np.zeros(len(ri), np.uint16), n_trees=cfg.n_trees, depth=cfg.depth,
                             seed=cfg.seed + r, objective=objective, base_margin=oglob.predict(Xk))
            models.append(O.gbt_concat(oglob, O.OracleGbt(fit["feat"], fit["thresh"], fit["leaf"])))
        best = 0.0
        if acq == "ei":
            best = float(O.predict_acq(models, X, kind="mean")[1].min())
        model, oacq = models, (acq, cfg.kappa, best)
        ex = tuner.model.export()
        cat = models[0]
        for m in models[1:]:
            cat = O.gbt_concat(cat, m)
        for f in ("feat", "thresh", "leaf"):
            assert_bits_equal(ex[f], getattr(cat, f), f"round {r} models {f}")
        assert np.float32(tuner.acq["best"]) == np.float32(best)
    assert tuner.state.best_cost == min(costs)


def test_fused_scoring_is_sa_with_zero_steps(at):
    """The fused scorer of config 5 (sa_explore with 0 steps: features in shared memory, never in HBM)
    gives the bit-identical scores of features_extract -> gbt_predict, and its distinct top-k is the
    top of the sorted scores (the sweep indices are distinct)."""
    ens = synth.ensemble(300, 8, seed=1805)
    sp = at.Space(synth.ALL_RESNET)
    n = 5000
    idx = synth.sweep_indices(sp.size(), 12345, n)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    s = g.predict(sp.features(u64(idx)), n=n).cpu().numpy()
    offs = np.array(sp.offsets[:12], dtype=np.uint64)
    w = (np.searchsorted(offs, idx, "right") - 1).astype(np.uint16)
    r = at.sa_explore(sp, g, u64(idx), torch.empty(0, dtype=torch.float32, device="cuda"), seed=1, round_=0,
                      k_out=16, chain_workload=dev(w.view(np.int16)), init=False)
    assert_bits_equal(r["chain_energy"].cpu().numpy(), s, "fused scores")
    for wl in range(12):
        m = w == wl
        order = np.lexsort((idx[m], s[m]))[:16]
        k = int(r["out_n"][wl])
        assert_bits_equal(host_u64(r["out_idx"][wl][:k]), idx[m][order][:k], f"workload {wl} top-k")



# ------------------------------------------------------------------ NCCL plumbing on the GPU (world size 1)
def test_nccl_world1_gather_merge_and_allreduce_fit(at):
    """The bench's NCCL code path on one B200: a world-size-1 NCCL process group, so the packed
    all_gather_into_tensor of the per-workload top-k lists, topk_merge of the gathered lists, the
    histogram all-reduce of the multi-rank subtraction refit (NCCL on the library's stream through the
    callback) and the max-over-ranks timing reduction all run through NCCL; each equals the group-free
    result bit for bit (with one rank every collective is the identity)."""
    import socket
    import torch.distributed as tdist
    from paper_1805_08166_b200 import dist as D
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sp = at.Space(synth.ALL_RESNET)
    ens = synth.ensemble(100, 8, seed=45)
    g = at.Gbt(ens["feat"], ens["thresh"], ens["leaf"])
    n, steps, K = 2400, 8, 24
    temps = dev(synth.temperatures(steps, synth.energy_scale(100)))
    one = at.sa_explore(sp, g, torch.zeros(n, dtype=torch.int64, device="cuda"), temps, seed=4, round_=0, k_out=K,
                        chain_workload=D.chain_workloads(0, n, 12, "cuda"), init=True)
    osp, idx, Xo, c, key = fit_inputs(3000, [synth.CFG2A, synth.CFG2B], seed=46)
    Xg = at.Space([synth.CFG2A, synth.CFG2B]).features(u64(idx))
    cg, kg = dev(c), dev(key.view(np.int16))
    ref = at.gbt_fit_hist(Xg, 3000, cg, kg, n_trees=4, depth=5).export()
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        gi, gs, gn = D.gather_lists(one["out_idx"], one["out_score"], one["out_n"])
        assert gi.shape == (1, 12, K)
        mi, ms, mn = at.topk_merge(sp, gi, gs, gn, K)
        assert torch.equal(mn, one["out_n"])
        for w in range(12):
            k = int(mn[w])
            assert torch.equal(mi[w][:k], one["out_idx"][w][:k])
            assert torch.equal(ms[w][:k].view(torch.int32), one["out_score"][w][:k].view(torch.int32))
        m = at.gbt_fit_hist(Xg, 3000, cg, kg, n_trees=4, depth=5, hist_range=(0, 3000), allreduce=D.make_allreduce())
        ex = m.export()
        for k in ("feat", "thresh", "leaf"):
            assert_bits_equal(ex[k], ref[k], f"NCCL-reduced fit {k}")
        assert D.max_over_ranks(1.5, torch.device("cuda", 0)) == 1.5
    finally:
        tdist.destroy_process_group()
