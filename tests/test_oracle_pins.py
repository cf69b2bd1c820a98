"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the passage (P:n = PAPER.md line) or DESIGN.md reading (Qn) it
pins, and checks the oracle against something other than itself: printed /
hand-computed worked examples (tests/golden), closed forms, brute force on tiny
inputs, library routines, invariants.
"""
import itertools
import json
import math
import os
from math import comb

import numpy as np
import pytest

import oracle as O
from paper_1805_08166_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ANN = {"serial": 0, "unroll": 1, "vectorize": 2, "parallel": 3, "blockIdx": 4, "vthread": 5, "threadIdx": 6}


def W(d):
    return O.workload(**d)


def space(*ws):
    return O.OracleSpace([W(w) for w in ws])


# ---------------------------------------------------------------- RNG / exp_det
def test_philox_known_answers():
    """Q28: Philox4x32-10 must reproduce Random123's published KAT vectors."""
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for v in kat["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        assert O.philox(ctr, key) == [int(x, 16) for x in v["out"]]


def test_mulhi64_against_bigint():
    g = np.random.default_rng(1)
    for _ in range(2000):
        a = int(g.integers(0, 2**63)) * 2 + int(g.integers(0, 2))
        b = int(g.integers(1, 2**62))
        assert O.mulhi64(a, b) == (a * b) >> 64


def test_exp_det_special_values_and_accuracy():
    """Q22: exp_det(0) = 1, clamps at -87 / 88, and is within 2 ulp of fp64 exp on [-87, 88]."""
    assert O.exp_det(0.0) == 1.0
    assert O.exp_det(-0.0) == 1.0
    assert O.exp_det(-87.5) == 0.0
    assert O.exp_det(88.5) == math.inf
    xs = np.concatenate([np.linspace(-87, 88, 20001), np.linspace(-1, 1, 5001)]).astype(np.float32)
    got = O.exp_det_array(xs).astype(np.float64)
    ref = np.exp(xs.astype(np.float64))
    ulp = np.spacing(ref.astype(np.float32)).astype(np.float64)
    assert np.max(np.abs(got - ref) / ulp) <= 2.0
    # monotone non-decreasing over the grid
    s = np.sort(xs)
    v = O.exp_det_array(s)
    assert np.all(np.diff(v.astype(np.float64)) >= 0)


# ---------------------------------------------------------------- space (a1, a2)
def _closed_form_factorizations(n, L):
    """Number of ordered L-factorizations of n = prod_p C(e_p + L - 1, L - 1)."""
    out, p, m = 1, 2, n
    while p * p <= m:
        e = 0
        while m % p == 0:
            m //= p
            e += 1
        out *= comb(e + L - 1, L - 1)
        p += 1
    if m > 1:
        out *= L
    return out


@pytest.mark.parametrize("n", [1, 2, 7, 12, 28, 56, 64, 112, 128, 224, 512, 1024])
@pytest.mark.parametrize("L", [2, 3, 4])
def test_factorization_counts_closed_form(n, L):
    assert O.count_factorizations(n, L) == _closed_form_factorizations(n, L)


def test_factor_tables_lexicographic_and_exhaustive():
    """O2: a split knob's domain is every ordered L-tuple with product = extent, lexicographic."""
    sp = space(synth.CFG2A)
    for j, (ext, L) in enumerate([(128, 4), (28, 4), (28, 4), (128, 2), (3, 2), (3, 2)]):
        tab = sp.factors(0, j)
        brute = sorted(t for t in itertools.product(range(1, ext + 1), repeat=L) if math.prod(t) == ext) \
            if ext <= 28 else None
        if brute is not None:
            assert tab == brute
        assert tab == sorted(tab)
        assert all(math.prod(t) == ext for t in tab)
        assert len(set(tab)) == len(tab) == _closed_form_factorizations(ext, L)


def test_space_cardinalities():
    """|S_e| = prod_j r_j (north_star pin); sizes quoted in DESIGN.md section 4."""
    assert space(synth.MATMUL_512).size() == 55 * 55 * 10 * 5 == 151_250
    assert space(synth.MATMUL_8).size() == 10 * 10 * 4 * 5 == 2000
    assert space(synth.CFG2A).size() == 221_184_000
    assert space(synth.CFG2B).size() == 48_660_480
    u = space(*synth.ALL_RESNET)
    assert u.size() == 1_740_983_040
    expect_dw = [158_054_400, 77_414_400, 110_592_000, 27_648_000, 38_016_000,
                 6_082_560, 8_110_080, 506_880, 658_944]
    d = space(*synth.ALL_DW)
    assert [d.size(w) for w in range(9)] == expect_dw
    for w in range(9):
        assert d.size(w) == math.prod(d.radices(w))


def test_mixed_radix_roundtrip():
    """S:138-146 mixed-radix bijection: 0 -> zeros, size-1 -> maxima, round trip."""
    for wl in (synth.MATMUL_512, synth.CFG2A, synth.ALL_DW[0]):
        sp = space(wl)
        r = sp.radices()
        assert sp.decode(0) == [0] * len(r)
        assert sp.decode(sp.size() - 1) == [x - 1 for x in r]
        for idx in synth.uniform_indices(sp.size(), 500, seed=3):
            ch = sp.decode(int(idx))
            assert all(0 <= c < x for c, x in zip(ch, r))
            assert sp.encode(ch) == int(idx)
            # knob 0 fastest
            assert int(idx) == sum(c * math.prod(r[:j]) for j, c in enumerate(ch))


# ---------------------------------------------------------------- features (a3, a4)
def _check_rows(sp, choices, gold, n_rows):
    ns, rows = sp.context(choices)
    assert ns.n == n_rows
    for k, (r, g) in enumerate(zip(rows, gold["rows"])):
        got = [r.length, r.top_down, r.bottom_up]
        for b in range(3):
            got += [r.touch[b], r.reuse[b], r.stride[b]]
        assert got == pytest.approx(g, abs=0), f"loop {gold['loops'][k]}"
        assert r.ann == ANN[gold["annotations"][k]], gold["loops"][k]


def test_appendix_c_matmul_example():
    """Fig. 1 matmul lowered with the tiled 8^3 schedule: every context column of P:630-637."""
    gold = json.load(open(os.path.join(GOLD, "appendix_c_matmul.json")))
    sp = space(gold["workload"])
    s = gold["splits"]
    ch = [sp.factors(0, 0).index(tuple(s["i"])), sp.factors(0, 1).index(tuple(s["j"])),
          sp.factors(0, 2).index(tuple(s["k"])), [1, 2, 4, 8, 16].index(gold["unroll"])]
    _check_rows(sp, ch, gold, 8)
    x = sp.features([sp.encode(ch)])[0]
    # the feature vector's row blocks (Appendix A: 19 columns per loop -- length, the
    # annotation one-hot, top-down, bottom-up, then (touch, reuse, stride) of C, A, B) hold the golden rows
    for k, g in enumerate(gold["rows"]):
        z = x[19 * k: 19 * k + 19]
        assert [z[0], z[8], z[9]] == g[:3], gold["loops"][k]
        assert list(z[10:19]) == g[3:12], gold["loops"][k]
        hot = [0.0] * 7
        hot[ANN[gold["annotations"][k]]] = 1.0
        assert list(z[1:8]) == hot, gold["loops"][k]
    rel = gold["relation_t1_6"]
    for b, name in enumerate("CAB"):
        assert list(x[342 + 40 * b: 342 + 40 * b + 6]) == rel[f"{name}_reuse"]
        assert list(x[362 + 40 * b: 362 + 40 * b + 6]) == rel[f"{name}_topdown"]
    assert list(x[462:468]) == [512, 64, 64, 64, 0, 0]
    assert np.all(x[8 * 19:342] == 0)          # absent rows are zero (Q15)


def test_appendix_c2_conv_example():
    """T_CONV worked example: thread binding, distinct-element touch (Q5), fractional reuse."""
    gold = json.load(open(os.path.join(GOLD, "appendix_c2_conv.json")))
    sp = space(gold["workload"])
    t = gold["tiles"]
    ch = [sp.factors(0, j).index(tuple(t[a])) for j, a in enumerate(["f", "y", "x", "rc", "ry", "rx"])]
    ch += [gold["reorder"], [0, 512, 1500].index(gold["unroll"]), gold["vectorize"]]
    _check_rows(sp, ch, gold, 18)
    x = sp.features([sp.encode(ch)])[0]
    assert x[462] == gold["total_iters"]


def test_naive_matmul_innermost_k():
    """SPEC S:231 example: naive 4^3, innermost k: C touch 1 reuse 4 stride 0; A touch 4 reuse 1 stride 4."""
    sp = space(dict(kind=0, n=4, m=4, k=4))
    ch = [sp.factors(0, 0).index((4, 1, 1)), sp.factors(0, 1).index((4, 1, 1)), sp.factors(0, 2).index((4, 1)), 0]
    ns, rows = sp.context(ch)
    k = 2                                       # k0 is the innermost non-unit loop of i0 j0 k0
    assert (rows[k].touch[0], rows[k].reuse[0], rows[k].stride[0]) == (1, 4.0, 0)
    assert (rows[k].touch[1], rows[k].reuse[1], rows[k].stride[1]) == (4, 1.0, 4)


def _random_choices(sp, n, seed):
    return [sp.decode(int(i)) for i in synth.uniform_indices(sp.size(), n, seed=seed)]


@pytest.mark.parametrize("wl", [synth.MATMUL_8, synth.CONV_TINY, dict(kind=1, h=6, w=6, ic=2, oc=4, ksize=3, stride=2, pad=1),
                                dict(kind=2, h=6, w=6, ic=4, oc=4, ksize=3, stride=2, pad=1),
                                dict(kind=1, h=5, w=5, ic=2, oc=2, ksize=1, stride=1, pad=0)])
def test_touch_equals_flat_bruteforce(wl):
    """P:635 literal: per-dimension enumeration == enumeration of the whole flat buffer on tiny nests."""
    sp = space(wl)
    for ch in _random_choices(sp, 30, seed=7):
        ns = sp.lower(ch)
        for k in range(ns.n):
            for b in range(3):
                assert sp.touch(ns, b, k) == sp.touch(ns, b, k, brute=True)


def _closed_touch(sp, ns, b, k):
    """Independent closed form: per-dim product of active extents, min(YR,(Y-1)S+R) for y*S+ry."""
    w = sp.workloads[0]
    act = {}
    for l in range(k, ns.n):
        act[ns.axis[l]] = act.get(ns.axis[l], 1) * ns.ext[l]
    A = lambda a: act.get(a, 1)
    S = w.stride
    comp = lambda Y, R: min(Y * R, (Y - 1) * S + R)
    if sp.s.sp[0].tmpl == 1:
        dims = {0: [A(0), A(1), A(2)], 1: [A(3), comp(A(1), A(4)), comp(A(2), A(5))], 2: [A(0), A(3), A(4), A(5)]}
    elif sp.s.sp[0].tmpl == 2:
        dims = {0: [A(0), A(1), A(2)], 1: [A(0), comp(A(1), A(3)), comp(A(2), A(4))], 2: [A(0), A(3), A(4)]}
    else:
        dims = {0: [A(0), A(1)], 1: [A(2), A(0)], 2: [A(2), A(1)]}
    return math.prod(dims[b])


@pytest.mark.parametrize("wl", [synth.CFG2A, synth.CFG2B, synth.resnet("C1"), synth.ALL_DW[1], synth.MATMUL_512])
def test_touch_closed_form_agrees(wl):
    sp = space(wl)
    for ch in _random_choices(sp, 25, seed=11):
        ns = sp.lower(ch)
        for k in range(ns.n):
            for b in range(3):
                assert sp.touch(ns, b, k) == _closed_touch(sp, ns, b, k)


@pytest.mark.parametrize("wl", [synth.MATMUL_512, synth.CFG2A, synth.ALL_DW[3], synth.resnet("C11")])
def test_feature_invariants(wl):
    """top_down * bottom_up = total; top_down(0) = 1; bottom_up(last) = extent;
    touch(b, 0) = full output / kernel buffer; R_t non-decreasing in t; exactly one annotation."""
    sp = space(wl)
    ss = sp.s.sp[0]
    full = [math.prod(ss.shape[b][d] for d in range(ss.n_dims[b])) for b in range(3)]
    idx = synth.uniform_indices(sp.size(), 40, seed=5)
    X = sp.features(idx)
    for i, x in zip(idx, X):
        ns, rows = sp.context(sp.decode(int(i)))
        total = math.prod(ns.ext[k] for k in range(ns.n))
        assert rows[0].top_down == 1 and rows[-1].bottom_up == rows[-1].length
        for k, r in enumerate(rows):
            assert r.top_down * r.bottom_up == total
            assert sum(x[19 * k + 1: 19 * k + 8]) == 1
        assert rows[0].touch[0] == full[0]
        if ss.tmpl == 0:
            assert rows[0].touch[1] == full[1] and rows[0].touch[2] == full[2]
        else:
            assert rows[0].touch[2] == full[2]
        for b in range(3):
            for p in range(2):
                R = x[342 + 40 * b + 20 * p: 342 + 40 * b + 20 * p + 20]
                assert np.all(np.diff(R) >= 0)
        assert x[462] == np.float32(total)
        assert x[466] == 0 and x[467] == 0


def test_relation_feature_spec_example():
    """touch column [100, 10] with reuse [4, 8] and beta = 32 -> 8 (only the inner loop qualifies).
    Realised as a 2-loop matmul-like nest: the relation value at t = 5 is the inner loop's reuse."""
    sp = space(dict(kind=0, n=100, m=1, k=1))
    # i = (1, 10, 10) -> loops i0(1) j0 k0 i1(10) j1 k1 i2(10) j2; pick the row values directly
    ch = [sp.factors(0, 0).index((1, 10, 10)), 0, 0, 0]
    x = sp.features([sp.encode(ch)])[0]
    ns, rows = sp.context(ch)
    t = 5
    qual = [r for r in rows if r.touch[0] < 2 ** t]
    assert x[342 + t - 1] == max(r.reuse[0] for r in qual)
    assert all(r.touch[0] >= 2 ** t for r in rows if r not in qual)


# ---------------------------------------------------------------- GBT (a5)
def test_hand_ensemble_predictions():
    """north_star pin: a tiny hand-built ensemble yields known predictions and leaf slots (Q18)."""
    e = O.OracleGbt(**synth.hand_ensemble())
    X = np.array([[1, 0], [2.5, 1.5], [3, 0.7]], np.float32)
    s, sl = e.predict(X, slots=True)
    assert list(s) == [1.25, 3.5, 3.25]
    assert sl.T.tolist() == [[0, 0], [3, 2], [2, 0]]


def test_gbt_canonical_sum_close_to_fp64_and_batch_equals_single():
    ens = synth.ensemble(333, 6, seed=9)
    e = O.OracleGbt(**ens)
    sp = space(synth.CFG2A)
    X = sp.features(synth.uniform_indices(sp.size(), 64, seed=2))
    s, sl = e.predict(X, slots=True)
    ni = 63
    ref = np.zeros(len(X))
    for i in range(len(X)):   # independent pointer-walk in fp64
        tot = 0.0
        for t in range(333):
            node = 0
            for _ in range(6):
                node = 2 * node + (1 if X[i, ens["feat"][t, node]] < ens["thresh"][t, node] else 2)
            assert sl[t, i] == node - ni
            tot += float(ens["leaf"][t, node - ni])
        ref[i] = tot
    assert np.allclose(s, ref, rtol=1e-6, atol=1e-6)
    for i in range(0, 64, 9):
        assert e.predict(X[i:i + 1])[0] == s[i]


# ---------------------------------------------------------------- SA + top-k (a6, a7)
def _tiny():
    sp = space(synth.MATMUL_8)
    ens = synth.ensemble(40, 6, seed=4)
    return sp, O.OracleGbt(**ens), ens


def test_sa_infinite_temperature_accepts_everything():
    sp, e, _ = _tiny()
    r = sp.sa_explore(e, 16, 40, seed=1805, round_=0, temps=np.full(40, np.inf, np.float32))
    assert np.all(r["accept_bits"][:, 0] == 0xFFFFFFFF)
    assert np.all(r["accept_bits"][:, 1] == (1 << 8) - 1)
    assert np.all(r["chain_idx"] == r["visited_idx"][:, -1])


def test_sa_zero_temperature_is_greedy_and_proposals_are_single_knob():
    sp, e, _ = _tiny()
    steps = 64
    r = sp.sa_explore(e, 24, steps, seed=7, round_=2, temps=np.zeros(steps, np.float32))
    X = sp.features(r["visited_idx"].ravel())
    E = e.predict(X).reshape(24, steps + 1)
    assert np.array_equal(E, r["visited_E"])
    for c in range(24):
        cur_i, cur_E = r["visited_idx"][c, 0], E[c, 0]
        for s in range(steps):
            prop = r["visited_idx"][c, s + 1]
            a, b = sp.decode(int(cur_i)), sp.decode(int(prop))
            assert sum(x != y for x, y in zip(a, b)) == 1        # S:151 single-knob move
            acc = (r["accept_bits"][c, s // 32] >> (s % 32)) & 1
            assert acc == (1 if E[c, s + 1] <= cur_E else 0)     # T = 0: accept iff E' <= E
            if acc:
                cur_i, cur_E = prop, E[c, s + 1]
        assert r["chain_idx"][c] == cur_i and r["chain_energy"][c] == cur_E


def test_sa_topk_equals_exhaustive_ranking_on_tiny_space():
    """north_star pin: SA top-k on a tiny space == brute-force exhaustive ranking."""
    sp, e, _ = _tiny()
    N = sp.size()
    allidx = np.arange(N, dtype=np.uint64)
    E_all = e.predict(sp.features(allidx))
    order = np.lexsort((allidx, E_all))
    r = sp.sa_explore(e, N, 3, seed=5, round_=0, temps=np.full(3, 0.05, np.float32), chain_idx=allidx)
    (ti, tE), = sp.topk(r["visited_E"], r["visited_idx"], 64)
    assert np.array_equal(ti, allidx[order[:64]])
    assert np.array_equal(tE, E_all[order[:64]])
    # measured configs are excluded
    meas = allidx[order[:10]]
    (ti2, _), = sp.topk(r["visited_E"], r["visited_idx"], 64, measured=meas)
    assert np.array_equal(ti2, allidx[order[10:74]])


def test_sa_deterministic_and_persistent():
    sp, e, _ = _tiny()
    T = synth.temperatures(30, 0.3)
    r1 = sp.sa_explore(e, 8, 30, seed=11, round_=0, temps=T)
    r2 = sp.sa_explore(e, 8, 30, seed=11, round_=0, temps=T)
    assert np.array_equal(r1["accept_bits"], r2["accept_bits"])
    r3 = sp.sa_explore(e, 8, 30, seed=11, round_=1, temps=T, chain_idx=r1["chain_idx"])
    assert np.array_equal(r3["visited_idx"][:, 0], r1["chain_idx"])          # P:187 persistence
    # chain ids are global: chains 4..7 alone reproduce the same trajectories (rank invariance)
    r4 = sp.sa_explore(e, 4, 30, seed=11, round_=0, temps=T, chain_id_base=4)
    assert np.array_equal(r4["visited_idx"], r1["visited_idx"][4:])


def test_sa_knob_frequencies_uniform():
    """each non-singleton knob is mutated with frequency 1/#non-singleton (+-5%)."""
    sp, e, _ = _tiny()
    r = sp.sa_explore(e, 64, 200, seed=3, round_=0, temps=np.full(200, np.inf, np.float32))
    cnt = np.zeros(4)
    for c in range(64):
        for s in range(200):
            a, b = sp.decode(int(r["visited_idx"][c, s])), sp.decode(int(r["visited_idx"][c, s + 1]))
            cnt[[i for i in range(4) if a[i] != b[i]][0]] += 1
    assert np.all(np.abs(cnt / cnt.sum() - 0.25) < 0.05 * 0.25 * 4)


def _philox_words(seed, g, step, round_, tag):
    """Philox4x32-10 words of counter (g, step, round, tag), key = seed (Q28; KAT-pinned above)."""
    return O.philox([g, step, round_, tag], [seed & 0xFFFFFFFF, seed >> 32])


def test_sa_metropolis_finite_temperature_decisions():
    """Alg. 1 P:152-153 / P:187 at 0 < T < inf: every decision of every chain-step equals the
    Metropolis rule written out independently here -- accept iff d = E' - E <= 0 or
    u < exp(-d / T), with u = (word 2 >> 8) 2^-24 of Philox(g, s, round, SA_STEP) and exp from the
    C library in fp64 (not exp_det).  Decisions within 1e-5 of the threshold are skipped (fp32 vs
    fp64 rounding of exp); a sign error in -d/T, a wrong Philox word for u, or a strict/non-strict
    mix-up of the d <= 0 branch fails here."""
    sp, e, _ = _tiny()
    seed, rnd, C, S = 0x1234_5678_9ABC, 3, 64, 60
    temps = synth.temperatures(S, 0.08, 0.1)          # 0.08 -> 0.008, spans many acceptance rates
    r = sp.sa_explore(e, C, S, seed=seed, round_=rnd, temps=temps, chain_id_base=1000)
    n_up_acc = n_up_rej = n_skip = 0
    for c in range(C):
        E = np.float32(r["visited_E"][c, 0])
        for st in range(S):
            E2 = np.float32(r["visited_E"][c, st + 1])
            d = np.float32(E2 - E)                     # fp32 RN difference, as the paper's energies are fp32
            acc = (int(r["accept_bits"][c, st // 32]) >> (st % 32)) & 1
            if d <= 0:
                assert acc == 1, (c, st)
            else:
                u = (_philox_words(seed, 1000 + c, st, rnd, 1)[2] >> 8) * 2.0 ** -24
                p = math.exp(-float(d) / float(temps[st]))
                if abs(u - p) < 1e-5:
                    n_skip += 1
                else:
                    assert acc == (1 if u < p else 0), (c, st, u, p)
                    n_up_acc += acc
                    n_up_rej += 1 - acc
            if acc:
                E = E2
        assert r["chain_energy"][c] == E
    assert n_up_acc > 100 and n_up_rej > 100 and n_skip < 10


def test_sa_uphill_acceptance_frequency_is_boltzmann_factor():
    """over many uphill proposals the number accepted equals sum exp(-d/T) within a
    binomial 5-sigma band (the statistical form of the Metropolis rule)."""
    sp, e, _ = _tiny()
    T = 0.03
    r = sp.sa_explore(e, 256, 80, seed=99, round_=0, temps=np.full(80, T, np.float32))
    acc_n, p_sum, var = 0, 0.0, 0.0
    for c in range(256):
        E = r["visited_E"][c, 0]
        for st in range(80):
            E2 = r["visited_E"][c, st + 1]
            a = (int(r["accept_bits"][c, st // 32]) >> (st % 32)) & 1
            if E2 > E:
                p = math.exp(-(float(E2) - float(E)) / T)
                acc_n += a
                p_sum += p
                var += p * (1 - p)
            if a:
                E = E2
    assert var > 100
    assert abs(acc_n - p_sum) <= 5 * math.sqrt(var), (acc_n, p_sum, var)


def test_sa_samples_the_boltzmann_distribution():
    """Metropolis with a symmetric proposal (single-knob move uniform over the non-singleton knobs,
    new value uniform among the others: S:151, Q20) has the stationary law pi(s) ~ exp(-f(s) / T)
    (P:152-153).  On the 2,000-configuration matmul 8^3 space at fixed T, the final states of
    3,000 independent chains match pi computed by exhaustive enumeration: chi-square over 10 energy
    bins of equal pi mass (p > 1e-4) and the mean energy within 5 standard errors.  A sign error in
    the acceptance exponent concentrates the chains on the worst configurations instead."""
    from scipy.stats import chi2
    sp, e, _ = _tiny()
    N = sp.size()
    allidx = np.arange(N, dtype=np.uint64)
    E = e.predict(sp.features(allidx)).astype(np.float64)
    T, C, S = 0.05, 3000, 150
    r = sp.sa_explore(e, C, S, seed=11, round_=0, temps=np.full(S, T, np.float32))
    fin = r["chain_idx"].astype(np.int64)
    w = np.exp(-(E - E.min()) / T)
    pi = w / w.sum()
    order = np.argsort(E, kind="stable")
    cum = np.cumsum(pi[order])
    nb = 10
    b_of = np.empty(N, np.int64)
    b_of[order] = np.searchsorted(np.linspace(0, 1, nb + 1)[1:-1], cum - pi[order] / 2)
    expect = np.array([pi[b_of == b].sum() for b in range(nb)]) * C
    obs = np.bincount(b_of[fin], minlength=nb)
    x2 = float(((obs - expect) ** 2 / expect).sum())
    assert chi2.sf(x2, nb - 1) > 1e-4, (obs, expect.round(1), x2)
    mean_pi = float((pi * E).sum())
    sd_pi = math.sqrt(float((pi * (E - mean_pi) ** 2).sum()))
    assert abs(E[fin].mean() - mean_pi) <= 5 * sd_pi / math.sqrt(C)


def test_sa_annealing_concentrates_on_the_optimum_of_a_unimodal_energy():
    """S:384 (the hill-climbing limit of SA, Alg. 1): on a unimodal energy, annealed chains
    end at the optimum.  The energy is a hand-built depth-2 ensemble on the matmul 8^3 space: one
    tree per loop i0, j0, k0, i1, j1 (rows 0-4 of the T_MM nest, length column 19 r) with penalty 1
    for an extent < 2, 0 for extent 2, 1 for extent > 2 -- unimodal in every knob, minimum 0 exactly
    at split_i = split_j = (2, 2, 2), split_k = (2, 4) (any unroll: 5 optimal configurations,
    0.25 % of the space).  Annealed from T = 1 to 0.01 over 400 steps, >= 90 % of 512 chains end at
    energy 0 (>= 90 % within the top 1 %); with the exponent's sign flipped they would climb."""
    sp = space(synth.MATMUL_8)
    rows = [0, 1, 2, 3, 4]
    inf = np.float32(np.inf)
    feat = np.array([[19 * r, 0, 19 * r] for r in rows], np.uint16)
    thr = np.array([[1.5, inf, 2.5] for _ in rows], np.float32)
    leaf = np.array([[1.0, 1.0, 0.0, 1.0] for _ in rows], np.float32)
    e = O.OracleGbt(feat, thr, leaf)
    N = sp.size()
    E = e.predict(sp.features(np.arange(N, dtype=np.uint64)))
    opt = np.flatnonzero(E == 0.0)
    assert len(opt) == 5 and all(sp.decode(int(i))[:3] == sp.decode(int(opt[0]))[:3] for i in opt)
    S = 400
    r = sp.sa_explore(e, 512, S, seed=5, round_=1, temps=synth.temperatures(S, 1.0, 0.01))
    assert np.mean(r["chain_energy"] == 0.0) >= 0.9
    assert set(r["chain_idx"][r["chain_energy"] == 0.0].tolist()) <= set(opt.tolist())


# ---------------------------------------------------------------- select (a8)
def test_select_alpha0_eps0_is_plain_topb():
    sp = space(synth.CFG2A)
    idx = synth.uniform_indices(sp.size(), 128, seed=8)
    E = np.random.default_rng(0).random(128).astype(np.float32)
    E[5] = E[6]                                  # a tie, broken by idx
    order = np.lexsort((idx, E))
    got = sp.select(0, idx[order], E[order], b=64, eps=0.0, alpha=0.0, seed=1, round_=0)
    assert np.array_equal(got, idx[order[:64]])


def test_select_epsilon_picks():
    """exactly ceil(eps b) random picks, never measured, never duplicated; greedy first."""
    sp = space(synth.CFG2B)
    idx = synth.uniform_indices(sp.size(), 128, seed=9)
    E = np.random.default_rng(1).random(128).astype(np.float32)
    order = np.lexsort((idx, E))
    meas = synth.uniform_indices(sp.size(), 50, seed=10)
    got = sp.select(0, idx[order], E[order], b=64, eps=0.05, alpha=0.1, seed=3, round_=4, measured=meas)
    assert len(got) == 64 and len(set(got.tolist())) == 64
    assert set(got[:60].tolist()) <= set(idx.tolist())
    assert not set(got.tolist()) & set(meas.tolist())


def test_select_exhausted_space_stops():
    sp = space(dict(kind=0, n=1, m=1, k=2))     # |S| = 1*1*2*5 = 10
    assert sp.size() == 10
    meas = np.array([0, 1, 2, 3], np.uint64)
    got = sp.select(0, np.array([4, 5], np.uint64), np.array([0.1, 0.2], np.float32), b=20, eps=0.5,
                    alpha=0.0, seed=1, round_=0, measured=meas)
    assert sorted(got.tolist()) == [4, 5, 6, 7, 8, 9]


def test_select_greedy_vs_bruteforce_subsets():
    """greedy L(S) >= (1 - 1/e) max_S L(S) (L shifted non-negative on singletons), pools of 8, b = 4."""
    sp = space(synth.CFG2A)
    g = np.random.default_rng(2)
    for trial in range(20):
        idx = synth.uniform_indices(sp.size(), 8, seed=100 + trial)
        E = g.random(8).astype(np.float32)
        alpha = 1.0
        got = sp.select(0, idx, E, b=4, eps=0.0, alpha=alpha, seed=1, round_=0)
        mu, sd = E.astype(np.float64).mean(), E.astype(np.float64).std()
        z = (E - mu) / sd
        ch = [sp.decode(int(i)) for i in idx]
        shift = max(0.0, max(z))                 # makes -z + shift >= 0 per element

        def L(S):
            cov = sum(len({ch[i][j] for i in S}) for j in range(9))
            return sum(-z[i] + shift for i in S) + alpha * cov

        best = max(L(S) for S in itertools.combinations(range(8), 4))
        mine = L([list(idx).index(i) for i in got])
        assert mine >= (1 - 1 / math.e) * best - 1e-12


def test_select_coverage_term_decides_at_the_hand_computed_threshold():
    """Eq. 3: the coverage term counts distinct values per knob over the selected
    set.  Pool of 3 on T_MM (4 knobs): A = (0,0,0,0) best, B = (0,1,0,0) (one knob differs from A),
    C = (1,1,1,1) (all four differ).  After A is picked, B adds coverage 1 and C adds 4 (S:393's
    example: {[1,2],[1,3]} covers |{1}| + |{2,3}| = 3 values -- A and B cover 4 + 1 = 5 here), so the
    second greedy pick switches from B to C exactly when alpha (4 - 1) > z_C - z_B."""
    sp = space(dict(kind=0, n=4, m=4, k=4))
    A, B, Cc = (sp.encode(v) for v in ([0, 0, 0, 0], [0, 1, 0, 0], [1, 1, 1, 1]))
    pool = np.array([A, B, Cc], np.uint64)
    E = np.array([-1.0, 0.25, 0.5], np.float32)
    Ed = E.astype(np.float64)
    mu = (Ed[0] + Ed[1] + Ed[2]) / 3
    sd = math.sqrt(((Ed[0] - mu) ** 2 + (Ed[1] - mu) ** 2 + (Ed[2] - mu) ** 2) / 3)
    a_star = ((Ed[2] - mu) / sd - (Ed[1] - mu) / sd) / (4 - 1)
    lo = sp.select(0, pool, E, b=2, eps=0.0, alpha=float(np.float32(a_star * 0.95)), seed=1, round_=0)
    hi = sp.select(0, pool, E, b=2, eps=0.0, alpha=float(np.float32(a_star * 1.05)), seed=1, round_=0)
    assert lo.tolist() == [A, B] and hi.tolist() == [A, Cc]
    # first pick: every knob value is new for every candidate (coverage 4 each) -> lowest z wins
    # even for a huge alpha
    big = sp.select(0, pool, E, b=1, eps=0.0, alpha=1e6, seed=1, round_=0)
    assert big.tolist() == [A]


def test_select_epsilon_count_is_ceil_of_the_fp32_product():
    """P:156, Q26: ceil(eps b) random picks with eps b formed in fp32 -- eps = 0.05 gives 1 of 20,
    4 of 64 and 5 of 100 (not 2 / 6 from ceil of the widened 0.0500000007 b)."""
    sp = space(synth.CFG2B)
    for b, want in ((20, 1), (64, 4), (100, 5)):
        n_pool = 2 * b
        idx = synth.uniform_indices(sp.size(), n_pool, seed=b)
        E = np.random.default_rng(b).random(n_pool).astype(np.float32)
        order = np.lexsort((idx, E))
        got = sp.select(0, idx[order], E[order], b=b, eps=0.05, alpha=0.0, seed=3, round_=0)
        # alpha = 0: the greedy part is the plain top (b - n_rand) of the pool
        n_g = b - want
        assert got[:n_g].tolist() == idx[order[:n_g]].tolist()
        assert got[n_g] != idx[order[n_g]]          # the next one is a random pick, not the pool's next
        assert len(got) == b


# ---------------------------------------------------------------- refit (a9)
def test_rank_loss_closed_forms():
    """Eq. 2: each ordered pair contributes log(1 + e^{-sign (f_i - f_j)})."""
    c = np.array([1, 2], np.float32)
    assert O.rank_loss(c, np.array([0, 0], np.float32)) == pytest.approx(2 * math.log(2), rel=1e-12)
    assert O.rank_loss(c, np.array([3, 1], np.float32)) == pytest.approx(2 * math.log(1 + math.e ** 2), rel=1e-12)


def test_pair_gradients_match_finite_difference():
    """g_i, h_i are the first/second derivatives of Eq. 2 summed over ordered pairs inside a group."""
    g = np.random.default_rng(5)
    n = 40                                       # one group (group_size 64)
    cost = g.random(n).astype(np.float32)
    pred = (g.random(n) - 0.5).astype(np.float32)
    key = np.zeros(n, np.uint16)
    G, H = O.pair_gradients(cost, pred, key, seed=1, tree=0, group_size=64)
    for i in range(0, n, 7):
        eps = 1e-3
        p1, p2 = pred.astype(np.float64).copy(), pred.astype(np.float64).copy()
        p1[i] += eps
        p2[i] -= eps
        # finite difference of Eq. 2 (libm exp, fp64) -- independent of exp_det
        def L(p):
            s = 0.0
            for a in range(n):
                for b in range(n):
                    if a != b:
                        sg = np.sign(cost[a] - cost[b])
                        s += math.log1p(math.exp(-sg * (p[a] - p[b])))
            return s
        fd = (L(p1) - L(p2)) / (2 * eps)
        fd2 = (L(p1) - 2 * L(pred.astype(np.float64)) + L(p2)) / eps ** 2
        assert G[i] / 2 ** 32 == pytest.approx(fd, rel=1e-4, abs=1e-6)
        assert H[i] / 2 ** 32 == pytest.approx(fd2, rel=2e-3, abs=1e-4)


def test_group_positions_are_permutations_within_workloads():
    key = synth.group_keys(3001, 5, seed=2)
    for tree in (0, 1, 7):
        pos = O.group_positions(key, seed=1805, tree=tree)
        for w in range(5):
            p = pos[key == w]
            assert sorted(p.tolist()) == list(range(len(p)))
    assert not np.array_equal(O.group_positions(key, 1805, 0), O.group_positions(key, 1805, 1))


def _fit_data(n=600, seed=3, nw=2):
    sp = space(synth.MATMUL_512, synth.CFG2B)
    key = synth.group_keys(n, nw, seed=seed)
    idx = np.array([sp.offset(int(w)) + int(synth.uniform_indices(sp.size(int(w)), 1, seed=seed * 1000 + i)[0])
                    for i, w in enumerate(key)], np.uint64)
    X = sp.features(idx)
    return X, synth.labels(X, seed=seed), key


def test_fit_label_affine_invariance():
    """only sign(c_i - c_j) enters Eq. 2, so labels c and 2c + 5 give a bit-identical ensemble."""
    X, c, key = _fit_data(300)
    a = O.fit_hist(X, c, key, n_trees=4, depth=4)
    b = O.fit_hist(X, (2 * c.astype(np.float64) + 5).astype(np.float32), key, n_trees=4, depth=4)
    for k in ("feat", "thresh", "leaf"):
        assert np.array_equal(a[k], b[k])


def test_fit_root_split_equals_exact_greedy():
    """Every feature here has <= 256 unique values, so histogram splits == exact greedy over all thresholds."""
    X, c, key = _fit_data(400)
    Xs = X[:, :120]                               # rows 0..5 of the context block
    out = O.fit_hist(Xs, c, key, n_trees=1, depth=1)
    G, H = O.pair_gradients(c, np.zeros(len(c), np.float32), key, seed=1805, tree=0)
    G, H = G.astype(np.float64) / 2 ** 32, H.astype(np.float64) / 2 ** 32
    lam = 1.0
    best = (-1, None, 0.0)
    for f in range(Xs.shape[1]):
        vals = np.unique(Xs[:, f])
        if len(vals) > 256:
            pytest.skip("feature with > 256 unique values")
        for th in vals[1:]:
            left = Xs[:, f] < th
            gl, hl, gr, hr = G[left].sum(), H[left].sum(), G[~left].sum(), H[~left].sum()
            if hl < 1 or hr < 1:
                continue
            gain = gl * gl / (hl + lam) + gr * gr / (hr + lam) - G.sum() ** 2 / (H.sum() + lam)
            if gain > best[2] * (1 + 1e-12) + 1e-300:
                best = (f, th, gain)
    assert out["feat"][0, 0] == best[0]
    assert out["thresh"][0, 0] == best[1]
    # leaves are -eta G / (H + lambda) of the two children
    left = Xs[:, best[0]] < best[1]
    for slot, m in ((0, left), (1, ~left)):
        w = -0.1 * (G[m].sum() / (H[m].sum() + lam))
        assert out["leaf"][0, slot] == pytest.approx(w, rel=1e-6)


def test_fit_min_gain_is_lambda_regularised():
    """Q37's gain G_L^2/(H_L+lam) + G_R^2/(H_R+lam) - G^2/(H+lam) decides whether the root splits at all.
    Regression loss (g = 2 (f - c), h = 2), one feature x = (0, 0, 1, 1), lam = 1: for costs
    (1, 1, 1 + d, 1 + d) the gain is positive iff (1 + (1+d)^2)/5 > (2+d)^2/9, i.e. d > 1 (by hand);
    d = 1.5 splits (leaves -G_L/(H_L+lam) = 0.8 and 10/5 = 2.0 at eta = 1), d = 0.5 does not (a
    pass-through root, threshold +inf, left leaf -G/(H+lam) = 10/9)."""
    X = np.array([[0.0], [0.0], [1.0], [1.0]], np.float32)
    key = np.zeros(4, np.uint16)
    out = O.fit_hist(X, np.array([1, 1, 2.5, 2.5], np.float32), key, n_trees=1, depth=1, eta=1.0, lam=1.0,
                     min_child_weight=1.0, objective="reg")
    assert out["feat"][0, 0] == 0 and out["thresh"][0, 0] == 1.0
    assert out["leaf"][0].tolist() == pytest.approx([0.8, 2.0], rel=1e-6)
    out = O.fit_hist(X, np.array([1, 1, 1.5, 1.5], np.float32), key, n_trees=1, depth=1, eta=1.0, lam=1.0,
                     min_child_weight=1.0, objective="reg")
    assert np.isinf(out["thresh"][0, 0])
    assert out["leaf"][0, 0] == pytest.approx(10.0 / 9.0, rel=1e-6)


def test_fit_min_child_weight_and_tie_rule():
    """Q37: a split needs H_L, H_R >= min_child_weight; equal gains go to the lower feature (then the lower
    split).  Regression loss (h = 2 per sample), x = (0, 0, 0, 1), costs (0, 0, 0, 10): the only split
    leaves H_R = 2, so min_child_weight 3 forbids it and 1 allows it (its gain 400/3 - 400/9 > 0 by hand).
    Two identical columns give two equal gains: feature 0 wins."""
    key = np.zeros(4, np.uint16)
    X = np.array([[0.0], [0.0], [0.0], [1.0]], np.float32)
    c = np.array([0, 0, 0, 10], np.float32)
    kw = dict(n_trees=1, depth=1, eta=1.0, lam=1.0, objective="reg")
    assert np.isinf(O.fit_hist(X, c, key, min_child_weight=3.0, **kw)["thresh"][0, 0])
    out = O.fit_hist(X, c, key, min_child_weight=1.0, **kw)
    assert out["feat"][0, 0] == 0 and out["thresh"][0, 0] == 1.0
    X2 = np.array([[0.0, 0.0], [0.0, 0.0], [1.0, 1.0], [1.0, 1.0]], np.float32)
    out = O.fit_hist(X2, np.array([1, 1, 2.5, 2.5], np.float32), key, min_child_weight=1.0, **kw)
    assert out["feat"][0, 0] == 0 and out["thresh"][0, 0] == 1.0


def test_fit_reduces_rank_loss():
    X, c, key = _fit_data(400, seed=4, nw=1)
    key = np.zeros_like(key)
    out = O.fit_hist(X, c, key, n_trees=15, depth=4)
    assert O.rank_loss(c, out["pred"]) < 0.9 * O.rank_loss(c, np.zeros(len(c), np.float32))
    # the fit's own predictions equal re-scoring the training set with the ensemble (up to order)
    e = O.OracleGbt(out["feat"], out["thresh"], out["leaf"])
    assert np.allclose(e.predict(X), out["pred"], rtol=1e-5, atol=1e-6)


def test_fit_cuts_rule():
    """Q36: <= max_bins unique values -> cuts are the unique values but the minimum; else quantiles."""
    g = np.random.default_rng(0)
    X = np.stack([g.integers(0, 10, 1000), g.random(1000) * 100], axis=1).astype(np.float32)
    cuts, nc = O.fit_cuts(X, 256)
    assert nc[0] == 9 and list(cuts[0, :9]) == list(range(1, 10))
    s = np.sort(X[:, 1])
    q = [s[((b + 1) * 1000) // 256] for b in range(255)]
    uq = [v for i, v in enumerate(q) if v != s[0] and (i == 0 or v != q[i - 1])]
    assert list(cuts[1, :nc[1]]) == uq


# ---------------------------------------------------------------- §8(f): regression objective
def test_reg_gradients_closed_form():
    """P:175 loss sum_i (f_i - c_i)^2: dl/df_i = 2 (f_i - c_i), d2l/df_i^2 = 2, in 2^-32 units;
    the gradient is checked against a central finite difference of the loss itself."""
    c = np.array([1.0, 2.5, -3.0, 7.25], np.float32)
    f = np.array([0.0, 3.0, -3.0, 1.0], np.float32)
    g, h = O.reg_gradients(c, f)
    assert g.tolist() == [-2 * 2**32, 2**32, 0, -int(12.5 * 2**32)]
    assert h.tolist() == [2**33] * 4
    loss = lambda ff: float(np.sum((ff.astype(np.float64) - c.astype(np.float64)) ** 2))
    for i in range(4):
        e = np.zeros(4)
        e[i] = 1e-3
        fd = (loss(f + e) - loss(f - e)) / 2e-3
        assert abs(fd - g[i] / 2**32) < 1e-6


def test_fit_regression_newton_step_is_the_group_mean():
    """With eta = 1, lambda = 0 a squared-loss leaf is -G/H = the mean residual of its samples, so
    one depth-1 tree on a single 2-valued feature predicts each value's mean cost exactly; the next
    tree sees zero gradients, finds no split (gain 0 is not > 0) and changes nothing."""
    X = np.array([[0.0], [0.0], [1.0], [1.0], [1.0]], np.float32)
    c = np.array([1.0, 3.0, 2.0, 4.0, 6.0], np.float32)
    key = np.zeros(5, np.uint16)
    r = O.fit_hist(X, c, key, n_trees=2, depth=1, eta=1.0, lam=0.0, min_child_weight=0.0, objective="reg")
    assert r["feat"][0, 0] == 0 and r["thresh"][0, 0] == 1.0
    assert r["leaf"][0].tolist() == [2.0, 4.0]
    assert r["pred"].tolist() == [2.0, 2.0, 4.0, 4.0, 4.0]
    assert r["thresh"][1, 0] == np.inf and r["leaf"][1, 0] == 0.0   # slot 1 is unreachable (0/0 at lambda 0)


def test_fit_regression_margin_equals_shifted_labels():
    """Transfer margin (Eq. 4): fitting c on top of margin m is fitting c - m from zero (exact here:
    small integers); the trees are identical and the predictions differ by exactly m."""
    rng = np.random.default_rng(5)
    n = 300
    X = rng.integers(0, 6, (n, 8)).astype(np.float32)
    m = rng.integers(-4, 5, n).astype(np.float32)
    c = (X[:, 0] * 2 + X[:, 3] + rng.integers(0, 3, n)).astype(np.float32)
    key = np.zeros(n, np.uint16)
    a = O.fit_hist(X, c, key, n_trees=1, depth=3, objective="reg", base_margin=m)
    b = O.fit_hist(X, (c - m).astype(np.float32), key, n_trees=1, depth=3, objective="reg")
    for k in ("feat", "thresh", "leaf"):
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(a["pred"], (b["pred"] + m).astype(np.float32))


def test_fit_rank_margin_constant_shift_invariance():
    """Eq. 2 sees only differences f_j - f_i: a constant margin leaves the first tree unchanged, and
    the training predictions are shifted by the margin."""
    osp = space(synth.CFG2B)
    n = 400
    idx = synth.uniform_indices(osp.size(), n, seed=2)
    X = osp.features(idx)
    c = synth.labels(X, seed=2)
    key = np.zeros(n, np.uint16)
    a = O.fit_hist(X, c, key, n_trees=1, depth=4)
    b = O.fit_hist(X, c, key, n_trees=1, depth=4, base_margin=np.full(n, 0.5, np.float32))
    for k in ("feat", "thresh", "leaf"):
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(b["pred"], (a["pred"] + np.float32(0.5)).astype(np.float32))


# ---------------------------------------------------------------- §8(f): transfer learning, Eq. 4
def _rand_ens(T, D, F, seed):
    rng = np.random.default_rng(seed)
    ni, nl = (1 << D) - 1, 1 << D
    return O.OracleGbt(rng.integers(0, F, (T, ni)).astype(np.uint16),
                       rng.integers(0, 8, (T, ni)).astype(np.float32) + 0.5,
                       rng.uniform(-1, 1, (T, nl)).astype(np.float32), base=float(rng.uniform(-1, 1)))


def test_padded_tree_keeps_every_value():
    """A depth-2 tree inside a depth-5 ensemble (pass-through nodes below, leaves at the leftmost
    descendants) returns the same leaf for every input: brute force over all 8^3 feature vectors."""
    small = O.OracleGbt(np.array([[0, 1, 2]], np.uint16), np.array([[3.5, 2.5, 5.5]], np.float32),
                        np.array([[1.0, 2.0, 3.0, 4.0]], np.float32), base=0.75)
    zero = O.OracleGbt(np.zeros((1, 31), np.uint16), np.full((1, 31), np.inf, np.float32),
                       np.zeros((1, 32), np.float32))
    cat = O.gbt_concat(small, zero)
    assert cat.depth == 5 and cat.n_trees == 2
    X = np.array(list(itertools.product(range(8), repeat=3)), np.float32)
    ref = O.OracleGbt(small.feat, small.thresh, small.leaf).predict(X)   # base 0: the leaf itself
    got = O.OracleGbt(cat.feat[:1], cat.thresh[:1], cat.leaf[:1]).predict(X)
    assert len(np.unique(ref)) == 4   # every leaf is reached
    assert np.array_equal(got, ref)


def test_concat_is_sum_of_models_within_fp32_rounding():
    """Eq. 4: f(x) = f_global(x) + f_local(x); the concatenated ensemble's canonical fp32 sum agrees
    with the fp64 sum of the two models' exact tree sums within (T + 2) ulp-scaled error."""
    a, b = _rand_ens(37, 6, 20, seed=3), _rand_ens(21, 4, 20, seed=4)
    cat = O.gbt_concat(a, b)
    assert cat.n_trees == 58 and cat.depth == 6
    assert cat.base == np.float32(np.float32(a.base) + np.float32(b.base))
    X = np.random.default_rng(6).integers(0, 8, (500, 20)).astype(np.float32)
    got = cat.predict(X).astype(np.float64)
    _, sa = a.predict(X, slots=True)
    _, sb = b.predict(X, slots=True)
    exact = (a.leaf.astype(np.float64)[np.arange(37)[:, None], sa].sum(0)
             + b.leaf.astype(np.float64)[np.arange(21)[:, None], sb].sum(0) + np.float64(cat.base))
    bound = (58 + 2) * 2.0 ** -24 * (np.abs(a.leaf).max() * 37 + np.abs(b.leaf).max() * 21 + 2)
    assert np.max(np.abs(got - exact)) <= bound


# ---------------------------------------------------------------- §8(f): bootstrap uncertainty, EI / UCB
def test_bootstrap_indices_are_uniform_with_replacement():
    """Q40: n draws with replacement: every index in range, the unique fraction of a bootstrap
    sample tends to 1 - 1/e, and over many models every sample is drawn ~uniformly (chi-square)."""
    n, K = 2000, 40
    cnt = np.zeros(n)
    fr = []
    for k in range(K):
        idx = O.bootstrap_indices(n, k, seed=9)
        assert idx.min() >= 0 and idx.max() < n
        assert np.array_equal(idx, O.bootstrap_indices(n, k, seed=9))
        fr.append(len(np.unique(idx)) / n)
        np.add.at(cnt, idx, 1)
    assert abs(np.mean(fr) - (1 - math.exp(-1))) < 0.01
    chi2 = np.sum((cnt - K) ** 2 / K)
    assert chi2 < n + 6 * math.sqrt(2 * n)          # n - 1 dof: mean n - 1, sd sqrt(2 (n - 1))
    assert not np.array_equal(O.bootstrap_indices(n, 0, seed=9), O.bootstrap_indices(n, 1, seed=9))


def test_acquisition_mean_std_ucb_against_numpy():
    """Q41/Q42: mean and population std of the K scores (numpy fp64 as the reference routine);
    UCB = mu - kappa sigma; kappa = 0 or K = 1 reduce to the mean."""
    rng = np.random.default_rng(4)
    for K in (1, 2, 5, 8):
        for _ in range(200):
            f = rng.normal(0, 2, K).astype(np.float32)
            v, m, s = O.acquisition("ucb", f, kappa=1.5)
            f64 = f.astype(np.float64)
            assert abs(m - np.mean(f64)) <= 1e-6 * max(1.0, abs(np.mean(f64)))
            assert abs(s - np.std(f64)) <= 1e-6 * max(1.0, np.std(f64))
            assert abs(v - (np.mean(f64) - 1.5 * np.std(f64))) <= 2e-6 * max(1.0, abs(v))
            assert O.acquisition("ucb", f, kappa=0.0)[0] == O.acquisition("mean", f)[0] == np.float32(m)
            if K == 1:
                assert s == 0.0 and v == f[0]


def test_expected_improvement_closed_forms_and_bound():
    """Q43: EI(mu = best) = sigma phi(0) = sigma / sqrt(2 pi); sigma = 0 gives max(best - mu, 0);
    on a grid EI matches the exact fp64 formula (math.erfc, math.exp) within the A&S 7.1.26 error
    bound plus fp32 rounding, is >= max(best - mu, 0) and decreases as mu grows."""
    for sd in (0.1, 1.0, 7.5):
        assert abs(O.expected_improvement(2.0, sd, 2.0) - sd / math.sqrt(2 * math.pi)) <= 3e-7 * sd
    assert O.expected_improvement(1.0, 0.0, 3.0) == 2.0 and O.expected_improvement(4.0, 0.0, 3.0) == 0.0
    prev = None
    for mu in np.linspace(-6, 6, 241):
        sd, best = 1.3, 0.4
        got = O.expected_improvement(float(mu), sd, best)
        d = best - float(np.float32(mu))
        z = d / sd
        Phi = 0.5 * math.erfc(-z / math.sqrt(2))
        ref = d * Phi + sd * math.exp(-z * z / 2) / math.sqrt(2 * math.pi)
        assert abs(got - ref) <= 2e-7 * (abs(d) + sd) + 1e-6 * abs(ref)
        assert got >= max(d, 0.0) - 1e-6
        if prev is not None:
            assert got <= prev + 1e-7
        prev = got
    assert O.acquisition("ei", np.array([1.0, 3.0], np.float32), best=2.5)[0] == -O.expected_improvement(2.0, 1.0, 2.5)


def test_sa_acquisition_over_identical_models_is_plain_sa():
    """K copies of one model have sigma = 0 and an fp64 mean equal to the model's fp32 score, so SA
    with the UCB energy over them replays plain SA exactly (P:208-215 reduces to f-hat)."""
    osp = space(synth.CFG2B)
    e = synth.ensemble(30, 5, seed=8)
    m = O.OracleGbt(e["feat"], e["thresh"], e["leaf"], base=0.3)
    temps = synth.temperatures(15, 0.2)
    a = osp.sa_explore(m, 20, 15, 1805, 1, temps)
    b = osp.sa_explore([m, m, m], 20, 15, 1805, 1, temps, acq=("ucb", 2.0, 0.0))
    for k in ("visited_idx", "visited_E", "accept_bits", "chain_idx"):
        assert np.array_equal(a[k], b[k]), k


# ---------------------------------------------------------------- §8(f): configuration features (Q44)
def test_knob_features_factor_products_and_ends():
    """Q44: each split knob's columns are an ordered factorization of its axis extent (product =
    extent); index 0 is the first lexicographic tuple (1, ..., 1, extent) with the other knobs at
    their first value; index |S| - 1 is (extent, 1, ..., 1) with every other knob at its last."""
    cases = [(synth.MATMUL_512, [3, 3, 2], [512, 512, 512], [("u", [1, 2, 4, 8, 16])]),
             (synth.CFG2A, [4, 4, 4, 2, 2, 2], [128, 28, 28, 128, 3, 3], [("p", 5), ("u", [0, 512, 1500]), ("v", 1)]),
             (synth.ALL_DW[3], [4, 4, 4, 2, 2], [128, 28, 28, 3, 3], [("p", 5), ("u", [0, 512, 1500]), ("v", 1)])]
    for wl, levels, ext, rest in cases:
        osp = space(wl)
        n_split = sum(levels)
        X = osp.features_knobs(synth.uniform_indices(osp.size(), 500, seed=3))
        c = 0
        for L, e in zip(levels, ext):
            assert np.all(np.prod(X[:, c:c + L].astype(np.int64), axis=1) == e)
            c += L
        assert np.all(X[:, n_split + len(rest):] == 0)
        first, last = osp.features_knobs([0, osp.size() - 1])
        c = 0
        for L, e in zip(levels, ext):
            assert first[c:c + L].tolist() == [1] * (L - 1) + [e]
            assert last[c:c + L].tolist() == [e] + [1] * (L - 1)
            c += L
        for k, (kind, v) in enumerate(rest):
            assert first[c + k] == (v[0] if kind == "u" else 0)
            assert last[c + k] == (v[-1] if kind == "u" else v)


def test_knob_features_identify_the_configuration():
    """The configuration representation is one-to-one: all 151,250 configurations of the config-1
    space have distinct knob-feature rows (brute force)."""
    osp = space(synth.MATMUL_512)
    X = osp.features_knobs(np.arange(osp.size(), dtype=np.uint64))
    assert len(np.unique(X, axis=0)) == osp.size() == 151250
