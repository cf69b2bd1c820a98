"""Multi-rank host logic on CPU: world_size-2 gloo process groups (no GPU).

The rank partition, the all-gather of per-rank top-k lists, the merge and the histogram
all-reduce wrapper of paper_1805_08166_b200.dist are exercised with the CPU oracle
standing in for the per-rank kernels (test-only injection): a 2-rank run must give
exactly the single-rank result (rank-count invariance).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1805_08166_b200 import dist as D
from paper_1805_08166_b200 import synth

WLS = [synth.CFG2B, synth.MATMUL_512]
N_PER_RANK, STEPS, K = 12, 15, 20


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_lists(rank, n_per_rank):
    osp = O.OracleSpace([O.workload(**w) for w in WLS])
    ens = O.OracleGbt(**synth.ensemble(30, 5, seed=2))
    base, cnt = D.chain_slice(n_per_rank, rank)
    cw = D.chain_workloads(base, cnt, len(WLS), "cpu").numpy().astype(np.uint16)
    temps = synth.temperatures(STEPS, 0.2)
    r = osp.sa_explore(ens, cnt, STEPS, 1805, 0, temps, chain_id_base=base, chain_workload=cw)
    top = osp.topk(r["visited_E"], r["visited_idx"], K)
    idx = np.zeros((len(WLS), K), np.uint64)
    sc = np.zeros((len(WLS), K), np.float32)
    n = np.zeros(len(WLS), np.int32)
    for w, (i, e) in enumerate(top):
        idx[w, :len(i)], sc[w, :len(i)], n[w] = i, e, len(i)
    return osp, r, idx, sc, n


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        osp, r, idx, sc, n = _rank_lists(rank, N_PER_RANK)
        gi, gs, gn = D.gather_lists(torch.from_numpy(idx.view(np.int64)), torch.from_numpy(sc), torch.from_numpy(n))
        # merge of the gathered lists (oracle top-k over their union)
        merged = []
        for w in range(len(WLS)):
            E = np.concatenate([gs[l, w, :gn[l, w]].numpy() for l in range(world)])
            I = np.concatenate([gi[l, w, :gn[l, w]].numpy().view(np.uint64) for l in range(world)])
            merged.append(osp.topk(E, I, K)[w])
        # histogram all-reduce wrapper: int64 sums are exact
        h = torch.arange(1000, dtype=torch.int64) * (rank + 1) + (1 << 40)
        D.make_allreduce()(h)
        b, e = D.sample_slice(1001, rank, world)
        rk, ws = D.world()
        q.put((rank, [(m[0].tolist(), m[1].tolist()) for m in merged], h.tolist(), (b, e), (rk, ws),
               D.max_over_ranks(float(rank)), D.sum_over_ranks(1.0)))
    finally:
        dist.destroy_process_group()


def test_two_rank_topk_and_allreduce_equal_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in ps]
    out = sorted([q.get(timeout=300) for _ in range(2)])
    [p.join(timeout=60) for p in ps]
    assert all(p.exitcode == 0 for p in ps)
    # single rank owning all 2 * N_PER_RANK chains
    osp, r, idx, sc, n = _rank_lists(0, 2 * N_PER_RANK)
    for rank, merged, h, sl, rw, mx, sm in out:
        assert rw == (rank, 2)
        for w in range(len(WLS)):
            assert merged[w][0] == idx[w, :n[w]].tolist()
            assert np.array_equal(np.array(merged[w][1], np.float32), sc[w, :n[w]])
        assert h == [int(i) * 3 + (1 << 41) for i in range(1000)]
        assert mx == 1.0 and sm == 2.0
    assert [o[3] for o in out] == [(0, 501), (501, 1001)]


def test_pack_unpack_roundtrip():
    """The packed exchange buffer (one collective per round) carries indices, score bits (incl. -0.0,
    inf) and counts unchanged, for even and odd n_w k."""
    for nw, k in ((12, 128), (1, 3), (3, 5)):
        g = np.random.default_rng(nw * k)
        idx = torch.from_numpy(g.integers(0, 2 ** 62, size=(nw, k)).astype(np.int64))
        sc = torch.from_numpy(g.standard_normal((nw, k)).astype(np.float32))
        sc[0, 0] = -0.0
        sc[-1, -1] = float("inf")
        n = torch.from_numpy(g.integers(0, k + 1, size=nw).astype(np.int32))
        buf = D.pack_lists(idx, sc, n)
        i2, s2, n2 = D.unpack_lists(torch.stack([buf, buf]), nw, k)
        assert torch.equal(i2[1], idx) and torch.equal(s2[0].view(torch.int32), sc.view(torch.int32))
        assert torch.equal(n2[1], n)


def test_partitions_cover_exactly():
    for n in (0, 1, 7, 1000, 100001):
        for ws in (1, 2, 3, 8):
            sl = [D.sample_slice(n, r, ws) for r in range(ws)]
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(sl[i][1] == sl[i + 1][0] for i in range(ws - 1))
    assert D.chain_slice(4096, 3) == (12288, 4096)
    assert [D.strong_slice(65536, r, 8) for r in (0, 7)] == [(0, 8192), (57344, 8192)]
    assert sum(D.strong_slice(65537, r, 3)[1] for r in range(3)) == 65537
    cw = D.chain_workloads(12, 13, 12, "cpu")
    assert cw.tolist() == [c % 12 for c in range(12, 25)]
