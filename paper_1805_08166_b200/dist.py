"""Multi-GPU plumbing for the hot path (one process per GPU, torch.distributed).

The path shards three ways:
  * SA chains: rank r owns global chain ids [r * n_per_rank, (r + 1) * n_per_rank); chain
    randomness is keyed by the global id, so trajectories do not depend on the rank count;
  * per-rank distinct top-k lists are all-gathered once (the exchange step of Alg. 1
    P:152 "collect candidates") and merged by topk_merge;
  * refit samples: every rank holds all samples, builds histograms over its contiguous
    slice, and the per-level int64 histograms are summed with one all-reduce.
Integer histograms and global-id RNG make every output bit-identical at any rank count.
Only host logic lives here; all arithmetic runs in the library kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def _grouped() -> bool:
    """A process group exists (of any size, 1 included): the collectives below then always run, so the
    NCCL path is exercised even on one GPU."""
    return dist.is_available() and dist.is_initialized()


def chain_slice(n_per_rank: int, rank: int):
    """Global chain-id base and count of this rank (weak scaling: n_per_rank chains per GPU)."""
    return rank * n_per_rank, n_per_rank


def sample_slice(n: int, rank: int, world_size: int):
    """Contiguous histogram slice [begin, end) of n samples for this rank."""
    q, r = divmod(n, world_size)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def chain_workloads(base: int, count: int, n_workloads: int, device) -> torch.Tensor:
    """Workload of each local chain: global chain c belongs to workload c mod n_workloads (config 3)."""
    c = torch.arange(base, base + count, device=device, dtype=torch.int64)
    return (c % n_workloads).to(torch.int16)


def pack_lists(out_idx: torch.Tensor, out_score: torch.Tensor, out_n: torch.Tensor) -> torch.Tensor:
    """One rank's [n_w][k] top-k lists as ONE int64 buffer (so the exchange is a single collective):
    [n_w k global indices | n_w k score bits + n_w counts as int32 pairs]."""
    nw, k = out_idx.shape
    tail = torch.cat([out_score.reshape(-1).view(torch.int32), out_n.reshape(-1).to(torch.int32)])
    if tail.numel() % 2:
        tail = torch.cat([tail, tail.new_zeros(1)])
    return torch.cat([out_idx.reshape(-1), tail.view(torch.int64)])


def unpack_lists(buf: torch.Tensor, nw: int, k: int):
    """[world][L] gathered buffers -> idx [world][nw][k] int64, score float32, n [world][nw] int32."""
    world = buf.shape[0]
    idx = buf[:, :nw * k].contiguous().view(world, nw, k)
    tail = buf[:, nw * k:].contiguous().view(torch.int32)
    score = tail[:, :nw * k].contiguous().view(torch.float32).view(world, nw, k)
    n = tail[:, nw * k:nw * k + nw].contiguous()
    return idx, score, n


def gather_lists(out_idx: torch.Tensor, out_score: torch.Tensor, out_n: torch.Tensor, group=None):
    """All-gather every rank's [n_w][k] top-k lists -> [world][n_w][k]: the lists are packed into one
    int64 buffer and exchanged by ONE all_gather_into_tensor (NCCL over NVLink on the GPU box)."""
    rank, ws = world()
    if not _grouped():
        return out_idx[None], out_score[None], out_n[None]
    nw, k = out_idx.shape
    mine = pack_lists(out_idx, out_score, out_n)
    allb = torch.empty(ws * mine.numel(), dtype=torch.int64, device=mine.device)
    dist.all_gather_into_tensor(allb, mine, group=group)
    return unpack_lists(allb.view(ws, -1), nw, k)


def strong_slice(n_total: int, rank: int, world_size: int):
    """Strong scaling: global chain ids [base, base + count) of this rank, contiguous."""
    b, e = sample_slice(n_total, rank, world_size)
    return b, e - b


def make_allreduce(group=None):
    """Sum an int64 tensor in place across ranks (the refit's histogram exchange)."""
    def _ar(t: torch.Tensor):
        assert t.dtype == torch.int64
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return _ar


def max_over_ranks(x: float, device=None) -> float:
    if not _grouped():
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    if not _grouped():
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
