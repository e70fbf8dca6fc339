"""Batch-sharded multi-GPU driver.

Sequences are independent, so the batch is split into contiguous shards, one
per rank (one process per GPU, ``torch.distributed`` over NCCL / NVLink).
Everything a sequence owns -- x, y, zi, zf, per-sequence or per-sample
coefficients and their gradients -- stays on its rank.  The only exchange of
the whole path is the sum of the SHARED-coefficient gradients (2 (M+1)
values, i.e. 72 B at M = 8): ``iir_backward`` returns local-batch sums and the
driver all-reduces them.

``sharded_step`` takes the per-shard compute as a callable so that the host
logic (sharding, the reduction, result assembly) can be tested on CPU with
the gloo backend; the product passes :func:`cuda_shard_compute`, which runs
the CUDA kernels through the C ABI.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_range(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous near-equal split of `batch` sequences: [start, stop) of `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world size")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


@dataclass
class ShardResult:
    y: torch.Tensor
    zf: torch.Tensor
    gx: torch.Tensor
    gzi: torch.Tensor
    gb: Optional[torch.Tensor]      # SHARED: summed over ALL ranks after the reduction
    ga: Optional[torch.Tensor]


def reduce_shared_grads(gb: torch.Tensor, ga: torch.Tensor, group=None, deterministic: bool = False):
    """Sum the shared-coefficient gradients over the ranks of `group`.

    deterministic=False: one all_reduce(SUM) of cat(gb, ga).
    deterministic=True : all_gather of the per-rank vectors and a sum in rank
    order (bitwise reproducible regardless of the collective's internal order;
    same latency class for a 2(M+1)-element message)."""
    n = gb.numel()
    buf = torch.cat([gb.reshape(-1), ga.reshape(-1)])
    world = dist.get_world_size(group)
    if world == 1:
        return gb, ga
    if deterministic:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        buf = parts[0].clone()
        for p in parts[1:]:
            buf += p
    else:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf[:n].view_as(gb), buf[n:].view_as(ga)


def sharded_step(compute: Callable, x: torch.Tensor, gy: torch.Tensor, b: torch.Tensor, a: torch.Tensor,
                 zi: Optional[torch.Tensor], gzf: Optional[torch.Tensor], form: str = "tdf", group=None,
                 deterministic: bool = False) -> ShardResult:
    """Forward + backward of this rank's shard, then the shared-gradient reduction.

    x, gy (B_local, T), zi, gzf (B_local, M) are this rank's shard; b, a are
    (M+1,) SHARED or (B_local, M+1) PER_SEQ.  `compute(x, gy, b, a, zi, gzf, form)`
    returns (y, zf, gx, gb, ga, gzi) for the shard (gb, ga local sums)."""
    y, zf, gx, gb, ga, gzi = compute(x, gy, b, a, zi, gzf, form)
    if b.dim() == 1 and dist.is_initialized():
        gb, ga = reduce_shared_grads(gb, ga, group, deterministic)
    return ShardResult(y=y, zf=zf, gx=gx, gzi=gzi, gb=gb, ga=ga)


def cuda_shard_compute(x, gy, b, a, zi, gzf, form):
    """Per-shard compute on the local GPU through the C ABI (no fallback)."""
    from . import _binding as B
    if not x.is_cuda:
        raise ValueError("cuda_shard_compute needs CUDA tensors")
    Bsz, T = x.shape
    M = b.shape[-1] - 1
    mode = B.IIR_COEF_SHARED if b.dim() == 1 else B.IIR_COEF_PER_SEQ
    desc = B.make_desc(Bsz, T, M, form, x.dtype, mode)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    tape = torch.empty(tb, dtype=torch.uint8, device=x.device)
    ws = torch.empty(wb, dtype=torch.uint8, device=x.device)
    y = torch.empty_like(x)
    gx = torch.empty_like(x)
    zf = torch.empty((Bsz, M), dtype=x.dtype, device=x.device)
    gzi = torch.empty_like(zf)
    gb = torch.empty_like(b)
    ga = torch.empty_like(a)
    B.iir_forward(desc, b, a, x, zi, y, zf, tape, tb, ws, wb)
    B.iir_backward(desc, gy, gzf, b, a, x, y, zi, tape, tb, gx, gb, ga, gzi, ws, wb)
    return y, zf, gx, gb, ga, gzi
