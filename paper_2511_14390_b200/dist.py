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


_SHARD_BUFFERS = {}


def _shard_buffers(Bsz, T, M, form, dtype, mode, device):
    """Tape and workspace of one shard shape, allocated and cleared (iir_workspace_init) once
    per (shape, device, stream); later calls pass IIR_FLAG_WS_READY (every completed call
    leaves the workspace cleared), so a training loop allocates and memsets nothing per step."""
    from . import _binding as B
    stream = torch.cuda.current_stream(device)
    key = (Bsz, T, M, form, dtype, mode, str(device), stream.cuda_stream)
    hit = _SHARD_BUFFERS.get(key)
    if hit is None:
        desc0 = B.make_desc(Bsz, T, M, form, dtype, mode)
        tb, wb = B.iir_tape_bytes(desc0), B.iir_workspace_bytes(desc0)
        tape = torch.empty(tb, dtype=torch.uint8, device=device)
        ws = torch.empty(wb, dtype=torch.uint8, device=device)
        B.iir_workspace_init(desc0, ws, wb, stream)
        desc = B.make_desc(Bsz, T, M, form, dtype, mode, flags=B.IIR_FLAG_WS_READY)
        hit = _SHARD_BUFFERS[key] = (desc, tape, tb, ws, wb)
    return hit


def cuda_shard_compute(x, gy, b, a, zi, gzf, form):
    """Per-shard compute on the local GPU through the C ABI (no fallback)."""
    from . import _binding as B
    from .autograd import _check
    if not x.is_cuda:
        raise ValueError("cuda_shard_compute needs CUDA tensors")
    Bsz, T = x.shape
    M = b.shape[-1] - 1
    coef = [(M + 1,)] if b.dim() == 1 else [(Bsz, M + 1)]
    _check(x, [("gy", gy, [(Bsz, T)]), ("b", b, coef), ("a", a, coef), ("zi", zi, [(Bsz, M)]),
               ("gzf", gzf, [(Bsz, M)])])
    mode = B.IIR_COEF_SHARED if b.dim() == 1 else B.IIR_COEF_PER_SEQ
    desc, tape, tb, ws, wb = _shard_buffers(Bsz, T, M, form, x.dtype, mode, x.device)
    y = torch.empty_like(x)
    gx = torch.empty_like(x)
    zf = torch.empty((Bsz, M), dtype=x.dtype, device=x.device)
    gzi = torch.empty_like(zf)
    gb = torch.empty_like(b)
    ga = torch.empty_like(a)
    B.iir_forward(desc, b, a, x, zi, y, zf, tape, tb, ws, wb)
    B.iir_backward(desc, gy, gzf, b, a, x, y, zi, tape, tb, gx, gb, ga, gzi, ws, wb)
    return y, zf, gx, gb, ga, gzi


# ---------------------------------------------------------------------------
# Time-sharded sequences: ONE long sequence (or a batch of
# them) split along time into consecutive segments, one per rank -- the way
# past one GPU's bandwidth for config 4's single 2^24-sample sequence.  The
# exchange is Eq.10 with the whole segment as the chunk:
#   forward : every rank filters its segment with a zero carry (rank 0 with the
#             true zi) -> final state w_r; all_gather(w); rank r's exact zi is
#             sum_{j<r} P^(r-1-j) w_j, P = A_f^seg_len (iir_state_carry); the
#             segment is filtered again from it (ranks > 0);
#   backward: the same in reverse time on the adjoint: a
#             zero-carry backward (the last rank with the true grad_zf) gives
#             the adjoint at the segment start g_r; all_gather(g); rank r's
#             exact grad_zf is sum_{j>r} (P^T)^(j-r-1) g_j; backward again
#             (ranks < G-1); the coefficient gradients are summed over ranks
#             (every rank holds a piece of the same sequences).
# Messages: B x M values per direction (32 B per sequence at M = 4, fp64
# gather not needed: the carry kernel accumulates in fp64).  zf is valid on the
# last rank, grad_zi on rank 0.

class TorchComm:
    """torch.distributed collectives of the time-sharded driver (NCCL on GPUs)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return t.unsqueeze(0)
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.stack(parts)

    def sum_grads(self, gb, ga, deterministic=False):
        if self.world == 1:
            return gb, ga
        return reduce_shared_grads(gb, ga, self.group, deterministic)


@dataclass
class TimeShardOps:
    """Per-segment compute of the time-sharded driver.
    forward(x, b, a, zi) -> (y, zf, ctx);  backward(gy, gzf, b, a, x, y, zi, ctx) -> (gx, gb, ga, gzi);
    carry(a, W, rank, seg_len, reverse, form) -> (B, M) exact carry into the segment."""
    forward: Callable
    backward: Callable
    carry: Callable


def time_sharded_step(ops: TimeShardOps, x, gy, b, a, zi, gzf, form: str, seg_len: int, comm=None,
                      deterministic: bool = False) -> ShardResult:
    """Forward + backward of this rank's time segment.  x, gy: (B, T_r) -- the
    rank-th of consecutive segments, all `seg_len` long except possibly the
    last; zi is read on rank 0 only, gzf on the last rank only.  Returns y, gx of
    the segment; zf (valid on the last rank), grad_zi (valid on rank 0) and the
    coefficient gradients summed over all ranks."""
    comm = comm or TorchComm()
    rank, world = comm.rank, comm.world
    if world > 1 and rank < world - 1 and x.shape[-1] != seg_len:
        raise ValueError("every segment but the last must hold seg_len samples")
    y, zf, ctx = ops.forward(x, b, a, zi if rank == 0 else None)
    zi_r = zi if rank == 0 else None
    if world > 1:
        W = comm.all_gather(zf)
        if rank > 0:
            zi_r = ops.carry(a, W, rank, seg_len, False, form)
            y, zf, ctx = ops.forward(x, b, a, zi_r)
    last = rank == world - 1
    gx, gb, ga, gzi = ops.backward(gy, gzf if last else None, b, a, x, y, zi_r, ctx)
    if world > 1:
        Gz = comm.all_gather(gzi)
        if not last:
            gzf_r = ops.carry(a, Gz, rank, seg_len, True, form)
            gx, gb, ga, gzi = ops.backward(gy, gzf_r, b, a, x, y, zi_r, ctx)
        gb, ga = comm.sum_grads(gb, ga, deterministic)
    return ShardResult(y=y, zf=zf, gx=gx, gzi=gzi, gb=gb, ga=ga)


def cuda_time_ops(form: str) -> TimeShardOps:
    """The product's per-segment compute for filter form `form`: iir_forward /
    iir_backward / iir_state_carry on the local GPU through the C ABI (no fallback)."""
    from . import _binding as B
    from .autograd import _check

    def fwd(x, b, a, zi):
        if not x.is_cuda:
            raise ValueError("cuda_time_ops needs CUDA tensors")
        Bsz, T = x.shape
        M = b.shape[-1] - 1
        coef = [(M + 1,)] if b.dim() == 1 else [(Bsz, M + 1)]
        _check(x, [("b", b, coef), ("a", a, coef), ("zi", zi, [(Bsz, M)])])
        d = B.make_desc(Bsz, T, M, form, x.dtype, B.IIR_COEF_SHARED if b.dim() == 1 else B.IIR_COEF_PER_SEQ)
        tb, wb = B.iir_tape_bytes(d), B.iir_workspace_bytes(d)
        tape = torch.empty(tb, dtype=torch.uint8, device=x.device)
        ws = torch.empty(wb, dtype=torch.uint8, device=x.device)
        y = torch.empty_like(x)
        zf = torch.empty((Bsz, M), dtype=x.dtype, device=x.device)
        B.iir_forward(d, b, a, x, zi, y, zf, tape, tb, ws, wb)
        return y, zf, (d, tape, tb, ws, wb)

    def bwd(gy, gzf, b, a, x, y, zi, ctx):
        d, tape, tb, ws, wb = ctx
        gx = torch.empty_like(x)
        gzi = torch.empty((x.shape[0], b.shape[-1] - 1), dtype=x.dtype, device=x.device)
        gb, ga = torch.empty_like(b), torch.empty_like(a)
        B.iir_backward(d, gy, gzf, b, a, x, y, zi, tape, tb, gx, gb, ga, gzi, ws, wb)
        return gx, gb, ga, gzi

    def carry(a, W, rank, seg_len, reverse, form_):
        G, Bsz, M = W.shape
        d = B.make_desc(Bsz, max(1, seg_len), M, form_, W.dtype,
                        B.IIR_COEF_SHARED if a.dim() == 1 else B.IIR_COEF_PER_SEQ)
        out = torch.empty((Bsz, M), dtype=W.dtype, device=W.device)
        B.iir_state_carry(d, a, W.contiguous(), G, rank, seg_len, reverse, out)
        return out

    return TimeShardOps(fwd, bwd, carry)
