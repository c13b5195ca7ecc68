"""Data parallelism host logic: one process per GPU, batch
sharded weakly, NCCL gradient all-reduce inside the runtime.

torch.distributed is plumbing only: it carries the NCCL unique id from rank 0
to the other ranks and provides barriers / max-over-ranks timing (bench.py).
The gradient all-reduce per bucket, the loss all-reduce and the momentum update
are the runtime's (runtime.cu flush_bucket / allreduce_loss), captured in the
step's CUDA graph.

Exactness contract: every rank compiles its plan with the loss cardinality
|N| = world * per_gpu_batch (the global batch), draws the synthetic samples
[rank * B, (rank + 1) * B) of each iteration, and keys dropout masks by the
*global* sample index, so the sum of the ranks' gradients equals the
single-process gradient of the global batch (up to summation order).
"""
from __future__ import annotations

from .network import CompiledNetwork, compile_network


def shard_offset(rank: int, per_gpu_batch: int) -> int:
    """Global index of this rank's first sample (n0)."""
    return rank * per_gpu_batch


def compile_shard(name: str, per_gpu_batch: int, world: int, **kw) -> CompiledNetwork:
    """Per-rank plan: batch B, loss divided by the global batch G*B."""
    return compile_network(name, per_gpu_batch, global_batch=world * per_gpu_batch, **kw)


def broadcast_nccl_id(rank: int) -> bytes:
    """Rank 0 creates the NCCL unique id; torch.distributed broadcasts it."""
    import torch.distributed as dist

    from .runtime import nccl_unique_id

    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]
