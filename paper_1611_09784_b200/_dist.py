"""Collectives on device tensors for any torch.distributed backend: NCCL works on the device tensors directly;
other backends (gloo, the CPU multi-process tests and the one-GPU functional test of the multi-rank path) go
through host copies."""

from __future__ import annotations


def _nccl(group=None) -> bool:
    import torch.distributed as dist

    return dist.get_backend(group) == "nccl"


def all_reduce(t, group=None, op=None):
    """In-place sum (or `op`) over the ranks of `group`."""
    import torch.distributed as dist

    op = dist.ReduceOp.SUM if op is None else op
    if not t.is_cuda or _nccl(group):
        dist.all_reduce(t, op=op, group=group)
        return t
    h = t.cpu()
    dist.all_reduce(h, op=op, group=group)
    t.copy_(h)
    return t


def all_gather_into_tensor(out, inp, group=None):
    """out[r * len(inp): (r + 1) * len(inp)] = inp of rank r."""
    import torch.distributed as dist

    if not inp.is_cuda or _nccl(group):
        dist.all_gather_into_tensor(out, inp, group=group)
        return out
    ho = out.new_empty(out.shape, device="cpu")
    dist.all_gather_into_tensor(ho, inp.cpu(), group=group)
    out.copy_(ho)
    return out
