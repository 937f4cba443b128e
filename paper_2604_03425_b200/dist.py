"""Multi-GPU plumbing: torch.distributed process groups and the reduce-scatter
hook libaegis calls for sharded PCMM.

Only the PCMM accumulators cross GPUs, and only when there are more ranks than
token groups (world = m * groups): each of the m ranks of a token group holds
partial sums for all of the group's output lanes; one reduce-scatter (uint64
sum -- residues < 2^46, so m * p never wraps) leaves each rank the complete
sums for the lanes it owns, which libaegis then reduces mod p.
"""
import torch
import torch.distributed as dist


class _CudaWords:
    """Zero-copy view of `words` int64 at a raw device pointer."""

    def __init__(self, ptr, words):
        self.__cuda_array_interface__ = {"shape": (int(words),), "typestr": "<i8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def reduce_scatter_words(full, part, group):
    """full: int64 tensor of m*W words; afterwards full[part*W:(part+1)*W] holds
    the element-wise sum over the group (two's-complement uint64 arithmetic)."""
    m = dist.get_world_size(group)
    w = full.numel() // m
    out = full[part * w:(part + 1) * w]
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, full, op=dist.ReduceOp.SUM, group=group)
    else:  # gloo has no reduce_scatter: all-reduce and keep our share
        tmp = full.clone()
        dist.all_reduce(tmp, op=dist.ReduceOp.SUM, group=group)
        out.copy_(tmp[part * w:(part + 1) * w])
    return out


def token_group_comms(world, tg_total):
    """One process group per token group when world = m * tg_total (m > 1).
    Every rank must call this (torch.distributed.new_group is collective)."""
    if world <= tg_total:
        return {}, 1
    m = world // tg_total
    groups = {}
    for t in range(tg_total):
        groups[t] = dist.new_group(ranks=list(range(t * m, (t + 1) * m)))
    return groups, m


def make_reducer(groups, part):
    """The callable handed to Graph.set_reducer: runs the NCCL reduce-scatter on
    the device buffer libaegis passes (its stream is idle at that point)."""
    def fn(buf_ptr, words_per_rank, group):
        g = groups[group]
        m = dist.get_world_size(g)
        full = torch.as_tensor(_CudaWords(buf_ptr, words_per_rank * m), device="cuda")
        reduce_scatter_words(full, part, g)
        torch.cuda.current_stream().synchronize()
    return fn
