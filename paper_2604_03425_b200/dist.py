"""Multi-GPU plumbing: torch.distributed process groups and the reduce-scatter
hook libaegis calls for sharded PCMM.

Only the PCMM accumulators cross GPUs, and only when there are more ranks than
token groups (world = m * groups): each of the m ranks of a token group holds
partial sums for all of the group's output lanes; one reduce-scatter (uint64
sum -- residues < 2^46, so m * p never wraps) leaves each rank the complete
sums for the lanes it owns, which libaegis then reduces mod p.
"""
import ctypes

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


class P2pReducer:
    """The reduce hook over CUDA IPC / NVLink peer memory (csrc/p2p.cu) instead of
    an NCCL collective: every rank of a token group exposes a staging window,
    and each rank's kernel sums its share directly out of the m windows.
    Windows are created lazily at the first reduction of a group (all m ranks
    reach it together) and grown collectively when a larger one is needed."""

    def __init__(self, ctx, groups, part):
        self.ctx, self.groups, self.part = ctx, groups, part
        self.win = {}  # token group -> (handle, bytes)
        self.fallback = None  # NCCL reducer if any rank of the group cannot map the windows

    def _window(self, group, nbytes):
        w = self.win.get(group)
        if w is not None and w[1] >= nbytes:
            return w[0]
        lib = self.ctx.lib
        if w is not None:  # forget the old window before freeing it (no second destroy in close())
            del self.win[group]
            lib.aegis_p2p_destroy(w[0])
        g = self.groups[group]
        m = dist.get_world_size(g)
        raw = (ctypes.c_char * 64)()
        h = ctypes.c_void_p()
        err = ""
        try:
            self.ctx._call("aegis_p2p_create", nbytes, ctypes.cast(raw, ctypes.c_void_p), ctypes.byref(h))
        except Exception as e:  # noqa: BLE001 -- decided collectively below
            err = repr(e)
            h = ctypes.c_void_p()
        handles = [None] * m  # every rank reaches this gather, so a local failure cannot hang the others
        dist.all_gather_object(handles, (bytes(raw), err), group=g)
        err = next((e for _, e in handles if e), "")
        if not err:
            allh = ctypes.create_string_buffer(b"".join(r for r, _ in handles), 64 * m)
            try:
                self.ctx._call("aegis_p2p_open", h, ctypes.cast(allh, ctypes.c_void_p), m, self.part)
            except Exception as e:  # noqa: BLE001 -- decided collectively below
                err = repr(e)
            errs = [None] * m
            dist.all_gather_object(errs, err, group=g)
            err = next((e for e in errs if e), "")
        if err:
            import sys
            print(f"aegis: peer-memory windows unavailable ({err}); using the NCCL reduce-scatter", file=sys.stderr)
            if h.value:
                lib.aegis_p2p_destroy(h)
            self.fallback = make_reducer(self.groups, self.part)
            return None
        self.win[group] = (h, nbytes)
        return h

    def __call__(self, buf_ptr, words_per_rank, group):
        if self.fallback:
            return self.fallback(buf_ptr, words_per_rank, group)
        g = self.groups[group]
        m = dist.get_world_size(g)
        h = self._window(group, words_per_rank * m * 8)
        if h is None:
            return self.fallback(buf_ptr, words_per_rank, group)
        self.ctx._call("aegis_p2p_stage", h, ctypes.c_void_p(buf_ptr), words_per_rank * m)
        dist.barrier(group=g)  # every window holds its rank's partial sums
        self.ctx._call("aegis_p2p_reduce", h, ctypes.c_void_p(buf_ptr + self.part * words_per_rank * 8),
                       words_per_rank, self.part)
        dist.barrier(group=g)  # nobody restages before every peer has read

    def close(self):
        for h, _ in self.win.values():
            self.ctx.lib.aegis_p2p_destroy(h)
        self.win = {}


def attach_p2p(ctx, graph, groups, part):
    """The default multi-GPU data plane: one peer-memory window per rank, opened
    over its token group through CUDA IPC (handles exchanged once, here), and
    attached to the graph so every sharded PCMM exchange runs on the context's
    comm stream with device-side flags -- no Python and no host barrier inside
    graph.run().  Returns the window (keep it alive while the graph runs), or
    None when no token group spans several ranks.  If any rank of the group
    cannot map the windows, every rank of it gets None (decided collectively)
    and the caller falls back to a reduce hook."""
    nbytes = graph.p2p_bytes()
    if nbytes == 0:
        return None
    g = groups[graph.shard_info()["tg_lo"]]
    m = dist.get_world_size(g)
    win, err = None, ""
    try:
        win = ctx.p2p_window(nbytes)
    except Exception as e:  # noqa: BLE001 -- decided collectively below
        err = repr(e)
    handles = [None] * m
    dist.all_gather_object(handles, (win.handle if win else b"", err), group=g)
    err = next((e for _, e in handles if e), "")
    if not err:
        try:
            win.open_ipc([h for h, _ in handles], part)
        except Exception as e:  # noqa: BLE001
            err = repr(e)
        errs = [None] * m
        dist.all_gather_object(errs, err, group=g)
        err = next((e for e in errs if e), "")
    if err:
        import sys
        print(f"aegis: peer-memory windows unavailable ({err}); using a reduce hook", file=sys.stderr)
        if win:
            win.close()
        return None
    graph.set_p2p(win)
    return win
