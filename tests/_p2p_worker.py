"""torchrun worker for tests/test_gpu_p2p.py: token-group shards whose PCMM
reduce-scatter runs over CUDA IPC peer memory (dist.P2pReducer, csrc/p2p.cu).
All ranks share GPU 0 (same-device IPC); rank 0 checks that the per-rank
bundle hashes sum to the unsharded run's and prints P2P_OK."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2604_03425_b200 import Context  # noqa: E402
from paper_2604_03425_b200.dist import P2pReducer, attach_p2p, make_reducer, token_group_comms  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, ws = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    tokens = int(os.environ.get("P2P_TOKENS", "64"))
    kind = int(os.environ.get("P2P_KIND", "0"))  # 1: the FFN graph (splittable at small T)
    c = Context(log_n=11)
    g = c.graph(kind=kind, tokens=tokens)
    if os.environ.get("P2P_STAGGER") == "1":  # this rank's staggered diagonal order (as bench.py runs ranks)
        g = g.in_plan_order(g.plan(ws, reorder=True), rank)
    g.set_shard(ws, rank)
    info = g.shard_info()
    groups, m = token_group_comms(ws, info["tg_total"])
    mode = os.environ.get("P2P_MODE", "device")
    g.set_fault(int(os.environ.get("P2P_FAULT", "0")))
    g.set_matmul_modes(os.environ.get("P2P_MODES", "0") == "1")  # before the window is sized
    win, red = None, None
    if mode == "device":  # the executor's own data plane: comm stream + flags in peer memory
        win = attach_p2p(c, g, groups, rank % m)
    else:
        red = P2pReducer(c, groups, rank % m)
        if mode == "collective":  # the torch.distributed path, for comparison
            red.fallback = make_reducer(groups, rank % m)
        g.set_reducer(red)
    trace = os.environ.get("P2P_TRACE") == "1"
    if trace:  # two-stream trace: the exchanges on the comm stream against the compute-stream ops
        g.set_profiling(True)
    h = g.run(hashes=True)
    if trace and rank == 0:
        ops = np.cumsum(np.concatenate([[0.0], g.op_times()]))
        _, bundles, opd, _ = g.export()
        for s0, s1, b in g.comm_times():
            busy = [(i, max(ops[i], s0), min(ops[i + 1], s1)) for i in range(len(ops) - 1)
                    if ops[i] < s1 and ops[i + 1] > s0]
            kinds = sorted({("encode", "padd", "cadd", "pmult", "cmult", "rot", "relin", "rescale", "boot")[opd[i].kind]
                            for i, _, _ in busy})
            print(f"TRACE exchange {bundles[b].tag.decode():28s} comm [{s0:9.3f}, {s1:9.3f}] ms; compute ops during it: "
                  f"{len(busy)} ({', '.join(kinds)}), first op {busy[0][0] if busy else -1}", flush=True)
    hs = [None] * ws
    dist.all_gather_object(hs, h.tolist())
    sent = [None] * ws
    dist.all_gather_object(sent, g.comm_bytes())
    planned = sum(e["bytes_total"] for e in g.plan(ws).events() if e["executed"])
    used = win is not None if mode == "device" else (red.fallback is None and len(red.win) > 0)
    if rank == 0:
        base = c.graph(kind=kind, tokens=tokens).run(hashes=True)
        total = np.zeros_like(base)
        for x in hs:
            total = total + np.array(x, dtype=np.uint64)
        bad = int((total != base).sum())
        print(f"P2P_{'OK' if bad == 0 else 'MISMATCH'} bundles={len(base)} bad={bad} m={m} used_p2p={used} "
              f"sent={sum(sent)} planned={planned}", flush=True)
    dist.barrier()  # no rank unmaps a window its peers may still read
    if red:
        red.close()
    if win:
        g.set_p2p(None)
        win.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
