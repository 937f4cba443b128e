"""Multi-GPU placement logic on CPU (no GPU needed).

Token-coherent sharding (placement.hpp:175-182): every lane of
every bundle belongs to exactly one rank, and no op reads a lane owned by
another rank -- except the PCMM inputs when several ranks share a token group,
which is exactly the reduce-scatter the executor performs.  The world-size-2
test runs two gloo processes.
"""
import gzip
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_03425_b200 import plan_graph

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def parse_ops(name):
    bundles, ops = [], []
    with gzip.open(os.path.join(GOLDEN, f"{name}.heops.gz"), "rt") as f:
        for ln in f:
            p = ln.split()
            if p and p[0] == "B":
                bundles.append((int(p[2]), int(p[5])))  # lanes, chunk
            elif p and p[0] == "O":
                nin = int(p[14])
                ins = [tuple(int(x) for x in p[15 + 3 * k:18 + 3 * k]) for k in range(nin)]
                ops.append(dict(kind=int(p[2]), out=(int(p[4]), int(p[5]), int(p[6])), ins=ins))
    return bundles, ops


def owned_masks(g, bundles):
    return [g.owned_lanes(b, lanes) for b, (lanes, _) in enumerate(bundles)]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_partition_complete_and_local(world):
    bundles, ops = parse_ops("block_n16_t2048")  # 4 token groups
    plans = []
    for r in range(world):
        g = plan_graph(log_n=16, tokens=2048, layers=1, kind=0)
        g.set_shard(world, r)
        plans.append(owned_masks(g, bundles))
        info = g.shard_info()
        assert info["tg_total"] == 4
        assert info["ranks_per_group"] == max(1, world // 4)
    # every non-weight lane owned exactly once
    for b, (lanes, _) in enumerate(bundles):
        cnt = sum(p[b].astype(int) for p in plans)
        if cnt.sum() == 0:
            continue  # kGenerate weight bundles carry no data
        assert (cnt == 1).all(), b
    # locality: owned output lane -> every operand lane owned by the same rank
    cross = 0
    for op in ops:
        if op["kind"] == 0:
            continue
        ob, ol, n = op["out"]
        for r in range(world):
            m = plans[r]
            for l in np.nonzero(m[ob][ol:ol + n])[0]:
                for (ib, il, ic) in op["ins"]:
                    if op["kind"] == 3:  # PMult: checked separately
                        continue
                    src = il + (l if ic == n else l % ic)
                    if not m[ib][src]:
                        cross += 1
    assert cross == 0
    # PMult inputs: local when ranks own whole token groups
    if world <= 4:
        for op in ops:
            if op["kind"] != 3:
                continue
            (xb, xl, xc), (wb, wl, wc) = op["ins"]
            ob, ol, n = op["out"]
            tg = int(round((xc * n / wc) ** 0.5))
            c_in = xc // tg
            for r in range(world):
                m = plans[r]
                for t in range(tg):
                    owns_x = m[xb][xl + t * c_in: xl + (t + 1) * c_in]
                    assert owns_x.all() or not owns_x.any()


def test_shard_rejects_bad_world():
    g = plan_graph(log_n=16, tokens=2048, layers=1, kind=0)
    with pytest.raises(ValueError):
        g.set_shard(6, 0)  # neither divides nor is a multiple of 4 token groups


def test_shard_detects_cross_group_coupling():
    """When score lanes < A.V output lanes the reference's A.V reads wrapped
    score lanes (he_ir.hpp:533-541) from another token
    group: token sharding would need a collective there, so it is refused
    with the reference's logic_error type.  BASELINE configs (T=2048, N=2^16)
    never wrap."""
    from paper_2604_03425_b200 import LogicError
    g = plan_graph(log_n=11, tokens=32, layers=1, kind=0)
    with pytest.raises(LogicError, match="token groups"):
        g.set_shard(2, 0)
    g = plan_graph(log_n=11, tokens=64, layers=1, kind=0)
    g.set_shard(8, 3)
    assert g.shard_info() == {"tg_total": 4, "tg_lo": 1, "tg_hi": 2, "ranks_per_group": 2, "part": 1}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_03425_b200.dist import reduce_scatter_words
    # ownership masks of every bundle, gathered across ranks
    g = plan_graph(log_n=16, tokens=2048, layers=1, kind=0)
    g.set_shard(world, rank)
    nb = g.info()[1]
    bundles, _ = parse_ops("block_n16_t2048")
    mine = torch.tensor(np.concatenate([g.owned_lanes(b, bundles[b][0]) for b in range(nb)]).astype(np.int64))
    allm = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allm, mine)
    total = sum(allm)
    # the reduce-scatter semantics used for PCMM partial sums (uint64 wrap)
    w = 5
    full = torch.arange(world * w, dtype=torch.int64) * (rank + 1) + (1 << 62)
    out = reduce_scatter_words(full.clone(), rank, dist.group.WORLD).clone()
    exp = sum(torch.arange(world * w, dtype=torch.int64) * (r + 1) + (1 << 62) for r in range(world))
    ok_rs = bool((out == exp[rank * w:(rank + 1) * w]).all())
    q.put((rank, int((total > 1).sum()), int(total.sum()), ok_rs))
    dist.destroy_process_group()


def test_two_rank_gloo_partition():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, overlaps, owned_total, ok_rs in res:
        assert overlaps == 0 and ok_rs
    assert res[0][2] == res[1][2] > 0


def test_split_token_group_refuses_wrapping_shapes():
    """A token group split over m > 1 ranks is exact only when every lane-local
    op reads lanes of its own part; at very small T the score accumulator wraps
    onto fewer lanes than its consumers, so the plan must refuse (not compute
    garbage), while the production shape (T = 2048, 8 ranks) is accepted."""
    from paper_2604_03425_b200.api import plan_graph
    g = plan_graph(log_n=11, tokens=16)
    with pytest.raises(ValueError, match="token group split"):
        g.set_shard(2, 0)
    g = plan_graph(log_n=11, tokens=64)
    g.set_shard(8, 1)
    assert g.shard_info()["ranks_per_group"] == 2
