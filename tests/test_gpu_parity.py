"""GPU parity: every libaegis kernel path vs the CPU oracle, bit-exact on every
RNS residue (the bar for integer work).  Runs on a B200 via gpurun.

Sizes: toy (N=2^4), small (2^10-2^12) and production (2^16, 2^17) rings.  At
production size the oracle is only asked for a few lanes / limbs; full-size
properties (inverse(forward(x)) == x, automorphism group law) cover the rest.
"""
import numpy as np
import pytest

from conftest import golden_graph
from oracle_py import Oracle, hash_bundle
from tools_params import main_primes, special_primes

pytestmark = pytest.mark.gpu

MP, SP = main_primes(), special_primes()


def prime_of(e):
    return MP[e] if e < 60 else SP[e - 60]


_ctx = {}
_orc = {}


def ctx(logn):
    from paper_2604_03425_b200 import Context
    if logn not in _ctx:
        _ctx[logn] = Context(log_n=logn)
    return _ctx[logn]


def orc(logn):
    if logn not in _orc:
        _orc[logn] = Oracle(logn)
    return _orc[logn]


def rand_bundle(rng, lanes, comps, level, n):
    a = np.empty((lanes, comps, level, n), dtype=np.uint64)
    for lb in range(level):
        a[:, :, lb, :] = rng.integers(0, prime_of(lb), (lanes, comps, n), dtype=np.uint64)
    return a


def upload(c, arr):
    b = c.bundle(arr.shape[0], arr.shape[1], arr.shape[2])
    b.upload(arr)
    return b


@pytest.fixture(params=[0, 1, 2], ids=["int", "f64", "f64v1"])
def ntt_impl(request):
    from paper_2604_03425_b200 import _lib
    lib = _lib.load()
    old = lib.aegis_ntt_impl(-1)
    lib.aegis_ntt_impl(request.param)
    yield request.param
    lib.aegis_ntt_impl(old)


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("logn", [4, 5, 10, 12, 13, 16, 17])
def test_ntt_forward_inverse(logn, ntt_impl):
    c, o = ctx(logn), orc(logn)
    rng = np.random.default_rng(logn)
    level = 3 if logn >= 16 else 6
    x = rand_bundle(rng, 2, 2, level, 1 << logn)
    b = upload(c, x)
    c.ntt(b)
    f = b.download()
    for ln in range(2):
        for cp in range(2):
            exp = o.ntt(x[ln, cp], list(range(level)))
            assert (f[ln, cp] == exp).all(), (ln, cp)
    c.ntt(b, inverse=True)
    assert (b.download() == x).all()


def test_ntt_all_primes_production(ntt_impl):
    """inverse(forward(x)) == x on every one of the 64 primes at N = 2^16, and
    bit-exact vs the oracle on a sample of them (including the specials)."""
    c, o = ctx(16), orc(16)
    n = 1 << 16
    rng = np.random.default_rng(1)
    x = rand_bundle(rng, 1, 1, 35, n)
    b = upload(c, x)
    c.ntt(b)
    f = b.download()
    for lb in (0, 1, 17, 34):
        assert (f[0, 0, lb] == o.ntt(x[0, 0, lb], [lb])).all()
    c.ntt(b, inverse=True)
    assert (b.download() == x).all()


def test_ntt_fragment_addressing():
    """FragSpan-style sub-ranges (poly_ir.hpp:87-99) touch only their limbs."""
    c, o = ctx(10), orc(10)
    rng = np.random.default_rng(2)
    x = rand_bundle(rng, 3, 2, 6, 1 << 10)
    b = upload(c, x)
    c.ntt(b, lane=1, lanes=1, lo=2, hi=4)
    f = b.download()
    exp = x.copy()
    for cp in range(2):
        exp[1, cp, 2:5] = o.ntt(x[1, cp, 2:5], [2, 3, 4])
    assert (f == exp).all()


@pytest.mark.parametrize("logn", [4, 10, 16])
def test_automorphism(logn):
    c, o = ctx(logn), orc(logn)
    n = 1 << logn
    rng = np.random.default_rng(3)
    x = rand_bundle(rng, 2, 2, 4, n)
    b = upload(c, x)
    out = c.bundle(2, 2, 4)
    for off in (1, 5, 63, -1):
        k = o.L.orc_galois(off, n)
        c.automorphism(out, b, k)
        got = out.download()
        for ln in range(2):
            for cp in range(2):
                assert (got[ln, cp] == o.automorphism_eval(x[ln, cp], k)).all()


def test_basis_convert_near_ties():
    c, o = ctx(4), orc(4)
    n = 16
    src, dst = [0, 1, 2, 3], [4, 5, 60, 63]
    B = 1
    for e in src:
        B *= prime_of(e)
    h = (B - 1) // 2
    vals = [0, 1, B - 1, h, h + 1, h - 1, h + 2, h - 2, B - 2, 12345, B // 3, 2 * B // 3, h + 7, h - 7, 2, 3]
    x = np.zeros((1, 1, 4, n), dtype=np.uint64)
    for i, e in enumerate(src):
        x[0, 0, i] = [v % prime_of(e) for v in vals]
    bi = upload(c, x)
    bo = c.bundle(1, 1, 6)
    c.basis_convert(bo, bi, src, [0, 1, 2, 3], dst, [0, 1, 2, 3])
    got = bo.download()[0, 0, :4]
    exp, fb = o.basis_convert(x[0, 0], src, dst)
    assert fb > 0
    assert (got == exp).all()


@pytest.mark.parametrize("logn,k", [(10, 1), (10, 4), (12, 21), (16, 4)])
def test_basis_convert_random(logn, k):
    c, o = ctx(logn), orc(logn)
    n = 1 << logn
    rng = np.random.default_rng(k)
    src = list(range(k))
    dst_ext = list(range(k, min(35, k + 10))) + [60, 63]
    x = rand_bundle(rng, 2, 1, k, n)
    bi = upload(c, x)
    bo = c.bundle(2, 1, len(dst_ext))
    c.basis_convert(bo, bi, src, src, dst_ext, list(range(len(dst_ext))))
    got = bo.download()
    for ln in range(2):
        exp, _ = o.basis_convert(x[ln, 0], src, dst_ext)
        assert (got[ln, 0] == exp).all()


@pytest.mark.parametrize("logn,level", [(4, 1), (4, 5), (10, 3), (10, 9), (12, 17), (16, 6), (16, 17), (16, 34)])
@pytest.mark.parametrize("key", [0, 1007])
def test_keyswitch(logn, level, key):
    c, o = ctx(logn), orc(logn)
    n = 1 << logn
    rng = np.random.default_rng(level)
    x = rand_bundle(rng, 2, 2, level, n)
    bi = upload(c, x)
    bo = c.bundle(2, 2, level)
    c.keyswitch(bo, bi, 1, level, key)
    got = bo.download()
    for ln in range(2):
        o0, o1 = o.keyswitch(x[ln, 1], level, key)
        assert (got[ln, 0] == o0).all() and (got[ln, 1] == o1).all()


@pytest.mark.parametrize("logn,level,offset", [(10, 5, 1), (10, 17, 63), (12, 9, -1), (16, 3, 32), (16, 17, -5)])
def test_rot(logn, level, offset):
    c, o = ctx(logn), orc(logn)
    n = 1 << logn
    rng = np.random.default_rng(offset & 0xff)
    x = rand_bundle(rng, 3, 2, level + 1, n)  # operand one level higher: limb-drop read
    bi = upload(c, x)
    bo = c.bundle(3, 2, level)
    c.rot(bo, bi, offset, level)
    got = bo.download()
    for ln in range(3):
        exp = o.rotate(x[ln, :, :level], level, offset)
        assert (got[ln] == exp).all(), ln


@pytest.mark.parametrize("logn,level,offset", [(10, 3, 0), (10, 3, -499), (10, 2, 511), (10, 1, 5), (17, 5, 7)])
def test_rot_edges(logn, level, offset):
    """Edge offsets and shapes: offset 0 (galois 1: a plain key switch), the most
    negative offset a key id allows (-499), N/2 - 1, level 1 (one digit of one
    prime) and the N = 2^17 ring."""
    c, o = ctx(logn), orc(logn)
    n = 1 << logn
    rng = np.random.default_rng(abs(offset) + level)
    x = rand_bundle(rng, 2, 2, level, n)
    bi = upload(c, x)
    bo = c.bundle(2, 2, level)
    c.rot(bo, bi, offset, level)
    got = bo.download()
    for ln in range(2):
        assert (got[ln] == o.rotate(x[ln], level, offset)).all(), ln
    with pytest.raises(ValueError):
        c.rot(bo, bi, -500, level)  # key id 500 would collide with the relin id space


def test_keyswitch_full_chain_60():
    """A 60-prime chain (the config-5 sweep's context) at its top level: 15 digits,
    64 extended slots -- the largest conversion and key product shapes."""
    from paper_2604_03425_b200 import Context
    from oracle_py import Oracle
    c, o = Context(log_n=16, chain_length=60, bootstrap_level=14), Oracle(16, chain=60)
    level = 60
    rng = np.random.default_rng(60)
    x = rand_bundle(rng, 1, 2, level, 1 << 16)
    bi = upload(c, x)
    bo = c.bundle(1, 2, level)
    c.rot(bo, bi, 3, level)
    assert (bo.download()[0] == o.rotate(x[0], level, 3)).all()
    c.close()


@pytest.mark.parametrize("logn,level", [(10, 4), (10, 16), (16, 3)])
def test_cmult_relin(logn, level):
    c, o = ctx(logn), orc(logn)
    n = 1 << logn
    rng = np.random.default_rng(level)
    a = rand_bundle(rng, 2, 2, level, n)
    b = rand_bundle(rng, 2, 2, level, n)
    ba, bb = upload(c, a), upload(c, b)
    prod = c.bundle(2, 3, level)
    c.cmult(prod, ba, bb, level)
    t = prod.download()
    for ln in range(2):
        assert (t[ln] == o.cmult(a[ln], b[ln], level)).all()
    c.relin(prod, level)
    r = prod.download()
    for ln in range(2):
        assert (r[ln, :2] == o.relin(t[ln], level)).all()


@pytest.mark.parametrize("logn,level", [(10, 4), (16, 7)])
def test_cmult_square(logn, level):
    """CMult of a ciphertext with itself takes the squaring kernel (2 operand
    streams, 3 products); it must equal the general tensor product."""
    c, o = ctx(logn), orc(logn)
    rng = np.random.default_rng(level + 100)
    a = rand_bundle(rng, 3, 2, level, 1 << logn)
    ba = upload(c, a)
    prod = c.bundle(3, 3, level)
    c.cmult(prod, ba, ba, level)
    t = prod.download()
    for ln in range(3):
        assert (t[ln] == o.cmult(a[ln], a[ln], level)).all()
    # the same bundle with different lane slices is a general product
    prod2 = c.bundle(2, 3, level)
    c.cmult(prod2, ba, ba, level, lanes=2, a_slice=(0, 2), b_slice=(1, 2))
    t2 = prod2.download()
    for ln in range(2):
        assert (t2[ln] == o.cmult(a[ln], a[ln + 1], level)).all()


def test_cmult_lane_maps():
    """emit_per_lane wrap rule (he_ir.hpp:200-222): b lane = l % count."""
    c, o = ctx(10), orc(10)
    n = 1 << 10
    rng = np.random.default_rng(5)
    a = rand_bundle(rng, 6, 2, 3, n)
    b = rand_bundle(rng, 2, 2, 3, n)
    ba, bb = upload(c, a), upload(c, b)
    prod = c.bundle(4, 3, 3)
    c.cmult(prod, ba, bb, 3, lanes=4, a_slice=(2, 4), b_slice=(0, 2))
    t = prod.download()
    for ln in range(4):
        assert (t[ln] == o.cmult(a[2 + ln], b[ln % 2], 3)).all()


@pytest.mark.parametrize("logn,level", [(10, 2), (10, 17), (16, 5), (16, 35)])
def test_rescale(logn, level):
    c, o = ctx(logn), orc(logn)
    n = 1 << logn
    rng = np.random.default_rng(level)
    x = rand_bundle(rng, 2, 2, level, n)
    bi = upload(c, x)
    bo = c.bundle(2, 2, level - 1)
    c.rescale(bo, bi, level)
    got = bo.download()
    for ln in range(2):
        assert (got[ln] == o.rescale(x[ln], level)).all()


@pytest.mark.parametrize("logn,level,out_level", [(10, 1, 21), (10, 3, 21), (16, 1, 21), (10, 9, 4)])
def test_boot(logn, level, out_level):
    c, o = ctx(logn), orc(logn)
    n = 1 << logn
    rng = np.random.default_rng(level)
    x = rand_bundle(rng, 2, 2, level, n)
    bi = upload(c, x)
    bo = c.bundle(2, 2, out_level)
    c.boot(bo, bi, level, out_level)
    got = bo.download()
    for ln in range(2):
        assert (got[ln] == o.boot(x[ln], level, out_level)).all()


def test_cadd_forms():
    c = ctx(10)
    n = 1 << 10
    rng = np.random.default_rng(8)
    a = rand_bundle(rng, 4, 2, 3, n)
    b = rand_bundle(rng, 2, 2, 5, n)
    ba, bb = upload(c, a), upload(c, b)
    out = c.bundle(4, 2, 3)
    c.cadd(out, ba, bb, 3, b_slice=(0, 2))
    got = out.download()
    q = np.array([prime_of(i) for i in range(3)], dtype=np.uint64)[None, :, None]
    for ln in range(4):
        assert (got[ln] == (a[ln] + b[ln % 2, :, :3]) % q).all()
    c.cadd(out, bb, None, 3, accumulate=True, a_slice=(0, 2))
    got2 = out.download()
    for ln in range(4):
        assert (got2[ln] == (got[ln] + b[ln % 2, :, :3]) % q).all()


@pytest.mark.parametrize("tg,c_in,c_out,chunk", [(1, 3, 4, 0), (2, 2, 3, 0), (2, 3, 6, 6), (5, 2, 2, 0), (1, 2, 9, 0), (4, 5, 7, 0)])
def test_pmult_acc(tg, c_in, c_out, chunk):
    """Bundled PCMM step with in-kernel kGenerate weights."""
    c, o = ctx(10), orc(10)
    n = 1 << 10
    level = 3
    rng = np.random.default_rng(tg * 10 + c_in)
    x = rand_bundle(rng, tg * c_in, 2, level, n)
    acc0 = rand_bundle(rng, tg * c_out, 2, level, n)
    bx, bacc = upload(c, x), upload(c, acc0)
    wb = 77
    c.pmult_acc(bacc, bx, wb, c_in * c_out, level, chunk_period=chunk)
    got = bacc.download()
    S = 1 if chunk == 0 else (tg * c_out) // chunk
    c_sub = c_out // S
    for lb in range(level):
        p = prime_of(lb)
        W = [o.weight_limb(wb, lane, lb).astype(object) for lane in range(c_in * c_out)]
        for t in range(tg):
            for oo in range(c_out):
                lane = t * c_out + oo if S == 1 else (oo // c_sub) * chunk + t * c_sub + oo % c_sub
                for cp in range(2):
                    s = acc0[lane, cp, lb].astype(object)
                    for ci in range(c_in):
                        s = s + x[t * c_in + ci, cp, lb].astype(object) * W[ci * c_out + oo]
                    assert list(got[lane, cp, lb]) == list(s % p)


def test_input_fill_matches_oracle():
    c, o = ctx(10), orc(10)
    b = c.bundle(3, 2, 4)
    b.fill_input(42)
    got = b.download()
    assert (got == o.input_bundle(42, 3, 2, 4)).all()
    assert b.hash() == hash_bundle(got)


def test_errors_are_raised_not_crashes():
    c = ctx(10)
    b = c.bundle(2, 2, 3)
    with pytest.raises(ValueError):
        c.rescale(c.bundle(2, 2, 1), b, 1)  # cannot rescale below level 1
    with pytest.raises(ValueError):
        c.rot(c.bundle(2, 2, 3), b, 1, 5)  # level exceeds operand
    with pytest.raises(ValueError):
        c.bundle(1, 2, 99)  # level beyond the chain


# ---------------------------------------------------------------------------
# Layer-level parity: full HE-op graphs (reference op sequence) on the GPU vs
# the oracle's exec_sequential.  Every bundle's content hash at death must match.
@pytest.mark.parametrize("name,logn", [("ffn_n10_t8", 10), ("block_n10_t8", 10), ("ffn_n11_t32", 11),
                                       ("block_n11_t32", 11)])
def test_graph_parity_small(name, logn, golden_dir):
    path = golden_graph(name, golden_dir)
    c = ctx(logn)
    g = c.load_graph(path)
    h_gpu = g.run(hashes=True)
    h_cpu = orc(logn).run_graph(path)
    assert len(h_gpu) == len(h_cpu)
    bad = [i for i in range(len(h_gpu)) if h_gpu[i] != h_cpu[i]]
    assert not bad, f"{len(bad)} bundles differ, first {bad[:5]}"
    assert (h_gpu != 0).sum() > 100
    # the GPU's own lowering produces the same graph and the same residues
    g2 = c.graph(kind=1 if name.startswith("ffn") else 0, tokens=int(name.split("_t")[1]))
    assert (g2.run(hashes=True) == h_gpu).all()


@pytest.mark.parametrize("world,dce,stagger", [(2, False, False), (4, False, False), (8, False, False),
                                               (8, True, False), (8, False, True)])
def test_sharded_execution_matches(world, dce, stagger, tmp_path):
    """Token-group sharding on one GPU: the per-rank bundle
    hashes (owned lanes only) sum to the unsharded hashes.  N = 2^11, T = 64
    gives 4 token groups (score lanes >= output lanes, so attention stays
    inside a group as at T = 2048, N = 2^16); world = 8 puts 2 ranks on each
    group and exercises the PCMM reduce-scatter: the ranks run concurrently in
    threads, each with its own context, and the reducer hook sums the partner
    buffers on the device."""
    import threading
    import torch
    from paper_2604_03425_b200 import Context
    g0 = ctx(11).graph(kind=0, tokens=64)
    base = g0.run(hashes=True)
    path = str(tmp_path / "g.heops")
    g0.dump(path)
    final = [int(ln.split()[4]) for ln in open(path) if ln.startswith("O ")][-1]
    ctxs = [Context(log_n=11) for _ in range(world)]
    graphs = [c_.graph(kind=0, tokens=64) for c_ in ctxs]
    if stagger:  # each rank runs its own staggered diagonal order (aegis_graph_from_plan)
        plan = graphs[0].plan(world, reorder=True)
        graphs = [g.in_plan_order(plan, r) for r, g in enumerate(graphs)]
    for r, g in enumerate(graphs):
        g.set_shard(world, r)
        g.set_dce(dce)
    m = graphs[0].shard_info()["ranks_per_group"]
    bar = threading.Barrier(world)
    bufs = {}

    def reducer(rank):
        def fn(ptr, words, group):
            from paper_2604_03425_b200.dist import _CudaWords
            part = rank % m
            full = torch.as_tensor(_CudaWords(ptr, words * m), device="cuda")
            bufs[rank] = full
            bar.wait()
            peers = [bufs[group * m + q] for q in range(m)]
            s = sum(p[part * words:(part + 1) * words].clone() for p in peers)
            torch.cuda.synchronize()
            bar.wait()
            full[part * words:(part + 1) * words].copy_(s)
            torch.cuda.synchronize()
            bar.wait()
        return fn

    out = [None] * world
    errs = []

    def work(r):
        try:
            graphs[r].set_reducer(reducer(r))
            out[r] = graphs[r].run(hashes=True)
        except Exception as e:  # surfaced below
            errs.append(e)
            bar.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    total = np.zeros_like(base)
    for h in out:
        total = total + h  # uint64 wrap-around == the hash's mod 2^64 sum
    if dce:  # dead-lane elimination: only the layer output is defined
        assert total[final] == base[final]
        return
    bad = np.nonzero(total != base)[0]
    assert len(bad) == 0, f"{len(bad)} bundles differ, first {bad[:5]}"


PROD_FIXTURES = ["prod_ffn_n16_t128", "prod_block_n16_t512", "prod_block_n16_t2048_tg0", "prod_blocks2_n16_t512"]


@pytest.mark.slow
@pytest.mark.parametrize("fixture", PROD_FIXTURES)
def test_graph_parity_production(fixture, golden_dir):
    """BASELINE configs at production size (N = 2^16, L = 35), whole graph,
    every bundle hash vs the CPU oracle (fixtures from
    tests/golden/make_prod_hashes.py): config 1 (FFN, T = 128, 426 ops),
    config 2 (block, T = 512, 1,511 ops) and the headline T = 2048 layer run
    UNSHARDED exactly as bench.py runs it, hashed over the lanes of token group
    0 of 4 (the oracle computes only those lanes)."""
    import json
    import os
    from conftest import GOLDEN
    path = os.path.join(GOLDEN, fixture + ".json")
    if not os.path.exists(path):
        pytest.skip(f"{fixture}.json not generated yet (tests/golden/make_prod_hashes.py)")
    with open(path) as f:
        rec = json.load(f)
    want = np.array([int(x, 16) for x in rec["hashes"]], dtype=np.uint64)
    g = ctx(16).load_graph(golden_graph(rec["graph"], golden_dir))
    if rec["tg_sel"] >= 0:
        g.set_hash_group(rec["tg_sel"])
    got = g.run(hashes=True)
    assert len(got) == len(want) == rec["bundles"]
    bad = np.nonzero(got != want)[0]
    assert len(bad) == 0, f"{len(bad)} of {len(want)} bundles differ, first {bad[:8].tolist()}"
    assert (want != 0).sum() > len(want) // 2  # the fixture covers real data


@pytest.mark.parametrize("logn,tokens", [(11, 64), (11, 32)])
def test_dead_lane_elimination_keeps_final_bundle(logn, tokens, tmp_path):
    """The separately reported DCE variant skips rotated lanes no later op reads
    (A.V consumes only the first out_lanes of each rotated
    score bundle); the layer's output bundle must stay bit-identical."""
    c = ctx(logn)
    g = c.graph(kind=0, tokens=tokens)
    path = str(tmp_path / "g.heops")
    g.dump(path)
    final = [int(ln.split()[4]) for ln in open(path) if ln.startswith("O ")][-1]
    h = g.run(hashes=True)
    g2 = c.graph(kind=0, tokens=tokens)
    g2.set_dce(True)
    h2 = g2.run(hashes=True)
    assert h2[final] == h[final]
    # the score rotations rotate all QKV lanes but CMult reads only the Q lanes:
    # those rotated bundles keep uncomputed (dead) lanes under DCE, so their
    # whole-bundle hashes differ while the output bundle does not
    assert (h2 != h).any()


@pytest.mark.parametrize("logn,tokens", [(12, 128)])  # score.acc: 96 lanes += 48-lane products
def test_wrap_defer_bit_identical(logn, tokens):
    """Wrapped accumulation (score.acc += prod[j mod m]) summed at the operand's
    width and applied once: every bundle hash equals op-by-op execution, with
    fewer kernel launches."""
    c = ctx(logn)
    g = c.graph(kind=0, tokens=tokens)
    g.set_wrap_defer(False)
    l0 = c.launch_count()
    h = g.run(hashes=True)
    l1 = c.launch_count()
    g2 = c.graph(kind=0, tokens=tokens)
    h2 = g2.run(hashes=True)
    l2 = c.launch_count()
    assert (h2 == h).all()
    assert l2 - l1 < l1 - l0


def _small_batch_ctx():
    """A production-size context whose operator workspaces hold 1-2 lanes, so
    every lane-batch loop (ModUp, key product / ModDown, rescale) iterates."""
    import os
    from paper_2604_03425_b200 import Context
    old = os.environ.get("AEGIS_WS_SCALE")
    os.environ["AEGIS_WS_SCALE"] = "0.01"
    try:
        return Context(log_n=16)
    finally:
        if old is None:
            del os.environ["AEGIS_WS_SCALE"]
        else:
            os.environ["AEGIS_WS_SCALE"] = old


def test_multibatch_keyswitch_rescale_production():
    """Rot / Relin / Rescale over 6 lanes at N = 2^16, l = 17 with 1-2 lanes per
    batch: first, middle and last lanes bit-exact vs the oracle."""
    c, o = _small_batch_ctx(), orc(16)
    n, L = 1 << 16, 17
    rng = np.random.default_rng(77)
    x = rand_bundle(rng, 6, 2, L, n)
    bi = upload(c, x)
    br = c.bundle(6, 2, L)
    c.rot(br, bi, 5, L)
    got_r = br.download()
    p3 = c.bundle(6, 3, L)
    c.cmult(p3, bi, bi, L)
    t = p3.download()
    c.relin(p3, L)
    got_l = p3.download()
    bs = c.bundle(6, 2, L - 1)
    c.rescale(bs, bi, L)
    got_s = bs.download()
    for ln in (0, 3, 5):
        assert (got_r[ln] == o.rotate(x[ln], L, 5)).all(), ("rot", ln)
        assert (got_l[ln, :2] == o.relin(t[ln], L)).all(), ("relin", ln)
        assert (got_s[ln] == o.rescale(x[ln], L)).all(), ("rescale", ln)


def test_multibatch_hoisted_rotations_production(tmp_path):
    """Three hoisted rotations of one 6-lane source at N = 2^16, l = 17 through
    the graph executor with 1-2 lanes per batch: bundle hashes vs the oracle."""
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from bench_ops import graph
    path = str(tmp_path / "rot.heops")
    open(path, "w").write(graph("rot", 6, 3))
    c = _small_batch_ctx()
    g = c.load_graph(path)
    c.keys_generate(g.key_ids())
    h_gpu = g.run(hashes=True)
    h_cpu = orc(16).run_graph(path)
    assert (h_gpu[: len(h_cpu)] == h_cpu).all()


@pytest.mark.parametrize("level", [17, 35])
def test_ckks_real_keys_decrypt(level):
    """SURVEY §8(f) rank 3, first step: with a ternary secret, keys from
    aegis_keys_upload and real symmetric encryption (paper_2604_03425_b200.ckks),
    the GPU operators are correct CKKS operations -- CMult+Relin+Rescale decrypts
    to z^2 and Rot by r to the left-rotated slots (tolerances in the asserts)."""
    from paper_2604_03425_b200 import Context
    from paper_2604_03425_b200.ckks import Ckks
    c = Context(log_n=11)  # private context: uploaded keys must not leak into other tests
    try:
        k = Ckks(c, seed=7)
        rng = np.random.default_rng(level)
        z = rng.uniform(-1, 1, c.n // 2) + 1j * rng.uniform(-1, 1, c.n // 2)
        scale = 2.0 ** 40
        ct = k.encrypt(z, scale, level)
        assert np.abs(k.decrypt(ct, scale, level) - z).max() < 1e-7
        k.upload_relin_key()
        sq = c.bundle(1, 3, level)
        c.cmult(sq, ct, ct, level)
        c.relin(sq, level)
        out = c.bundle(1, 2, level - 1)
        c.rescale(out, sq, level)
        s2 = scale * scale / k.q[level - 1]
        assert np.abs(k.decrypt(out, s2, level - 1) - z * z).max() < 1e-6
        for r in (1, 7, -3):
            k.upload_rotation_key(r)
            o = c.bundle(1, 2, level)
            c.rot(o, ct, r, level)
            assert np.abs(k.decrypt(o, scale, level) - np.roll(z, -r)).max() < 1e-7
    finally:
        c.close()
