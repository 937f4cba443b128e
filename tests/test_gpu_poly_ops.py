"""GPU parity of the poly-instruction surface of the C-ABI (SURVEY §8(a) A18/A19,
§8(b)): the pointwise kLimbMulAdd opcodes on a FragSpan (poly_ir.hpp:49-58,
192-213), kLimbDrop (poly_ir.hpp:341-354), kPAdd, kEncode/kGenerate and the
multi-offset hoisted rotation.  Expected values: Python big-integer arithmetic
(pointwise ops), the CPU oracle (weights, rescale, rotation) and, for the
hoisted rotation, bit-identity with separate aegis_rot calls.
"""
import numpy as np
import pytest

from oracle_py import Oracle
from tools_params import main_primes

pytestmark = pytest.mark.gpu

MP = main_primes()
_ctx = {}


def ctx(logn):
    from paper_2604_03425_b200 import Context
    if logn not in _ctx:
        _ctx[logn] = Context(log_n=logn)
    return _ctx[logn]


def rand_bundle(rng, lanes, comps, level, n):
    a = np.empty((lanes, comps, level, n), dtype=np.uint64)
    for lb in range(level):
        a[:, :, lb, :] = rng.integers(0, MP[lb], (lanes, comps, n), dtype=np.uint64)
    return a


def upload(c, arr):
    b = c.bundle(arr.shape[0], arr.shape[1], arr.shape[2])
    b.upload(arr)
    return b


def big(a):
    return a.astype(object)


def modp(v, lb):
    return np.asarray(v % MP[lb], dtype=np.uint64)


@pytest.mark.parametrize("logn", [10, 16])
def test_limb_ops_on_a_fragspan(logn):
    """Every LimbOpcode on limbs [1, 3] of lanes [1, 3) with wrapped operand lanes;
    limbs and lanes outside the span are untouched."""
    from paper_2604_03425_b200 import _lib as L
    c = ctx(logn)
    n, level, lo, hi = 1 << logn, 5, 1, 3
    rng = np.random.default_rng(7)
    A = rand_bundle(rng, 2, 2, level, n)     # ciphertext operand, 2 lanes (wrapped onto 2 out lanes)
    Bc = rand_bundle(rng, 1, 2, level, n)    # ciphertext, 1 lane (broadcast)
    Pt = rand_bundle(rng, 1, 1, level, n)    # plaintext
    O0 = rand_bundle(rng, 4, 3, level, n)    # prior output contents
    a, bc, pt = upload(c, A), upload(c, Bc), upload(c, Pt)

    def run(op, b_arr, b_buf, comps_out):
        o = upload(c, O0)
        c.limb_op(op, o, a, b_buf, lo=lo, hi=hi, lanes=2, out_lane=1, a_slice=(0, 2),
                  b_slice=(0, 1) if b_buf is not None else None)
        got = o.download()
        exp = O0.copy()
        for l in range(2):
            for lb in range(lo, hi + 1):
                x = [big(A[l, cc, lb]) for cc in range(2)]
                y = [big(b_arr[0, cc, lb]) for cc in range(b_arr.shape[1])] if b_arr is not None else None
                prev = [big(O0[1 + l, cc, lb]) for cc in range(3)]
                if op == L.LIMB_ADD:
                    r = [x[0] + y[0], x[1] + (y[1] if len(y) > 1 else 0)]
                elif op == L.LIMB_SUB:
                    r = [x[0] - y[0], x[1] - (y[1] if len(y) > 1 else 0)]
                elif op in (L.LIMB_MUL, L.LIMB_MULACC):
                    if len(y) == 2:
                        r = [x[0] * y[0], x[0] * y[1] + x[1] * y[0], x[1] * y[1]]
                    else:
                        r = [x[0] * y[0], x[1] * y[0]]
                    if op == L.LIMB_MULACC:
                        r = [r[k] + prev[k] for k in range(len(r))]
                elif op == L.LIMB_ADDACC:
                    r = [prev[0] + x[0], prev[1] + x[1], prev[2]]
                for k in range(comps_out):
                    exp[1 + l, k, lb] = modp(r[k], lb)
        assert (got == exp).all(), op
        o.free()

    run(L.LIMB_ADD, Bc, bc, 2)
    run(L.LIMB_SUB, Bc, bc, 2)
    run(L.LIMB_ADD, Pt, pt, 2)     # PAdd form: pt feeds component 0
    run(L.LIMB_MUL, Bc, bc, 3)     # ciphertext tensor ("component product")
    run(L.LIMB_MUL, Pt, pt, 2)     # PMult form
    run(L.LIMB_MULACC, Pt, pt, 2)
    run(L.LIMB_MULACC, Bc, bc, 3)
    run(L.LIMB_ADDACC, None, None, 3)
    for b in (a, bc, pt):
        b.free()


def test_limb_op_rejects_bad_requests():
    from paper_2604_03425_b200 import _lib as L
    c = ctx(10)
    a, o = c.bundle(2, 2, 4), c.bundle(2, 3, 4)
    with pytest.raises(ValueError, match="kKeyMul"):
        c.limb_op(L.LIMB_KEYMUL, o, a, a)
    with pytest.raises(ValueError, match="prime range"):
        c.limb_op(L.LIMB_ADD, o, a, a, lo=0, hi=4)
    with pytest.raises(ValueError, match="overlaps"):
        c.limb_op(L.LIMB_ADD, a, a, a, lanes=1, out_lane=1, a_slice=(0, 2))
    with pytest.raises(ValueError):
        c.limb_op(99, o, a, a)
    small = c.bundle(2, 2, 4)
    with pytest.raises(ValueError, match="too few components"):
        c.limb_op(L.LIMB_MUL, small, a, a)  # the tensor needs 3 components
    for b in (a, o, small):
        b.free()


def test_padd_and_encode_match_the_oracle_weights():
    """kEncode writes the kGenerate rows the PMult kernel generates in-kernel
    (oracle weight_limb), and PAdd adds them to component 0."""
    c, o = ctx(10), Oracle(10)
    n, level, wb = 1 << 10, 4, 17
    rng = np.random.default_rng(3)
    W = c.bundle(3, 1, level)
    c.encode(W, wb, level)
    w = W.download()
    for lane in range(3):
        for lb in range(level):
            assert (w[lane, 0, lb] == o.weight_limb(wb, lane, lb)).all()
    X = rand_bundle(rng, 3, 2, level, n)
    x = upload(c, X)
    out = c.bundle(3, 2, level)
    c.padd(out, x, W, level)
    got = out.download()
    for lb in range(level):
        assert (got[:, 0, lb] == modp(big(X[:, 0, lb]) + big(w[:, 0, lb]), lb)).all()
        assert (got[:, 1, lb] == X[:, 1, lb]).all()
    for b in (W, x, out):
        b.free()


def test_stored_weights_reproduce_the_fused_pcmm():
    """PCMM through stored plaintexts (kEncode + per-limb MulAcc) equals the
    fused aegis_pmult_acc, whose weights are generated in-kernel."""
    from paper_2604_03425_b200 import _lib as L
    c = ctx(10)
    n, level, c_in, c_out, wb = 1 << 10, 3, 2, 3, 5
    rng = np.random.default_rng(11)
    X = rand_bundle(rng, c_in, 2, level, n)
    x = upload(c, X)
    fused, stored = c.bundle(c_out, 2, level), c.bundle(c_out, 2, level)
    zero = np.zeros((c_out, 2, level, n), dtype=np.uint64)
    fused.upload(zero)
    stored.upload(zero)
    c.pmult_acc(fused, x, wb, c_in * c_out, level)
    W = c.bundle(c_in * c_out, 1, level)
    c.encode(W, wb, level)
    for ci in range(c_in):
        for o_ in range(c_out):
            c.limb_op(L.LIMB_MULACC, stored, x, W, lanes=1, out_lane=o_, a_slice=(ci, 1),
                      b_slice=(ci * c_out + o_, 1))
    assert (fused.download() == stored.download()).all()
    for b in (x, fused, stored, W):
        b.free()


@pytest.mark.parametrize("logn,level", [(10, 5), (16, 17)])
def test_limb_drop_modes(logn, level):
    from paper_2604_03425_b200 import _lib as L
    c, o = ctx(logn), Oracle(logn)
    rng = np.random.default_rng(5)
    X = rand_bundle(rng, 2, 2, level, 1 << logn)
    x = upload(c, X)
    out = c.bundle(2, 2, level - 1)
    c.limb_drop(out, x, level, mode=L.MODE_NONE)
    assert (out.download() == X[:, :, :level - 1]).all()
    c.limb_drop(out, x, level, mode=L.MODE_RESCALE_TAIL)
    got = out.download()
    for ln in range(2):
        assert (got[ln] == o.rescale(X[ln], level)).all()
    with pytest.raises(ValueError, match="mode"):
        c.limb_drop(out, x, level, mode=L.MODE_BOOT_RESET)
    x.free()
    out.free()


@pytest.mark.parametrize("logn,level,lanes", [(10, 6, 3), (16, 17, 2)])
def test_rot_hoisted_equals_separate_rotations(logn, level, lanes):
    """One ModUp shared by several offsets (he_ir.hpp:224-241 rotation ladder) is
    bit-identical to separate rotations, and to the oracle."""
    c, o = ctx(logn), Oracle(logn)
    offsets = [1, 5, -3]
    c.keys_generate([1000 + r for r in offsets])
    rng = np.random.default_rng(9)
    X = rand_bundle(rng, lanes, 2, level, 1 << logn)
    x = upload(c, X)
    hoisted = [c.bundle(lanes + 1, 2, level) for _ in offsets]
    c.rot_hoisted(hoisted, x, offsets, level, out_lanes=[1] * len(offsets))
    for k, r in enumerate(offsets):
        sep = c.bundle(lanes, 2, level)
        c.rot(sep, x, r, level)
        h = hoisted[k].download()[1:]
        assert (h == sep.download()).all(), r
        if logn == 10 or k == 0:
            assert (h[0] == o.rotate(X[0], level, r)).all(), r
        sep.free()
    for b in hoisted + [x]:
        b.free()


# ---------------------------------------------------------------------------
# stored plaintexts and the wire format (SURVEY §8(d) stored variant, §8(f) rank 4)
@pytest.mark.parametrize("logn,tg,c_in,c_out,level", [(10, 1, 2, 3, 3), (16, 2, 3, 4, 5)])
def test_pmult_acc_stored_equals_generated(logn, tg, c_in, c_out, level):
    """PCMM reading stored weights (aegis_pmult_acc_stored) is bit-identical to
    the fused kernel that generates them in registers."""
    c = ctx(logn)
    n, wb = 1 << logn, 9
    rng = np.random.default_rng(13)
    X = rand_bundle(rng, tg * c_in, 2, level, n)
    x = upload(c, X)
    A0 = rand_bundle(rng, tg * c_out, 2, level, n)
    fused, stored = upload(c, A0), upload(c, A0)
    c.pmult_acc(fused, x, wb, c_in * c_out, level)
    W = c.bundle(c_in * c_out, 1, level)
    c.encode(W, wb, level)
    c.pmult_acc_stored(stored, x, W, level)
    assert (fused.download() == stored.download()).all()
    for b in (x, fused, stored, W):
        b.free()


def test_stored_weights_graph_matches_oracle(golden_dir):
    """The whole config-1 op sequence (N = 2^10) with every Encode written to HBM
    and every PMult reading it: every ciphertext bundle hash equals the oracle's."""
    from conftest import golden_graph
    c, o = ctx(10), Oracle(10)
    path = golden_graph("ffn_n10_t8", golden_dir)
    g = c.load_graph(path)
    g.set_stored_weights(True)
    got = g.run(hashes=True)
    want = o.run_graph(path)
    assert (got == want).all()
    g.set_stored_weights(False)


def test_bundle_store_round_trip(tmp_path):
    from paper_2604_03425_b200 import Context
    c = ctx(10)
    rng = np.random.default_rng(21)
    X = rand_bundle(rng, 3, 2, 6, 1 << 10)
    b = upload(c, X)
    p = tmp_path / "b.aegs"
    c.bundle_save(b, p)
    r = c.bundle_load(p)
    assert (r.lanes, r.comps, r.level) == (3, 2, 6)
    assert (r.download() == X).all()
    raw = bytearray(open(p, "rb").read())
    raw[128 + 8 * 1000] ^= 1  # one flipped payload bit
    open(tmp_path / "bad.aegs", "wb").write(raw)
    with pytest.raises(ValueError, match="hash mismatch"):
        c.bundle_load(tmp_path / "bad.aegs")
    open(tmp_path / "short.aegs", "wb").write(bytes(raw[:len(raw) // 2]))
    with pytest.raises(ValueError, match="truncated"):
        c.bundle_load(tmp_path / "short.aegs")
    other = Context(log_n=11)
    with pytest.raises(ValueError, match="different ring"):
        other.bundle_load(p)
    with pytest.raises(ValueError, match="not a key"):
        c.keys_load(1001, p)
    for x in (b, r):
        x.free()


@pytest.mark.parametrize("logn", [10, 16])
def test_key_store_round_trip(logn, tmp_path):
    """A rotation key saved from one context and streamed into a fresh one
    (different key seed) rotates exactly as the original."""
    from paper_2604_03425_b200 import Context
    c = ctx(logn)
    level, off = 5, 3
    c.keys_generate([1000 + off])
    rng = np.random.default_rng(2)
    X = rand_bundle(rng, 2, 2, level, 1 << logn)
    x = upload(c, X)
    ref = c.bundle(2, 2, level)
    c.rot(ref, x, off, level)
    p = tmp_path / "k.aegs"
    c.keys_save(1000 + off, p)
    c2 = Context(log_n=logn, seed_key=0x1234)
    c2.keys_load(1000 + off, p)
    x2 = upload(c2, X)
    got = c2.bundle(2, 2, level)
    c2.rot(got, x2, off, level)
    assert (got.download() == ref.download()).all()
    with pytest.raises(ValueError, match="different forms"):
        c2.keys_load(0, p)  # a rotation key cannot become the relinearisation key
    for b in (x, ref):
        b.free()
