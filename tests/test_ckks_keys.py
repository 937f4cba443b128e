"""CPU check of the secret-derived key format (paper_2604_03425_b200.ckks) against
the hybrid key switch the library implements (poly_ir.hpp:219-298):
ModUp = exact centred lift of each digit's residues to Q_l u P, key product,
ModDown = round(x / P).  Simulated with Python integers at N = 16 on the
production prime chain; the GPU test test_ckks_real_keys_decrypt runs the same
keys through the CUDA key switch."""
import numpy as np
import pytest

from tools_params import main_primes, special_primes

from paper_2604_03425_b200.ckks import ALPHA, SPECIAL_BASE, Ckks, automorphism_int, negacyclic_int

MP, SP = main_primes(), special_primes()


class _Primes:
    """Just enough of a Context for Ckks' key generation (no device)."""

    def __init__(self, log_n, chain):
        self.n, self.log_n, self.chain = 1 << log_n, log_n, chain

    def prime(self, e):
        return MP[e] if e < SPECIAL_BASE else SP[e - SPECIAL_BASE]


def _polymul(a, b, m):
    n = len(a)
    out = [0] * n
    for i, x in enumerate(a):
        if x:
            for j, y in enumerate(b):
                k = i + j
                if k < n:
                    out[k] += x * y
                else:
                    out[k - n] -= x * y
    return [v % m for v in out]


def _centre(x, m):
    x %= m
    return x - m if x > m // 2 else x


def _keyswitch(d, key, q, p, level):
    """Exact hybrid KS of integer polynomial d (mod Q_l) with a coefficient-domain key."""
    n = len(d)
    slots = q + p
    ext_slots = list(range(level)) + list(range(len(q), len(q) + len(p)))
    digits = -(-level // ALPHA)
    acc = [[[0] * n for _ in ext_slots] for _ in range(2)]
    for j in range(digits):
        dq = q[ALPHA * j: min(ALPHA * (j + 1), level)]
        Qj = 1
        for x in dq:
            Qj *= x
        lift = [_centre(v, Qj) for v in d]  # centred lift of [d]_{Q_j}
        for si, s in enumerate(ext_slots):
            m = slots[s]
            e = [v % m for v in lift]
            for c in range(2):
                prod = _polymul(e, [int(v) for v in key[j, c, s]], m)
                acc[c][si] = [(a + b) % m for a, b in zip(acc[c][si], prod)]
    P = 1
    for x in p:
        P *= x
    Ql = 1
    for x in q[:level]:
        Ql *= x
    mods = [slots[s] for s in ext_slots]
    M = Ql * P
    out = []
    for c in range(2):
        res = []
        for t in range(n):
            x = 0
            for si, m in enumerate(mods):
                mh = M // m
                x += acc[c][si][t] * pow(mh % m, -1, m) * mh
            x = _centre(x, M)
            r = (abs(x) + P // 2) // P  # round half away from zero (rns_math.hpp:196-202)
            res.append((r if x >= 0 else -r) % Ql)
        out.append(res)
    return out, Ql


@pytest.mark.parametrize("kind,level", [("relin", 35), ("relin", 6), ("rot", 17)])
def test_key_switch_with_secret_keys(kind, level):
    ctx = _Primes(4, 35)
    k = Ckks(ctx, seed=3, hamming=6)
    s = [int(v) for v in k.s]
    if kind == "relin":
        sp = negacyclic_int(k.s, k.s)
    else:
        sp = automorphism_int(k.s, pow(5, 3, 2 * ctx.n))
    key = k.key(sp)
    rng = np.random.default_rng(level)
    Ql = 1
    for x in k.q[:level]:
        Ql *= x
    d = [int.from_bytes(rng.bytes(256), "little") % Ql for _ in range(ctx.n)]  # uniform mod Q_l
    (c0, c1), Ql = _keyswitch(d, key, k.q, k.p, level)
    got = [(a + b) % Ql for a, b in zip(c0, _polymul(c1, s, Ql))]
    want = _polymul(d, [int(v) for v in sp], Ql)
    err = max(abs(_centre(g - w, Ql)) for g, w in zip(got, want))
    print(kind, level, "key-switch error", err)
    assert err < 2**20, err  # key-switch noise (e_j * ext_j / P plus rounding): tens, vs Q_l > 2^250
