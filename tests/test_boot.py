"""Real CKKS bootstrapping (paper_2604_03425_b200/boot.py).
CPU: the encoding matrix the homomorphic CoeffToSlot / SlotToCoeff use is the
canonical embedding of the encoder.  GPU: a level-1 ciphertext is bootstrapped
with library operators only (ModRaise = aegis_boot from level 1, BSGS linear
transforms, conjugation, EvalMod) and decrypts to the original message."""
import numpy as np
import pytest


@pytest.mark.parametrize("log_n", [4, 6, 10])
def test_encoding_matrix_is_the_canonical_embedding(log_n):
    from paper_2604_03425_b200.boot import encoding_matrix
    N = 1 << log_n
    n = N // 2
    rng = np.random.default_rng(log_n)
    t = rng.integers(-1000, 1000, N)
    g = [pow(5, j, 2 * N) for j in range(n)]
    zeta = np.exp(1j * np.pi / N)
    direct = np.array([sum(t[k] * zeta ** ((gj * k) % (2 * N)) for k in range(N)) for gj in g])
    A = encoding_matrix(N)
    assert np.allclose(A @ (t[:n] + 1j * t[n:]), direct, atol=1e-6 * N * 1000)


@pytest.mark.gpu
def test_bootstrap_decrypts_to_the_message():
    from paper_2604_03425_b200 import Context
    from paper_2604_03425_b200.boot import Bootstrapper
    from paper_2604_03425_b200.ckks import Ckks
    c = Context(log_n=10)
    k = Ckks(c, seed=5, hamming=64)
    bs = Bootstrapper(c, k)
    bs.upload_keys()
    rng = np.random.default_rng(1)
    z = rng.uniform(-1, 1, c.n // 2) + 1j * rng.uniform(-1, 1, c.n // 2)
    delta = 2.0 ** 36
    ct = k.encrypt(z, delta, 1)
    assert np.abs(k.decrypt(ct, delta, 1) - z).max() < 1e-6
    out = bs.bootstrap(ct, delta)
    assert out.level == 21  # = post_boot_level (ckks.hpp:32): L - l_boot = 35 - 14
    got = k.decrypt(out.b, out.scale, out.level)
    err = np.abs(got - z).max()
    print(f"bootstrap: max |error| {err:.2e} over {len(z)} slots")
    assert err < 1e-3
    # the refreshed ciphertext computes: one more multiplication at the new level
    sq = bs.mul(out, out)
    e2 = np.abs(k.decrypt(sq.b, sq.scale, sq.level) - z * z).max()
    assert e2 < 4e-3
    for x in (out, sq):
        x.free()
    bs.close()
