"""Real GELU / exp / inverse-sqrt on real CKKS ciphertexts (
paper_2604_03425_b200/nonlinear.py): polynomial approximations evaluated with
the library's GPU operators, decrypted and compared with NumPy.  The CPU part
checks the approximations themselves."""
import math

import numpy as np
import pytest

from paper_2604_03425_b200.nonlinear import power_coeffs


def _gelu(t):
    return 0.5 * t * (1.0 + np.vectorize(math.erf)(t / math.sqrt(2.0)))


def test_approximations_on_their_intervals():
    u = np.linspace(-1, 1, 2001)
    for f, lo, hi, deg, tol in ((_gelu, -4.0, 4.0, 16, 2e-3), (lambda t: np.exp(t / 4), -8.0, 0.0, 12, 1e-9),
                                (lambda t: 1 / np.sqrt(t), 0.25, 4.0, 6, 5e-2)):
        c = power_coeffs(f, lo, hi, deg)
        x = 0.5 * (hi - lo) * u + 0.5 * (hi + lo)
        assert np.abs(np.polynomial.polynomial.polyval(u, c) - f(x)).max() < tol


@pytest.fixture(scope="module")
def env():
    from paper_2604_03425_b200 import Context
    from paper_2604_03425_b200.boot import Bootstrapper
    from paper_2604_03425_b200.ckks import Ckks
    from paper_2604_03425_b200.nonlinear import Nonlinear
    c = Context(log_n=10)
    k = Ckks(c, seed=7, hamming=64)
    k.upload_relin_key()
    bs = Bootstrapper(c, k)
    yield c, k, bs, Nonlinear(bs)
    bs.close()


def _run(env, fn, lo, hi, ref, level=30):
    from paper_2604_03425_b200.boot import Ct
    c, k, bs, nl = env
    rng = np.random.default_rng(3)
    x = rng.uniform(lo, hi, c.n // 2)
    scale = 2.0 ** 40
    ct = Ct(k.encrypt(x, scale, level), level, scale)
    out = fn(nl, ct)
    got = k.decrypt(out.b, out.scale, out.level).real
    err = np.abs(got - ref(x)).max()
    ct.free()
    out.free()
    return err, out.level


@pytest.mark.gpu
def test_gelu_on_ciphertexts(env):
    err, lv = _run(env, lambda nl, ct: nl.gelu(ct), -4.0, 4.0, _gelu)
    print(f"gelu: max error {err:.2e}, output level {lv}")
    assert err < 3e-3


@pytest.mark.gpu
def test_exp_on_ciphertexts(env):
    err, lv = _run(env, lambda nl, ct: nl.exp(ct), -8.0, 0.0, np.exp)
    print(f"exp: max error {err:.2e}, output level {lv}")
    assert err < 1e-4


@pytest.mark.gpu
def test_inv_sqrt_on_ciphertexts(env):
    err, lv = _run(env, lambda nl, ct: nl.inv_sqrt(ct), 0.25, 4.0, lambda t: 1 / np.sqrt(t))
    print(f"inv_sqrt: max error {err:.2e}, output level {lv}")
    assert err < 1e-3


@pytest.mark.gpu
def test_gpu_side_encrypt_decrypt(env):
    """encrypt_gpu / decrypt_gpu (ring arithmetic in library kernels) agree with the
    host-side forms: decrypting either way recovers the message, and a GPU
    encryption rotates and multiplies like a host one."""
    c, k, bs, nl = env
    rng = np.random.default_rng(9)
    z = rng.uniform(-1, 1, c.n // 2) + 1j * rng.uniform(-1, 1, c.n // 2)
    scale, level = 2.0 ** 40, 12
    ct = k.encrypt_gpu(z, scale, level)
    assert np.abs(k.decrypt(ct, scale, level) - z).max() < 1e-6
    assert np.abs(k.decrypt_gpu(ct, scale, level) - z).max() < 1e-6
    ct2 = k.encrypt(z, scale, level)
    assert np.abs(k.decrypt_gpu(ct2, scale, level) - z).max() < 1e-6
    for b in (ct, ct2):
        b.free()


@pytest.mark.gpu
def test_encrypted_mlp_block_with_bootstrap():
    """A real encrypted MLP block end to end on the GPU operators, against NumPy
    float64: y = W2 . bootstrap(gelu(W1 . x)).  W1, W2 are dense 512 x 512
    matrices applied by BSGS over the slot diagonals, GELU is the degree-16
    approximation, and the ciphertext is refreshed by real bootstrapping
    (level 1 -> 21) before the second matmul."""
    from paper_2604_03425_b200 import Context
    from paper_2604_03425_b200.boot import Bootstrapper, Ct
    from paper_2604_03425_b200.ckks import Ckks
    from paper_2604_03425_b200.nonlinear import Nonlinear
    c = Context(log_n=10)
    k = Ckks(c, seed=13, hamming=64)
    bs = Bootstrapper(c, k)
    bs.upload_keys()
    nl = Nonlinear(bs)
    n = c.n // 2
    rng = np.random.default_rng(21)
    x = rng.uniform(-1, 1, n)
    W1 = rng.uniform(-1, 1, (n, n)) * (2.0 / np.sqrt(n))
    W2 = rng.uniform(-1, 1, (n, n)) * (1.0 / np.sqrt(n))
    want = W2 @ _gelu(W1 @ x)
    scale = 2.0 ** 40
    ct = Ct(k.encrypt(x, scale, 35), 35, scale)
    h1 = bs.linear(ct, W1)                    # level 34
    assert np.abs(W1 @ x).max() < 4.0         # inside GELU's approximation interval
    g = nl.gelu(h1)
    low = bs.mul_const(g, 1.0, 2.0 ** 34)     # same values at scale 2^34: q_0 / (Delta |m|) >= 2^10
    one = bs.drop(low, 1)
    fresh = bs.bootstrap(one.b, 2.0 ** 34)    # level 21
    y = bs.linear(fresh, W2)
    got = k.decrypt(y.b, y.scale, y.level).real
    err = np.abs(got - want).max()
    print(f"encrypted MLP block (matmul, GELU, bootstrap, matmul): max error {err:.2e}, "
          f"|y| <= {np.abs(want).max():.2f}, output level {y.level}")
    assert err < 2e-2
    for t in (ct, h1, g, low, one, fresh, y):
        t.free()
    bs.close()
