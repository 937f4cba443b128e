"""Real polynomial approximations of the Transformer nonlinearities on CKKS
ciphertexts.

The reference replays stand-in squaring chains for GELU, softmax's exp and
LayerNorm's inverse square root (he_ir.hpp:305-322, 477-599: `depth` CMult +
Relin + Rescale steps with no coefficients); the executor reproduces those
bit-exactly.  This module evaluates the real functions on real encryptions,
with the same library operators (every polynomial operation on the GPU):

  gelu(x)      x * Phi(x): Chebyshev interpolant of degree `deg` on [-a, a]
  exp(x)       Chebyshev interpolant on [lo, 0] (softmax inputs after the max
               shift), optionally refined by squaring: exp(x) = exp(x/2^k)^(2^k)
  inv_sqrt(x)  1/sqrt(x) on [lo, hi]: a low-degree Chebyshev start refined by
               Newton steps y <- y (3 - x y^2) / 2

Evaluation: the interval is mapped affinely onto [-1, 1] (one constant
multiply), the power basis u^1 .. u^d is built by binary products (depth
ceil(log2 d)), and every term c_k u^k is brought to one target scale by the
encoding scale of its coefficient (Bootstrapper.mul_const), so ciphertexts of
different scales are never added.  Coefficients come from NumPy's Chebyshev
interpolation converted to the power basis on [-1, 1] (degree <= 16 keeps the
power-basis coefficients small enough for 2^42 scales).
"""
import math

import numpy as np
from numpy.polynomial import chebyshev as C

from .boot import Bootstrapper, Ct


def power_coeffs(f, lo, hi, deg):
    """Power-basis coefficients of the degree-`deg` Chebyshev interpolant of f
    on [lo, hi], in the variable u = (2x - lo - hi) / (hi - lo) in [-1, 1]."""
    k = np.arange(deg + 1)
    u = np.cos(np.pi * (k + 0.5) / (deg + 1))
    x = 0.5 * (hi - lo) * u + 0.5 * (hi + lo)
    cheb = C.chebfit(u, f(x), deg)
    return C.cheb2poly(cheb)


class Nonlinear:
    """Polynomial evaluation on ciphertexts through a Bootstrapper's operators
    (only its ciphertext arithmetic is used: relin key + no rotations)."""

    def __init__(self, bs: Bootstrapper, scale=2.0 ** 42):
        self.bs, self.scale = bs, scale

    def poly(self, x: Ct, coeffs, lo, hi):
        """sum_k coeffs[k] u^k with u = (2x - lo - hi) / (hi - lo); returns a Ct."""
        bs = self.bs
        a, b = 2.0 / (hi - lo), -(hi + lo) / (hi - lo)
        u0 = bs.mul_const(x, a, self.scale)
        u = bs.add_const(u0, b)
        u0.free()
        d = len(coeffs) - 1
        pw = {1: u}
        k = 1
        while 2 * k <= d:
            pw[2 * k] = bs.mul(pw[k], pw[k])
            k *= 2
        for e in range(2, d + 1):
            if e in pw:
                continue
            hi_ = 1 << (e.bit_length() - 1)
            pw[e] = bs.mul(pw[hi_], pw[e - hi_])
        tgt_level = min(p.level for p in pw.values()) - 1
        acc = None
        for e in range(1, d + 1):
            if coeffs[e] == 0:
                continue
            ye = bs.drop(pw[e], tgt_level + 1)
            term = bs.mul_const(ye, float(coeffs[e]), self.scale)
            if ye is not pw[e]:
                ye.free()
            if acc is None:
                acc = term
            else:
                s = bs.add(acc, term)
                acc.free()
                term.free()
                acc = s
        for p in pw.values():
            p.free()
        out = bs.add_const(acc, float(coeffs[0]))
        acc.free()
        return out

    # ---- the Transformer nonlinearities -----------------------------------------
    def gelu(self, x: Ct, a=4.0, deg=16):
        f = lambda t: 0.5 * t * (1.0 + np.vectorize(math.erf)(t / math.sqrt(2.0)))  # noqa: E731
        return self.poly(x, power_coeffs(f, -a, a, deg), -a, a)

    def exp(self, x: Ct, lo=-8.0, deg=12, squarings=2):
        """exp on [lo, 0]: exp(x / 2^k) by a polynomial, then k squarings."""
        s = 2 ** squarings
        c = power_coeffs(lambda t: np.exp(t / s), lo, 0.0, deg)
        y = self.poly(x, c, lo, 0.0)
        for _ in range(squarings):
            y2 = self.bs.mul(y, y)
            y.free()
            y = y2
        return y

    def inv_sqrt(self, x: Ct, lo=0.25, hi=4.0, deg=6, newton=2):
        """1/sqrt(x) on [lo, hi]: Chebyshev start, then Newton y <- y (3 - x y^2) / 2."""
        bs = self.bs
        y = self.poly(x, power_coeffs(lambda t: 1.0 / np.sqrt(t), lo, hi, deg), lo, hi)
        for _ in range(newton):
            y2 = bs.mul(y, y)                              # y^2
            xd = bs.drop(x, y2.level) if x.level > y2.level else x
            xy2 = bs.mul(xd, y2)                           # x y^2
            if xd is not x:
                xd.free()
            y2.free()
            t = bs.mul_const(xy2, -0.5, self.scale)        # -x y^2 / 2
            xy2.free()
            t2 = bs.add_const(t, 1.5)                      # (3 - x y^2) / 2
            t.free()
            yn = bs.mul(y, t2)
            y.free()
            t2.free()
            y = yn
        return y
