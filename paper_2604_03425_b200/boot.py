"""Real CKKS bootstrapping on the GPU operators.

The reference lowers Boot to a value-preserving lift (PolyMode::kBootReset,
poly_ir.hpp:355-368; he_ir.hpp:601-613) -- the executor's
aegis_boot reproduces that bit-exactly.  This module is the real thing, built
only from library operators so every polynomial operation runs on the GPU:

  ModRaise     aegis_boot from level 1 (the exact centred lift of each residue
               mod q_0 to q_1 .. q_{L-1}): the ciphertext now decrypts to
               t = Delta m + e + q_0 I over the integers, I small
  CoeffToSlot  slots <- (t_k + i t_{k+n}) / q_0: the inverse of the encoding
               matrix A (z_j = sum_k u_k zeta^(5^j k), u = t_lo + i t_hi),
               baby-step giant-step (n1 x n2 diagonals, n1 + n2 - 2 rotation
               keys), one rescale
  split        real / imaginary parts with the conjugation automorphism
               (galois 2N - 1, keyswitch with key id 2) and the exact
               monomial X^(N/2) (multiplication by i in every slot)
  EvalMod      sin(2 pi x) = cos(2 pi (x - 1/4)): theta = 2 pi (x - 1/4) / 2^r,
               cos(theta) by its Taylor series in y = theta^2 (power basis, every
               term brought to one scale by its coefficient's encoding scale),
               then r double angles cos(2a) = 2 cos(a)^2 - 1
  SlotToCoeff  the encoding matrix A (same BSGS), one rescale; the 1/(2 pi)
               and q_0 / Delta factors are folded into the declared scale

Every ciphertext carries its exact scale (a float); a constant or diagonal is
encoded at whatever scale makes the product land where it must, so no two
ciphertexts of different scales are ever added.  Levels: 35 after ModRaise,
21 at the end (= the reference's post_boot_level, ckks.hpp:32, with l_boot 14).
Host-side work is only encoding (NumPy FFT) and bookkeeping.
"""
import numpy as np

from . import _lib as L
from .ckks import Ckks, automorphism_int

CONJ_KEY = 2  # key id of the conjugation key (s(X^-1) -> s); ids < 500 are not pre-permuted


def encoding_matrix(N):
    """A[j, k] = zeta^((2 t_j + 1) k), zeta = exp(i pi / N), 2 t_j + 1 = 5^j mod 2N:
    slot j of a plaintext with coefficients t equals (A @ (t[:N/2] + 1j * t[N/2:]))[j]
    (zeta^(5^j N/2) = i because 5^j = 1 mod 4)."""
    n = N // 2
    g = np.ones(n, dtype=np.int64)
    for j in range(1, n):
        g[j] = g[j - 1] * 5 % (2 * N)
    e = np.outer(g, np.arange(n)) % (2 * N)
    return np.exp(1j * np.pi * e / N)


class Ct:
    """A ciphertext bundle lane with its level and exact (declared) scale."""

    def __init__(self, bundle, level, scale):
        self.b, self.level, self.scale = bundle, level, float(scale)

    def free(self):
        if self.b is not None:
            self.b.free()
            self.b = None


class Bootstrapper:
    def __init__(self, ctx, ckks: Ckks, n1=None, r=6, taylor_terms=8, top_level=None):
        self.c, self.k = ctx, ckks
        self.N, self.n = ctx.n, ctx.n // 2
        self.r, self.terms = r, taylor_terms
        self.top = top_level or ctx.chain
        n = self.n
        self.n1 = n1 or int(2 ** np.ceil(np.log2(np.sqrt(n))))
        self.n2 = n // self.n1
        self.A = encoding_matrix(self.N)
        self.Ainv = np.linalg.inv(self.A)
        self.q = ckks.q
        self._pt = {}

    # ---- keys ------------------------------------------------------------------
    def rotations(self):
        return sorted(set(list(range(1, self.n1)) + [g * self.n1 for g in range(1, self.n2)]))

    def upload_keys(self):
        k = self.k
        k.upload_relin_key()
        for r in self.rotations():
            k.upload_rotation_key(r)
        self.c.keys_upload(CONJ_KEY, k.key(automorphism_int(k.s, 2 * self.N - 1)))

    # ---- plaintexts ------------------------------------------------------------
    def _upload_poly(self, coef, level):
        """Integer coefficients -> 1-component NTT-domain bundle at `level`."""
        res = Ckks._reduce_int(coef, self.q[:level])
        pt = self.c.bundle(1, 1, level)
        pt.upload(res.reshape(1, 1, level, self.N))
        self.c.ntt(pt)
        return pt

    def pt_slots(self, z, scale, level):
        return self._upload_poly(self.k.encode(z, scale), level)

    def pt_const(self, v, scale, level):
        coef = np.zeros(self.N, dtype=np.int64)
        coef[0] = int(np.rint(v * scale))
        return self._upload_poly(coef, level)

    def pt_monomial(self, j, sign, level):
        key = ("mono", j, sign, level)
        if key not in self._pt:
            coef = np.zeros(self.N, dtype=np.int64)
            coef[j] = sign
            self._pt[key] = self._upload_poly(coef, level)
        return self._pt[key]

    # ---- ciphertext operators (all on the GPU) ---------------------------------
    def new(self, level, comps=2):
        return self.c.bundle(1, comps, level)

    def add(self, a, b, sub=False):
        assert a.level == b.level and abs(a.scale / b.scale - 1) < 1e-12, "scale / level mismatch"
        out = self.new(a.level)
        self.c.limb_op(L.LIMB_SUB if sub else L.LIMB_ADD, out, a.b, b.b, lo=0, hi=a.level - 1)
        return Ct(out, a.level, a.scale)

    def add_const(self, a, v):
        out = self.new(a.level)
        pt = self.pt_const(v, a.scale, a.level)
        self.c.padd(out, a.b, pt, a.level)
        pt.free()
        return Ct(out, a.level, a.scale)

    def drop(self, a, level):
        if level == a.level:
            return a
        cur = a.b
        for lv in range(a.level, level, -1):
            nxt = self.new(lv - 1)
            self.c.limb_drop(nxt, cur, lv, mode=L.MODE_NONE)
            if cur is not a.b:
                cur.free()
            cur = nxt
        return Ct(cur, level, a.scale)

    def rescale(self, a):
        out = self.new(a.level - 1)
        self.c.rescale(out, a.b, a.level)
        return Ct(out, a.level - 1, a.scale / self.q[a.level - 1])

    def mul(self, a, b):
        """CMult + Relin + Rescale at the lower of the two levels."""
        lv = min(a.level, b.level)
        a2, b2 = self.drop(a, lv), self.drop(b, lv)
        prod = self.new(lv, comps=3)
        self.c.cmult(prod, a2.b, b2.b, lv)
        self.c.relin(prod, lv)
        out = self.new(lv - 1)
        self.c.rescale(out, prod, lv)
        prod.free()
        for x, y in ((a2, a), (b2, b)):
            if x is not y:
                x.free()
        return Ct(out, lv - 1, a.scale * b.scale / self.q[lv - 1])

    def mul_const(self, a, v, target_scale):
        """a * v (real constant), rescaled, landing exactly on target_scale."""
        lv = a.level
        enc = target_scale * self.q[lv - 1] / a.scale
        pt = self.pt_const(v, enc, lv)
        prod = self.new(lv)
        self.c.limb_op(L.LIMB_MUL, prod, a.b, pt, lo=0, hi=lv - 1)
        pt.free()
        out = self.new(lv - 1)
        self.c.rescale(out, prod, lv)
        prod.free()
        # the plaintext is round(v * enc) at scale enc: the product's scale is exactly
        # a.scale * enc / q = target (the rounding only perturbs the value, by <= 0.5 / enc)
        return Ct(out, lv - 1, target_scale)

    def mul_i(self, a, sign=1):
        """Every slot times sign * i: the monomial sign * X^(N/2), exact, no level."""
        out = self.new(a.level)
        self.c.limb_op(L.LIMB_MUL, out, a.b, self.pt_monomial(self.N // 2, sign, a.level), lo=0, hi=a.level - 1)
        return Ct(out, a.level, a.scale)

    def rot(self, a, r):
        if r % self.n == 0:  # a copy (the BSGS giant step 0)
            out = self.new(a.level)
            self.c.cadd(out, a.b, self._zero(a.level), a.level)
            return Ct(out, a.level, a.scale)
        out = self.new(a.level)
        self.c.rot(out, a.b, r, a.level)
        return Ct(out, a.level, a.scale)

    def _zero(self, level):
        key = ("zero", level)
        if key not in self._pt:
            z = self.c.bundle(1, 2, level)
            z.upload(np.zeros((1, 2, level, self.N), dtype=np.uint64))
            self._pt[key] = z
        return self._pt[key]

    def conj(self, a):
        """Slot-wise complex conjugate: automorphism X -> X^(2N-1), then keyswitch s(X^-1) -> s."""
        lv = a.level
        t = self.new(lv)
        self.c.automorphism(t, a.b, 2 * self.N - 1, level=lv)
        ks = self.new(lv)
        self.c.keyswitch(ks, t, 1, lv, CONJ_KEY)
        h = t.download()
        c0 = self.c.bundle(1, 1, lv)
        c0.upload(np.ascontiguousarray(h[:, :1]))
        out = self.new(lv)
        self.c.padd(out, ks, c0, lv)
        for x in (t, ks, c0):
            x.free()
        return Ct(out, lv, a.scale)

    def linear(self, a, M):
        """Slots <- M @ slots (BSGS over the n diagonals), one rescale."""
        n, n1, n2, lv = self.n, self.n1, self.n2, a.level
        enc = self.q[lv - 1]  # diagonals at the dropped prime: the scale survives the rescale
        baby = [a if b == 0 else self.rot(a, b) for b in range(n1)]
        acc = None
        j = np.arange(n)
        for g in range(n2):
            inner = self.new(lv)
            inner.upload(np.zeros((1, 2, lv, self.N), dtype=np.uint64))
            for b in range(n1):
                d = g * n1 + b
                diag = M[j, (j + d) % n]
                pt = self.pt_slots(np.roll(diag, g * n1), enc, lv)  # rot_{-g n1}(diag)
                self.c.limb_op(L.LIMB_MULACC, inner, baby[b].b, pt, lo=0, hi=lv - 1)
                pt.free()
            term = self.rot(Ct(inner, lv, a.scale * enc), g * n1)
            inner.free()
            if acc is None:
                acc = term
            else:
                s = self.add(acc, term)
                acc.free()
                term.free()
                acc = s
        for b in range(1, n1):
            baby[b].free()
        out = self.rescale(acc)
        acc.free()
        return out

    # ---- EvalMod ------------------------------------------------------------------
    def eval_mod(self, x, half):
        """sin(2 pi x') for the slots x' = half * x (real), via cos + r double angles."""
        r = self.r
        # theta = 2 pi (x' - 1/4) / 2^r
        a = 2 * np.pi * half / 2 ** r
        th = self.mul_const(x, a, 2.0 ** 42)
        th2 = self.add_const(th, -2 * np.pi * 0.25 / 2 ** r)
        th.free()
        # powers of y = theta^2
        pw = {1: self.mul(th2, th2)}
        th2.free()
        k = 1
        while 2 * k < self.terms:
            pw[2 * k] = self.mul(pw[k], pw[k])
            k *= 2
        for e in range(2, self.terms):
            if e in pw:
                continue
            hi = 1 << (e.bit_length() - 1)
            pw[e] = self.mul(pw[hi], pw[e - hi])
        # cos(theta) = sum_k (-1)^k y^k / (2k)!, every term at one scale
        tgt_level = min(p.level for p in pw.values()) - 1
        tgt_scale = 2.0 ** 42
        acc = None
        fact = 1.0
        for e in range(1, self.terms):
            fact *= (2 * e - 1) * (2 * e)
            ye = self.drop(pw[e], tgt_level + 1)
            term = self.mul_const(ye, (-1) ** e / fact, tgt_scale)
            if ye is not pw[e]:
                ye.free()
            if acc is None:
                acc = term
            else:
                s = self.add(acc, term)
                acc.free()
                term.free()
                acc = s
        for p in pw.values():
            p.free()
        c = self.add_const(acc, 1.0)
        acc.free()
        # r double angles: cos(2a) = 2 cos(a)^2 - 1
        for _ in range(r):
            sq = self.mul(c, c)
            c.free()
            two = self.add(sq, sq)
            sq.free()
            c = self.add_const(two, -1.0)
            two.free()
        return c  # ~ sin(2 pi x')

    # ---- the whole bootstrap ----------------------------------------------------------
    def bootstrap(self, ct, delta):
        """ct: level-1 ciphertext of slots m at scale delta (delta |m| << q_0).
        Returns a Ct at level top - 14 whose declared scale decrypts to m."""
        q0 = self.q[0]
        raised = self.new(self.top)
        self.c.boot(raised, ct, 1, self.top)  # ModRaise: exact centred lift of every residue mod q_0
        x = Ct(raised, self.top, q0)          # slots = t / q_0 (declared scale q_0)
        u = self.linear(x, self.Ainv)         # slots = (t_lo + i t_hi) / q_0
        x.free()
        uc = self.conj(u)
        re2 = self.add(u, uc)                 # 2 t_lo / q_0
        im2i = self.add(u, uc, sub=True)      # 2 i t_hi / q_0
        u.free()
        uc.free()
        im2 = self.mul_i(im2i, sign=-1)       # 2 t_hi / q_0
        im2i.free()
        s_re = self.eval_mod(re2, 0.5)
        s_im = self.eval_mod(im2, 0.5)
        re2.free()
        im2.free()
        s_im_i = self.mul_i(s_im)
        s_im.free()
        v = self.add(s_re, s_im_i)            # ~ 2 pi (t mod q_0) / q_0, complex packed
        s_re.free()
        s_im_i.free()
        out = self.linear(v, self.A)          # slots ~ 2 pi (Delta m + e) / q_0
        v.free()
        out.scale = out.scale * 2 * np.pi * delta / q0
        return out

    def close(self):
        for p in self._pt.values():
            p.free()
        self._pt = {}
