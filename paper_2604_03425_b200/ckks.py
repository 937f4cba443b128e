"""Real CKKS encode / encrypt / decrypt and secret-derived key-switching keys
around the GPU operators (first step).

The reference idealises encryption away (graph inputs are "fresh
activations", he_ir.hpp:178-188) and its keys are opaque.  This module turns the
residue-exact GPU path into something that decrypts: a ternary secret s, keys
in the hybrid form the library's key switch expects (include/aegis.h,
aegis_keys_upload), the canonical-embedding encoder, and symmetric
encryption.  Host-side NumPy + Python integers, meant for small rings
(N <= 2^12) in tests and demos; the homomorphic operators themselves are the
library's (Context.cmult / relin / rescale / rot).

Conventions (all checked by tests/test_gpu_parity.py::test_ckks_*):
  * slot j <-> evaluation at zeta^(5^j), zeta = exp(i pi / N); Rot by r (galois
    5^r, rns_math.hpp:142-149) is a left rotation of the slot vector;
  * a ciphertext (c0, c1) decrypts as c0 + c1 s; CMult gives (c0, c1, c2)
    against (1, s, s^2); key-switching key digit j = (b_j, a_j) with
    b_j = -a_j s + e_j + F_j s' (mod Q_L P), F_j = P Qhat_j [Qhat_j^-1]_{Q_j},
    s' = s^2 (relin, id 0) or s(X^(5^r)) (rotation, id 1000 + r).
"""
import numpy as np

SPECIAL_BASE = 60  # include/aegis_params.h AEGIS_MAX_MAIN_PRIMES: ext index of P_0
ALPHA = 4          # AEGIS_SPECIAL_PRIMES: primes per key-switching digit


def _shift(a, j, mods):
    """X^j * a (negacyclic) for rows of residues a[k, N] mod mods[k]."""
    n = a.shape[1]
    r = np.empty_like(a)
    r[:, j:] = a[:, :n - j]
    r[:, :j] = (mods[:, None] - a[:, n - j:]) % mods[:, None]
    return r


def mul_small(a, t, mods):
    """a * t mod (X^N + 1, mods) for a small-integer polynomial t (|t_i| < 2^16)."""
    acc = np.zeros_like(a)
    m = mods[:, None]
    for j in np.nonzero(t)[0]:
        c = int(t[j])
        sh = _shift(a, int(j), mods)
        if c < 0:
            sh = (m - sh) % m
            c = -c
        acc = (acc + sh * np.uint64(c)) % m
    return acc


def negacyclic_int(a, b):
    """Exact product of two small integer polynomials mod X^N + 1."""
    n = len(a)
    full = np.convolve(a.astype(np.int64), b.astype(np.int64))
    out = full[:n].copy()
    out[: len(full) - n] -= full[n:]
    return out


def automorphism_int(t, k):
    """t(X^k) mod X^N + 1 for an integer polynomial t."""
    n = len(t)
    e = (np.arange(n, dtype=np.int64) * k) % (2 * n)
    out = np.zeros_like(t)
    lo = e < n
    out[e[lo]] = t[lo]
    out[e[~lo] - n] = -t[~lo]
    return out


class Ckks:
    """Secret key, key generation, encoder and symmetric encryption for `ctx`."""

    def __init__(self, ctx, seed=1, hamming=64, sigma=3.2):
        self.ctx = ctx
        self.n = ctx.n
        self.chain = ctx.chain
        self.rng = np.random.default_rng(seed)
        self.sigma = sigma
        self.q = [int(ctx.prime(i)) for i in range(self.chain)]
        self.p = [int(ctx.prime(SPECIAL_BASE + i)) for i in range(ALPHA)]
        s = np.zeros(self.n, dtype=np.int64)
        idx = self.rng.choice(self.n, size=min(hamming, self.n), replace=False)
        s[idx] = self.rng.choice([-1, 1], size=len(idx))
        self.s = s
        # canonical embedding: slot j is the evaluation at zeta^(5^j), zeta =
        # exp(i pi / N).  m(zeta^(2t+1)) = sum_k (m_k zeta^k) w^(tk), w = zeta^2,
        # is one N-point DFT, so encode / decode are O(N log N) at any N
        n, m = self.n, self.n // 2
        g = np.ones(m, dtype=np.int64)
        for j in range(1, m):
            g[j] = g[j - 1] * 5 % (2 * n)
        self.slot_t = (g - 1) // 2                  # 2t + 1 = 5^j
        self.conj_t = (2 * n - g - 1) // 2          # the conjugate root
        self.twist = np.exp(1j * np.pi * np.arange(n) / n)  # zeta^k

    # ---- encoding --------------------------------------------------------------
    def encode(self, z, scale):
        """Slot vector (N/2 complex) -> int64 coefficients of round(scale * m)."""
        z = np.asarray(z, dtype=np.complex128)
        v = np.zeros(self.n, dtype=np.complex128)
        v[self.slot_t] = z
        v[self.conj_t] = np.conj(z)
        coef = np.real(np.fft.fft(v) / self.n / self.twist)  # m_k = zeta^-k (1/N) sum_t v_t w^-tk
        return np.rint(coef * scale).astype(np.int64)

    def decode(self, coef, scale):
        """Integer (centred) coefficients -> slot vector / scale."""
        c = np.array([float(x) for x in coef])
        v = np.fft.ifft(c * self.twist) * self.n
        return v[self.slot_t] / scale

    # ---- sampling --------------------------------------------------------------
    def _error(self):
        return np.rint(self.rng.normal(0.0, self.sigma, self.n)).astype(np.int64)

    def _uniform(self, mods):
        return np.stack([self.rng.integers(0, int(p), self.n, dtype=np.uint64) for p in mods])

    @staticmethod
    def _reduce_int(t, mods):
        """Small integer polynomial (int64, |t| < 2^62) -> residues [k, N]."""
        t = np.asarray(t, dtype=np.int64)
        return np.stack([(t % np.int64(p)).astype(np.uint64) for p in mods])

    # ---- keys ------------------------------------------------------------------
    def key(self, s_prime):
        """Hybrid key-switching key from s to s_prime, library layout (coefficient domain)."""
        slots = self.q + self.p
        mods = np.array(slots, dtype=np.uint64)
        digits = -(-self.chain // ALPHA)
        Q = 1
        for x in self.q:
            Q *= x
        P = 1
        for x in self.p:
            P *= x
        out = np.zeros((digits, 2, len(slots), self.n), dtype=np.uint64)
        for j in range(digits):
            Qj = 1
            for x in self.q[ALPHA * j: ALPHA * (j + 1)]:
                Qj *= x
            qhat = Q // Qj
            F = P * qhat * pow(qhat, -1, Qj)
            a = self._uniform(slots)
            e = self._reduce_int(self._error(), slots)
            fs = self._scaled(s_prime, F, slots)
            b = (mods[:, None] - mul_small(a, self.s, mods)) % mods[:, None]
            b = (b + e) % mods[:, None]
            b = (b + fs) % mods[:, None]
            out[j, 0], out[j, 1] = b, a
        return out

    @staticmethod
    def _scaled(t, F, mods):
        """(F * t) mod each modulus for a small-integer polynomial t (|t| < 2^16), exact."""
        t = np.asarray(t, dtype=np.int64)
        if np.abs(t).max(initial=0) >= 1 << 16:
            raise ValueError("_scaled: coefficients too large")
        return np.stack([((np.int64(F % m) * t) % np.int64(m)).astype(np.uint64) for m in mods])

    def upload_relin_key(self):
        self.ctx.keys_upload(0, self.key(negacyclic_int(self.s, self.s)))

    def upload_rotation_key(self, r):
        if r <= -500:  # key ids >= 500 mark rotation keys (1000 + r, poly_ir.hpp:300-305)
            raise ValueError("rotation offset must be > -500")
        k = pow(5, r % self.n, 2 * self.n)
        self.ctx.keys_upload(1000 + r, self.key(automorphism_int(self.s, k)))

    # ---- encryption ------------------------------------------------------------
    def encrypt(self, z, scale, level, bundle=None, lane=0):
        """Symmetric encryption of slot vector z at `level` into lane `lane` of a
        (new) 2-component bundle, NTT (evaluation) domain as the library keeps it."""
        mods = np.array(self.q[:level], dtype=np.uint64)
        m = self._reduce_int(self.encode(z, scale), self.q[:level])
        a = self._uniform(self.q[:level])
        e = self._reduce_int(self._error(), self.q[:level])
        c0 = (mods[:, None] - mul_small(a, self.s, mods)) % mods[:, None]
        c0 = (c0 + e + m) % mods[:, None]
        if bundle is None:
            bundle = self.ctx.bundle(1, 2, level)
        host = bundle.download()
        host[lane, 0, :level], host[lane, 1, :level] = c0, a
        bundle.upload(host)
        self.ctx.ntt(bundle, lane=lane, lanes=1, lo=0, hi=level - 1)
        return bundle

    def secret_bundle(self, level):
        """The secret s as a 1-component NTT-domain bundle (cached per level): the
        GPU-side encryption / decryption multiply by it with aegis_limb_op."""
        cache = self.__dict__.setdefault("_s_dev", {})
        if level not in cache:
            b = self.ctx.bundle(1, 1, level)
            b.upload(self._reduce_int(self.s, self.q[:level]).reshape(1, 1, level, self.n))
            self.ctx.ntt(b)
            cache[level] = b
        return cache[level]

    def encrypt_gpu(self, z, scale, level):
        """The same symmetric encryption with the ring arithmetic on the GPU: the
        host only samples (a uniform, e Gaussian) and encodes m; a * s, the sum and
        the NTTs run as library kernels (aegis_ntt, aegis_limb_op)."""
        from . import _lib as L
        c = self.ctx
        a = self._uniform(self.q[:level])
        em = self._reduce_int(self.encode(z, scale) + self._error(), self.q[:level])
        ct = c.bundle(1, 2, level)
        host = np.zeros((1, 2, level, self.n), dtype=np.uint64)
        host[0, 0], host[0, 1] = em, a
        ct.upload(host)
        c.ntt(ct)  # both components to the evaluation domain
        a_pt = c.bundle(1, 1, level)  # component 1 (a) as a plaintext operand
        a_pt.upload(host[:, 1:2])
        c.ntt(a_pt)
        prod = c.bundle(1, 1, level)
        c.limb_op(L.LIMB_MUL, prod, a_pt, self.secret_bundle(level))  # a * s
        c.limb_op(L.LIMB_SUB, ct, ct, prod, lanes=1)  # c0 = (e + m) - a s (plaintext b feeds comp 0)
        a_pt.free()
        prod.free()
        return ct

    def decrypt_gpu(self, bundle, scale, level, lane=0):
        """c0 + c1 s and the inverse NTT on the GPU; CRT + decoding on the host."""
        from . import _lib as L
        c = self.ctx
        m = c.bundle(1, 1, level)
        c1 = c.bundle(1, 1, level)
        h = bundle.download()[lane: lane + 1, :2, :level]
        c1.upload(np.ascontiguousarray(h[:, 1:2]))
        c0 = c.bundle(1, 1, level)
        c0.upload(np.ascontiguousarray(h[:, 0:1]))
        c.limb_op(L.LIMB_MUL, m, c1, self.secret_bundle(level))
        c.limb_op(L.LIMB_ADD, m, m, c0)
        c.ntt(m, inverse=True)
        x = m.download()[0, 0]
        for b in (m, c1, c0):
            b.free()
        return self.decode(self.crt(x, level), scale)

    def decrypt(self, bundle, scale, level, lane=0):
        """Slot vector of lane `lane` (first two components, `level` limbs)."""
        tmp = self.ctx.bundle(1, bundle.comps, bundle.level)
        host = bundle.download()
        tmp.upload(host[lane: lane + 1])
        self.ctx.ntt(tmp, lanes=1, lo=0, hi=level - 1, inverse=True)
        h = tmp.download()
        tmp.free()
        mods = np.array(self.q[:level], dtype=np.uint64)
        c0 = h[0, 0, :level] % mods[:, None]
        c1 = h[0, 1, :level] % mods[:, None]
        x = (c0 + mul_small(c1, self.s, mods)) % mods[:, None]
        return self.decode(self.crt(x, level), scale)

    def crt(self, x, level):
        """Residues [level, N] -> centred integers (Python ints, object array)."""
        q = self.q[:level]
        Q = 1
        for v in q:
            Q *= v
        acc = np.zeros(self.n, dtype=object)
        for i, v in enumerate(q):
            qh = Q // v
            inv = pow(qh % v, -1, v)
            acc = acc + (x[i].astype(object) * inv % v) * qh
        acc = acc % Q
        return np.where(acc > Q // 2, acc - Q, acc)
