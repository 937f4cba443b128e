"""ctypes wrapper of oracle/liboracle.so -- the CPU CHECKER (test infrastructure).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
"""
import ctypes
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libheplan_ref.so")

u64p = ctypes.POINTER(ctypes.c_uint64)
u32p = ctypes.POINTER(ctypes.c_uint32)
vp = ctypes.c_void_p

_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(ORACLE_SO)
        sig = {
            "orc_create": (vp, [ctypes.c_uint32] * 3 + [ctypes.c_uint64] * 3 + [ctypes.c_int]),
            "orc_destroy": (None, [vp]),
            "orc_prime": (ctypes.c_uint64, [vp, ctypes.c_uint32]),
            "orc_psi": (ctypes.c_uint64, [vp, ctypes.c_uint32]),
            "orc_mix64": (ctypes.c_uint64, [ctypes.c_uint64]),
            "orc_row_key": (ctypes.c_uint64, [ctypes.c_uint64] * 6),
            "orc_fill_uniform": (None, [ctypes.c_uint64, ctypes.c_uint64, u64p, ctypes.c_uint32]),
            "orc_ntt": (ctypes.c_int, [vp, u64p, u32p, ctypes.c_uint32, ctypes.c_int]),
            "orc_automorphism_eval": (ctypes.c_int, [vp, u64p, u64p, ctypes.c_uint32, ctypes.c_uint64]),
            "orc_automorphism_coeff": (ctypes.c_int, [vp, u64p, u64p, ctypes.c_uint64, ctypes.c_uint64]),
            "orc_ntt_prime": (ctypes.c_int, [vp, u64p, ctypes.c_uint64, ctypes.c_int]),
            "orc_galois": (ctypes.c_uint64, [ctypes.c_int, ctypes.c_uint32]),
            "orc_basis_convert": (ctypes.c_int64, [vp, u64p, u32p, ctypes.c_uint32, u64p, u32p, ctypes.c_uint32]),
            "orc_basis_convert_bigint": (ctypes.c_int, [vp, u64p, u32p, ctypes.c_uint32, u64p, u32p,
                                                        ctypes.c_uint32]),
            "orc_keyswitch": (ctypes.c_int, [vp, u64p, ctypes.c_uint32, ctypes.c_uint64, u64p, u64p]),
            "orc_rotate": (ctypes.c_int, [vp, u64p, ctypes.c_uint32, ctypes.c_int, u64p]),
            "orc_relin": (ctypes.c_int, [vp, u64p, ctypes.c_uint32, u64p]),
            "orc_rescale": (ctypes.c_int, [vp, u64p, ctypes.c_uint32, u64p]),
            "orc_boot_reset": (ctypes.c_int, [vp, u64p, ctypes.c_uint32, ctypes.c_uint32, u64p]),
            "orc_cmult": (ctypes.c_int, [vp, u64p, u64p, ctypes.c_uint32, u64p]),
            "orc_key_limb": (None, [vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, u64p]),
            "orc_weight_limb": (None, [vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, u64p]),
            "orc_input_limb": (None, [vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, u64p]),
            "orc_run_graph": (ctypes.c_int64, [vp, ctypes.c_char_p, ctypes.c_int64, u64p, ctypes.c_uint64]),
            "orc_run_graph_tg": (ctypes.c_int64, [vp, ctypes.c_char_p, ctypes.c_int64, u64p, ctypes.c_uint64,
                                                 ctypes.c_uint32, ctypes.c_int32]),
            "orc_hash_bundle_data": (ctypes.c_uint64, [u64p] + [ctypes.c_uint32] * 6),
            "orc_last_error": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def P(a):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(u64p)


def U(xs):
    a = np.ascontiguousarray(np.asarray(xs, dtype=np.uint32))
    return a, a.ctypes.data_as(u32p)


class Oracle:
    """CPU oracle context (same parameters and seeds as an aegis Context)."""

    def __init__(self, log_n, chain=35, lboot=14, seed_input=0xAE615, seed_weight=0xAE616,
                 seed_key=0xAE617, threads=0):
        self.L = lib()
        self.h = self.L.orc_create(log_n, chain, lboot, seed_input, seed_weight, seed_key, threads)
        if not self.h:
            raise ValueError(self.L.orc_last_error().decode())
        self.n = 1 << log_n
        self.log_n = log_n

    def __del__(self):
        try:
            self.L.orc_destroy(self.h)
        except Exception:
            pass

    def _chk(self, rc):
        if rc < 0:
            raise RuntimeError(self.L.orc_last_error().decode())
        return rc

    def prime(self, e):
        return self.L.orc_prime(self.h, e)

    def psi(self, e):
        return self.L.orc_psi(self.h, e)

    def ntt(self, data, ext, inverse=False):
        a = np.ascontiguousarray(data, dtype=np.uint64).copy()
        e, pe = U(ext)
        self._chk(self.L.orc_ntt(self.h, P(a), pe, len(e), 1 if inverse else 0))
        return a

    def automorphism_eval(self, data, k):
        a = np.ascontiguousarray(data, dtype=np.uint64)
        out = np.empty_like(a)
        self.L.orc_automorphism_eval(self.h, P(a), P(out), a.size // self.n, k)
        return out

    def automorphism_coeff(self, data, p, k):
        a = np.ascontiguousarray(data, dtype=np.uint64)
        out = np.empty_like(a)
        self.L.orc_automorphism_coeff(self.h, P(a), P(out), p, k)
        return out

    def ntt_prime(self, data, p, inverse=False):
        a = np.ascontiguousarray(data, dtype=np.uint64).copy()
        self._chk(self.L.orc_ntt_prime(self.h, P(a), p, 1 if inverse else 0))
        return a

    def basis_convert(self, data, src, dst, bigint=False):
        a = np.ascontiguousarray(data, dtype=np.uint64)
        out = np.zeros((len(dst), self.n), dtype=np.uint64)
        s, ps = U(src)
        d, pd = U(dst)
        if bigint:
            self._chk(self.L.orc_basis_convert_bigint(self.h, P(a), ps, len(s), P(out), pd, len(d)))
            return out, 0
        fb = self._chk(self.L.orc_basis_convert(self.h, P(a), ps, len(s), P(out), pd, len(d)))
        return out, fb

    def keyswitch(self, d, level, key_id):
        a = np.ascontiguousarray(d, dtype=np.uint64)
        o0 = np.empty((level, self.n), dtype=np.uint64)
        o1 = np.empty_like(o0)
        self._chk(self.L.orc_keyswitch(self.h, P(a), level, key_id, P(o0), P(o1)))
        return o0, o1

    def rotate(self, ct, level, offset):
        a = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.empty((2, level, self.n), dtype=np.uint64)
        self._chk(self.L.orc_rotate(self.h, P(a), level, offset, P(out)))
        return out

    def relin(self, ct3, level):
        a = np.ascontiguousarray(ct3, dtype=np.uint64)
        out = np.empty((2, level, self.n), dtype=np.uint64)
        self._chk(self.L.orc_relin(self.h, P(a), level, P(out)))
        return out

    def rescale(self, ct, level):
        a = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.empty((2, level - 1, self.n), dtype=np.uint64)
        self._chk(self.L.orc_rescale(self.h, P(a), level, P(out)))
        return out

    def boot(self, ct, level, out_level):
        a = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.empty((2, out_level, self.n), dtype=np.uint64)
        self._chk(self.L.orc_boot_reset(self.h, P(a), level, out_level, P(out)))
        return out

    def cmult(self, a, b, level):
        x = np.ascontiguousarray(a, dtype=np.uint64)
        y = np.ascontiguousarray(b, dtype=np.uint64)
        out = np.empty((3, level, self.n), dtype=np.uint64)
        self._chk(self.L.orc_cmult(self.h, P(x), P(y), level, P(out)))
        return out

    def key_limb(self, key_id, digit, comp, ext):
        out = np.empty(self.n, dtype=np.uint64)
        self.L.orc_key_limb(self.h, key_id, digit, comp, ext, P(out))
        return out

    def weight_limb(self, bundle, lane, limb):
        out = np.empty(self.n, dtype=np.uint64)
        self.L.orc_weight_limb(self.h, bundle, lane, limb, P(out))
        return out

    def input_limb(self, bundle, lane, comp, limb):
        out = np.empty(self.n, dtype=np.uint64)
        self.L.orc_input_limb(self.h, bundle, lane, comp, limb, P(out))
        return out

    def input_bundle(self, bundle, lanes, comps, level):
        out = np.empty((lanes, comps, level, self.n), dtype=np.uint64)
        for ln in range(lanes):
            for c in range(comps):
                for lb in range(level):
                    out[ln, c, lb] = self.input_limb(bundle, ln, c, lb)
        return out

    def run_graph(self, path, max_ops=-1, nbundles=1 << 16):
        h = np.zeros(nbundles, dtype=np.uint64)
        nb = self._chk(self.L.orc_run_graph(self.h, str(path).encode(), max_ops, P(h), nbundles))
        return h[:nb]

    def run_graph_tg(self, path, tg_total, tg_sel, max_ops=-1, nbundles=1 << 16):
        """Lanes of token group tg_sel only (hashes over those lanes)."""
        h = np.zeros(nbundles, dtype=np.uint64)
        nb = self._chk(self.L.orc_run_graph_tg(self.h, str(path).encode(), max_ops, P(h), nbundles,
                                               tg_total, tg_sel))
        return h[:nb]


def hash_bundle(a, comps=None, level=None):
    """DESIGN.md §2.4 hash of a [lanes][comps][level][N] array (first comps/level)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    lanes, cs, lv, n = a.shape
    return lib().orc_hash_bundle_data(P(a), lanes, cs, cs if comps is None else comps, lv,
                                      lv if level is None else level, n)
