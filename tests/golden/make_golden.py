"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Runs only in the build container, where /root/reference exists: it loads
oracle/_ref/libheplan_ref.so (compiled in place from
/root/reference/proj/include/heplan by oracle/Makefile; see oracle/ref_shim.cpp)
and records
  * ref_kats.json  -- rns_math.hpp known answers: NTT forward/inverse vectors
                      (rns_math.hpp:68-100) for toy and production primes,
                      galois powers (:142-149), coefficient-domain automorphisms
                      (:127-139), centred CRT lifts (:171-186), div_round
                      (:196-202), ckks.hpp byte models (:147-157, :217-223);
  * *.heops.gz     -- HE-op graphs emitted by lower_app_to_he (he_ir.hpp:683)
                      for the BASELINE configs and small-N parity configs.
Usage:  python tests/golden/make_golden.py
"""
import ctypes
import gzip
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

u64p = ctypes.POINTER(ctypes.c_uint64)

# Graph fixtures: (name, log_n, tokens, layers, kind)  kind 0 = blocks, 1 = FFN only
GRAPHS = [
    ("ffn_n16_t128", 16, 128, 1, 1),        # config 1
    ("block_n16_t128", 16, 128, 1, 0),
    ("block_n16_t512", 16, 512, 1, 0),      # config 2
    ("block_n16_t2048", 16, 2048, 1, 0),    # config 3 (one layer)
    ("blocks2_n16_t512", 16, 512, 2, 0),    # steady-state block levels
    ("blocks12_n16_t2048", 16, 2048, 12, 0),  # config 4
    ("ffn_n10_t8", 10, 8, 1, 1),            # small-N parity configs
    ("block_n10_t8", 10, 8, 1, 0),
    ("block_n11_t32", 11, 32, 1, 0),        # 2 token groups, chunked QKV
    ("ffn_n11_t32", 11, 32, 1, 1),
]


def load_ref():
    path = os.path.join(ROOT, "oracle", "_ref", "libheplan_ref.so")
    lib = ctypes.CDLL(path)
    lib.ref_ntt.argtypes = [ctypes.c_uint32, ctypes.c_uint64, u64p, ctypes.c_int]
    lib.ref_automorphism.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, u64p, u64p]
    lib.ref_galois.restype = ctypes.c_uint64
    lib.ref_galois.argtypes = [ctypes.c_int, ctypes.c_uint32]
    lib.ref_lift_centered.argtypes = [u64p, ctypes.c_uint32, u64p, u64p, ctypes.POINTER(ctypes.c_int64)]
    lib.ref_div_round.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64,
                                  u64p, ctypes.POINTER(ctypes.c_int64)]
    lib.ref_ciphertext_bytes.restype = ctypes.c_uint64
    lib.ref_ciphertext_bytes.argtypes = [ctypes.c_uint32] * 3
    lib.ref_key_switch_key_bytes.restype = ctypes.c_uint64
    lib.ref_key_switch_key_bytes.argtypes = [ctypes.c_uint32] * 3
    lib.ref_dump_he.argtypes = [ctypes.c_uint32] * 8 + [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                                                        ctypes.c_int, ctypes.c_char_p]
    return lib


def P(a):
    return a.ctypes.data_as(u64p)


def ntt_input(n, p, seed):
    """Deterministic NTT input: numpy PCG64(seed) uniform in [0, p)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, p, n, dtype=np.uint64)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def main():
    from tools_params import main_primes, special_primes  # noqa: E402
    ref = load_ref()
    mp, sp = main_primes(), special_primes()
    kats = {"ntt": [], "galois": [], "automorphism": [], "crt": [], "div_round": [], "bytes": {}}
    # --- NTT: full vectors for small n, sha256 for production sizes ---
    cases = [(16, 97, 1), (16, 193, 2), (1024, 12289, 3)]
    for logn in (4, 10, 16, 17):
        for e, p in ((0, mp[0]), (1, mp[1]), (34, mp[34]), (60, sp[0])):
            cases.append((1 << logn, p, 100 + logn * 64 + e))
    for n, p, seed in cases:
        a = ntt_input(n, p, seed)
        f = a.copy()
        assert ref.ref_ntt(n, p, P(f), 0) == 0
        g = f.copy()
        assert ref.ref_ntt(n, p, P(g), 1) == 0
        assert (g == a).all()
        rec = {"n": n, "p": int(p), "seed": seed}
        if n <= 1024:
            rec["forward"] = [int(x) for x in f]
        else:
            rec["forward_sha256"] = sha(f)
            rec["forward_head"] = [int(x) for x in f[:8]]
        kats["ntt"].append(rec)
    # --- galois powers and automorphisms ---
    for n in (16, 1024, 1 << 16, 1 << 17):
        for off in (0, 1, 2, 3, 5, 32, 63, -1, -5):
            kats["galois"].append({"n": n, "offset": off, "k": int(ref.ref_galois(off, n))})
    for n, p in ((16, 97), (16, mp[0]), (64, mp[3])):
        a = ntt_input(n, p, 7 + n)
        for off in (1, 3, 7, -1):
            k = ref.ref_galois(off, n)
            out = np.zeros(n, dtype=np.uint64)
            ref.ref_automorphism(n, k, p, P(a), P(out))
            kats["automorphism"].append({"n": n, "p": int(p), "seed": 7 + n, "k": int(k),
                                         "out": [int(x) for x in out]})
    # --- centred CRT (toy bases: prod < 2^127) and div_round ---
    rng = np.random.default_rng(11)
    for basis in ([97, 193, 257], [12289, 40961], [mp[1], mp[2]], [97]):
        arr = np.array(basis, dtype=np.uint64)
        Q = 1
        for b in basis:
            Q *= b
        vals = [0, 1, Q - 1, (Q - 1) // 2, (Q + 1) // 2, Q // 3] + [int(x) for x in rng.integers(0, min(Q, 2**62), 4)]
        for v in vals:
            r = np.array([v % b for b in basis], dtype=np.uint64)
            lo, hi = ctypes.c_uint64(), ctypes.c_int64()
            assert ref.ref_lift_centered(P(arr), len(basis), P(r), ctypes.byref(lo), ctypes.byref(hi)) == 0
            lifted = (hi.value << 64) | lo.value
            kats["crt"].append({"basis": [int(b) for b in basis], "residues": [int(x) for x in r],
                                "lift": int(lifted)})
    for num, den in ((7, 2), (-7, 2), (5, 3), (-5, 3), (9, 6), (-9, 6), (10**20 + 7, 97), (-(10**20) - 7, 97)):
        nlo, nhi = num & (2**64 - 1), num >> 64
        dlo, dhi = den & (2**64 - 1), den >> 64
        qlo, qhi = ctypes.c_uint64(), ctypes.c_int64()
        ref.ref_div_round(nlo, nhi, dlo, dhi, ctypes.byref(qlo), ctypes.byref(qhi))
        kats["div_round"].append({"num": num, "den": den, "q": (qhi.value << 64) | qlo.value})
    kats["bytes"] = {
        "ciphertext_65536_35_2": int(ref.ref_ciphertext_bytes(65536, 35, 2)),
        "ciphertext_32_3_2": int(ref.ref_ciphertext_bytes(32, 3, 2)),
        "key_switch_65536_35_4": int(ref.ref_key_switch_key_bytes(65536, 35, 4)),
    }
    with open(os.path.join(HERE, "ref_kats.json"), "w") as f:
        json.dump(kats, f, indent=0)
    # --- HE-op graphs ---
    for name, logn, T, layers, kind in GRAPHS:
        tmp = f"/tmp/{name}.heops"
        nops = ref.ref_dump_he(1 << logn, 35, 4, 14, 64, 768, 64, 3072, T, layers, kind, 0, tmp.encode())
        assert nops > 0, name
        with open(tmp, "rb") as fi, gzip.GzipFile(os.path.join(HERE, f"{name}.heops.gz"), "wb", mtime=0) as fo:
            fo.write(fi.read())
        print(f"{name}: {nops} ops")


if __name__ == "__main__":
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    main()
