"""Real CKKS round trip through the GPU operators: ternary
secret, keys via aegis_keys_upload, symmetric encryption, then CMult + Relin +
Rescale, Rot and a 4-step rotate-and-sum; prints max |decrypted - expected|.
Dev tool; GPU.

    python tools/ckks_demo.py [--log-n 16] [--levels 5,17,35]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2604_03425_b200 import Context  # noqa: E402
from paper_2604_03425_b200.ckks import Ckks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log-n", type=int, default=16)
    ap.add_argument("--levels", default="5,17,35")
    ap.add_argument("--scale-bits", type=int, default=40)
    a = ap.parse_args()
    c = Context(log_n=a.log_n)
    k = Ckks(c, seed=11)
    k.upload_relin_key()
    for r in (1, 2, 4, 8):
        k.upload_rotation_key(r)
    scale = 2.0 ** a.scale_bits
    rng = np.random.default_rng(0)
    z = rng.uniform(-1, 1, c.n // 2) + 1j * rng.uniform(-1, 1, c.n // 2)
    print(f"N = 2^{a.log_n}, {c.n // 2} slots, scale 2^{a.scale_bits}, ternary secret (h = 64)")
    for L in map(int, a.levels.split(",")):
        ct = k.encrypt(z, scale, L)
        e_fresh = np.abs(k.decrypt(ct, scale, L) - z).max()
        sq = c.bundle(1, 3, L)
        c.cmult(sq, ct, ct, L)
        c.relin(sq, L)
        out = c.bundle(1, 2, L - 1)
        c.rescale(out, sq, L)
        e_sq = np.abs(k.decrypt(out, scale * scale / k.q[L - 1], L - 1) - z * z).max()
        acc = c.bundle(1, 2, L)
        c.cadd(acc, ct, ct, L)  # 2z
        tmp = c.bundle(1, 2, L)
        want = 2 * z
        for r in (1, 2, 4, 8):
            c.rot(tmp, acc, r, L)
            c.cadd(acc, tmp, None, L, accumulate=True)
            want = want + np.roll(want, -r)
        e_sum = np.abs(k.decrypt(acc, scale, L) - want).max()
        print(f"level {L:2d}: fresh {e_fresh:.2e}   CMult+Relin+Rescale {e_sq:.2e}   "
              f"rotate-and-sum (4 Rot) {e_sum:.2e}  (|want| <= {np.abs(want).max():.1f})", flush=True)
        for b in (ct, sq, out, acc, tmp):
            b.free()
    c.close()


if __name__ == "__main__":
    main()
