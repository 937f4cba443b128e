"""A small end-to-end pass for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once -- v2 NTT + fused conversion + finish at N = 2^16 (one
rotation and one relinearisation at level 6), the generic passes at N = 2^10,
the FFN graph (PCMM, CMult, Relin, Rescale, Boot), the limb ops and the stored
PCMM.  GPU; prints one line."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from paper_2604_03425_b200 import Context, _lib  # noqa: E402


def main():
    c16 = Context(log_n=16)
    x = c16.bundle(2, 2, 6)
    x.fill_input(1)
    out = c16.bundle(2, 2, 6)
    c16.keys_generate([0, 1003])
    c16.rot(out, x, 3, 6)
    p3 = c16.bundle(2, 3, 6)
    c16.cmult(p3, x, x, 6)
    c16.relin(p3, 6)
    r = c16.bundle(2, 2, 5)
    c16.rescale(r, p3, 6)
    c16.sync()
    c10 = Context(log_n=10)
    from conftest import golden_graph
    with tempfile.TemporaryDirectory() as d:
        g = c10.load_graph(golden_graph("ffn_n10_t8", d))
        h = g.run(hashes=True)
        g.set_stored_weights(True)
        h2 = g.run(hashes=True)
    assert (h == h2).all()
    a = c10.bundle(2, 2, 4)
    a.fill_input(3)
    o = c10.bundle(2, 3, 4)
    c10.limb_op(_lib.LIMB_MUL, o, a, a, lo=1, hi=3)
    c10.sync()
    print(f"sanitize smoke ok: {c16.launch_count() + c10.launch_count()} kernels", flush=True)


if __name__ == "__main__":
    main()
