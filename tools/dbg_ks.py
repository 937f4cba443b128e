import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_2604_03425_b200 import Context
from oracle_py import Oracle
from tools_params import main_primes, special_primes
MP, SP = main_primes(), special_primes()
for logn in (4, 10):
    c = Context(log_n=logn); o = Oracle(logn); n = 1 << logn
    for level in (1, 2, 4, 5, 8):
        for key in (0, 1007, 1001):
            rng = np.random.default_rng(level)
            x = np.stack([np.stack([np.stack([rng.integers(0, MP[lb], n, dtype=np.uint64) for lb in range(level)]) for _ in range(2)]) for _ in range(2)])
            bi = c.bundle(2, 2, level); bi.upload(x)
            bo = c.bundle(2, 2, level)
            c.keyswitch(bo, bi, 1, level, key)
            got = bo.download()
            ok = []
            for ln in range(2):
                o0, o1 = o.keyswitch(x[ln, 1], level, key)
                ok.append(((got[ln, 0] == o0).all(), (got[ln, 1] == o1).all(),
                           [int((got[ln, 0][i] == o0[i]).all()) for i in range(level)]))
            print(logn, level, key, ok)
