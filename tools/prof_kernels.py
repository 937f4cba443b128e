"""Run each hot kernel once on production shapes (for ncu captures)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_03425_b200 import Context  # noqa: E402

c = Context(log_n=16)
b = c.bundle(48, 1, 17)
b.fill_input(1)
c.ntt(b)                 # warm
c.ntt(b)                 # profiled forward (2 passes)
c.ntt(b, inverse=True)   # profiled inverse
x = c.bundle(16, 2, 17)
x.fill_input(2)
o = c.bundle(16, 2, 17)
c.rot(o, x, 5, 17)       # one key switch batch at l = 17
c.sync()
print("done")
