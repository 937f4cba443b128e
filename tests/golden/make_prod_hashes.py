"""Generate the production-size whole-graph parity fixtures (TEST INFRASTRUCTURE).

Runs the CPU oracle (oracle/liboracle.so, built by oracle/Makefile) over the
HE-op graphs the unmodified reference lowering emitted for the BASELINE
configs (tests/golden/*.heops.gz, made by make_golden.py) and records the
DESIGN.md §2.4 hash of every bundle, at N = 2^16 with the BERT parameters:

  prod_ffn_n16_t128.json          config 1, every lane             (426 ops)
  prod_block_n16_t512.json        config 2, every lane             (1,511 ops)
  prod_block_n16_t2048_tg0.json   the headline T = 2048 layer, the lanes of
                                  token group 0 of 4 (orc_run_graph_tg: the
                                  oracle's own token-coherent lane tagging)
  prod_blocks2_n16_t512.json      two blocks at T = 512 (3,022 ops): block 2 at
                                  the steady-state levels of config 4

tests/test_gpu_parity.py compares every hash with the GPU executor's (the
headline run is unsharded; it hashes the token-group-0 lanes only).
Usage: python tests/golden/make_prod_hashes.py [name ...]   (hours for tg0)
"""
import json
import os
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import golden_graph  # noqa: E402
from oracle_py import Oracle  # noqa: E402

JOBS = {  # fixture -> (graph, tg_total, tg_sel)
    "prod_ffn_n16_t128": ("ffn_n16_t128", 1, -1),
    "prod_block_n16_t512": ("block_n16_t512", 1, -1),
    "prod_block_n16_t2048_tg0": ("block_n16_t2048", 4, 0),
    # two blocks at T = 512: the second runs at the steady-state levels of config 4's blocks 2..12
    "prod_blocks2_n16_t512": ("blocks2_n16_t512", 1, -1),
}


def run(name):
    graph, tg_total, tg_sel = JOBS[name]
    orc = Oracle(16)
    with tempfile.TemporaryDirectory() as d:
        path = golden_graph(graph, d)
        t0 = time.time()
        h = orc.run_graph(path) if tg_sel < 0 else orc.run_graph_tg(path, tg_total, tg_sel)
        dt = time.time() - t0
    rec = {"graph": graph, "log_n": 16, "tg_total": tg_total, "tg_sel": tg_sel,
           "bundles": len(h), "hashes": [f"{int(v):016x}" for v in h],
           "oracle_seconds": round(dt, 1), "threads": os.cpu_count()}
    out = os.path.join(HERE, name + ".json")
    with open(out, "w") as f:
        json.dump(rec, f)
    print(f"{name}: {len(h)} bundles, {dt:.1f} s -> {out}", flush=True)


if __name__ == "__main__":
    for n in (sys.argv[1:] or list(JOBS)):
        run(n)
