"""Layer drivers: libaegis' lowering must emit exactly the reference's HE-op graph.

The golden graphs were emitted by the unmodified reference lower_app_to_he
(he_ir.hpp:683) -- see tests/golden/make_golden.py.  Bundle ids seed the
generated weights, so a single differing field would change every residue.
"""
import collections
import gzip
import os

import pytest

from paper_2604_03425_b200 import plan_graph

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = [
    ("ffn_n16_t128", 16, 128, 1, 1),
    ("block_n16_t128", 16, 128, 1, 0),
    ("block_n16_t512", 16, 512, 1, 0),
    ("block_n16_t2048", 16, 2048, 1, 0),
    ("blocks2_n16_t512", 16, 512, 2, 0),
    ("blocks12_n16_t2048", 16, 2048, 12, 0),
    ("ffn_n10_t8", 10, 8, 1, 1),
    ("block_n10_t8", 10, 8, 1, 0),
    ("block_n11_t32", 11, 32, 1, 0),
    ("ffn_n11_t32", 11, 32, 1, 1),
]
KINDS = ["encode", "padd", "cadd", "pmult", "cmult", "rot", "relin", "rescale", "boot"]


def golden_lines(name):
    with gzip.open(os.path.join(GOLDEN, f"{name}.heops.gz"), "rt") as f:
        return f.read().splitlines()


@pytest.mark.parametrize("name,logn,T,layers,kind", CASES, ids=[c[0] for c in CASES])
def test_lowering_matches_reference(name, logn, T, layers, kind, tmp_path):
    g = plan_graph(log_n=logn, tokens=T, layers=layers, kind=kind)
    out = tmp_path / "mine.heops"
    g.dump(out)
    mine = out.read_text().splitlines()
    ref = golden_lines(name)
    assert mine[0] == ref[0]  # header: same profile / config
    assert len(mine) == len(ref)
    for i, (a, b) in enumerate(zip(mine, ref)):
        assert a == b, f"line {i}: {a!r} != {b!r}"


def lane_ops(lines):
    c = collections.Counter()
    for ln in lines:
        if ln.startswith("O "):
            f = ln.split()
            work, lanes = int(f[10]), int(f[6])
            c[KINDS[int(f[2])]] += work if work else lanes
    return c


def test_config1_op_counts():
    """SURVEY Appendix A, config 1."""
    c = lane_ops(golden_lines("ffn_n16_t128"))
    assert c["rot"] == 756 + 3024
    assert c["relin"] == 672 and c["cmult"] == 672
    assert c["pmult"] == 73_728
    assert c["rescale"] == 732
    assert sum(1 for ln in golden_lines("ffn_n16_t128") if ln.startswith("O ")) == 426


def test_block_op_counts():
    """SURVEY Appendix A totals: 1511 HE ops per block; KS lane-ops 10,806 / 18,456 / 171,744."""
    for name, ks in (("block_n16_t128", 10_806), ("block_n16_t512", 18_456), ("block_n16_t2048", 171_744)):
        lines = golden_lines(name)
        assert sum(1 for ln in lines if ln.startswith("O ")) == 1511
        c = lane_ops(lines)
        assert c["rot"] + c["relin"] == ks
    c = lane_ops(golden_lines("block_n16_t2048"))
    assert c["boot"] == 4 * 48 and c["rescale"] == 30_816


def test_twelve_layers():
    lines = golden_lines("blocks12_n16_t2048")
    assert sum(1 for ln in lines if ln.startswith("O ")) == 18_132
    assert sum(1 for ln in lines if ln.startswith("B ")) == 11_101
    c = lane_ops(lines)
    assert c["rot"] + c["relin"] == 2_060_928
    assert c["boot"] == 2_304


def test_lowering_errors():
    with pytest.raises(ValueError):
        plan_graph(log_n=16, tokens=128, chain_length=20, bootstrap_level=14)  # usable depth < 21
    with pytest.raises(ValueError):
        plan_graph(log_n=16, tokens=128, slots_per_token=48)  # not a divisor of the slot count
    with pytest.raises(ValueError):
        plan_graph(log_n=2, tokens=8)
