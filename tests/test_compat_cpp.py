"""The heplan-side C++ binding (paper_2604_03425_b200/csrc/heplan_compat.hpp),
compiled against the UNMODIFIED reference headers by tests/cpp/Makefile
(__graft_entry__.build() runs it where /root/reference exists; the binary
travels to the GPU box with the snapshot)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "compat_test")

needs_bin = pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/_bin/compat_test not built "
                               "(needs the reference headers at build time)")


@needs_bin
def test_reference_graph_ingested_in_memory_equals_own_lowering(tmp_path):
    """heplan::lower_app_to_he output handed over in memory (aegis_graph_from_ops)
    is the graph libaegis lowers itself; malformed graphs throw
    std::invalid_argument through the wrapper."""
    r = subprocess.run([BIN, "plan", str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ffn_n16_t128: 426 ops, ingested == own lowering" in r.stdout
    assert "malformed graph rejected" in r.stdout


@needs_bin
@pytest.mark.gpu
def test_reference_graph_runs_through_the_wrapper(golden_dir):
    """Executor::exec_sequential (heplan_compat.hpp) runs the reference-lowered
    FFN on the GPU; every bundle hash equals the CPU oracle's on the same graph."""
    from conftest import golden_graph
    from oracle_py import Oracle
    r = subprocess.run([BIN, "run"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    got = np.array([int(x, 16) for x in r.stdout.split()], dtype=np.uint64)
    want = Oracle(10).run_graph(golden_graph("ffn_n10_t8", golden_dir))
    assert len(got) == len(want)
    assert (got == want).all()
