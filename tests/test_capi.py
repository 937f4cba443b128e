"""The C-ABI boundary: library loads, exports every declared symbol, and
reports errors through codes (no exceptions) -- CPU only, no compute calls."""
import ctypes
import os
import re

import pytest

from paper_2604_03425_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "aegis.h")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(aegis_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(declared()) == bound


def test_ctx_create_rejects_bad_params():
    lib = _lib.load()
    h = ctypes.c_void_p()
    p = _lib.AegisParams(16, 35, 3, 14, 1, 2, 3)  # |P| must be 4
    assert lib.aegis_ctx_create(ctypes.byref(p), 0, ctypes.byref(h)) == _lib.AEGIS_EINVAL
    assert b"special_prime_count" in lib.aegis_last_error(None)
    p = _lib.AegisParams(16, 35, 4, 40, 1, 2, 3)  # l_boot > chain (ckks.hpp:45)
    assert lib.aegis_ctx_create(ctypes.byref(p), 0, ctypes.byref(h)) == _lib.AEGIS_EINVAL


def test_null_arguments_are_errors_not_crashes():
    lib = _lib.load()
    assert lib.aegis_ctx_create(None, 0, None) == _lib.AEGIS_EINVAL
    assert lib.aegis_graph_info(None, None, None) == _lib.AEGIS_EINVAL
    assert lib.aegis_bundle_info(None, None, None, None, None) == _lib.AEGIS_EINVAL
    assert lib.aegis_graph_dump(None, b"/tmp/x") == _lib.AEGIS_EINVAL


def test_graph_key_ids_cover_rotations_and_relin():
    from paper_2604_03425_b200 import plan_graph
    g = plan_graph(log_n=16, tokens=128, layers=1)
    ids = set(int(x) for x in g.key_ids())
    assert 0 in ids and all(1000 + r in ids for r in range(1, 64))
    assert len(ids) == 64


def _load(path):
    lib = _lib.load()
    g = ctypes.c_void_p()
    rc = lib.aegis_graph_load(None, str(path).encode(), ctypes.byref(g))
    if rc == 0:
        lib.aegis_graph_free(g)
    return rc, lib.aegis_last_error(None)


def test_graph_load_validates_every_index(tmp_path, golden_dir):
    """aegis_graph_load (no device needed) accepts every reference-emitted graph
    and rejects out-of-range bundle / lane / level / offset fields with
    AEGIS_EINVAL instead of letting the executor index past its tables."""
    from conftest import golden_graph
    for name in ("ffn_n10_t8", "block_n11_t32", "block_n16_t2048"):
        assert _load(golden_graph(name, golden_dir))[0] == 0, name
    base = open(golden_graph("ffn_n10_t8", golden_dir)).read().splitlines()
    first_op = next(i for i, ln in enumerate(base) if ln.startswith("O ") and ln.split()[2] == "5")  # a Rot
    f = base[first_op].split()

    def mutate(idx, value, what):
        g = list(f)
        g[idx] = str(value)
        p = tmp_path / f"bad_{idx}.heops"
        p.write_text("\n".join(base[:first_op] + [" ".join(g)] + base[first_op + 1:]) + "\n")
        rc, msg = _load(p)
        assert rc == _lib.AEGIS_EINVAL, (what, rc)
        return msg

    nb = sum(1 for ln in base if ln.startswith("B "))
    mutate(4, nb + 7, "output bundle out of range")          # O id kind rot out.b ...
    mutate(6, 1 << 20, "output lane count beyond the bundle")
    mutate(11, 60, "use_level above the operand level")
    mutate(3, -700, "rotation offset aliasing the relin key ids")


def test_graph_from_ops_round_trip(tmp_path):
    """In-memory HeOpGraph ingest (aegis_graph_from_ops): exporting a lowered
    graph to descriptor arrays and ingesting them back gives the identical
    graph (same heops dump), with no text round trip and no device."""
    from paper_2604_03425_b200 import plan_graph
    from paper_2604_03425_b200.api import graph_from_ops
    for kind, tokens in ((1, 128), (0, 512)):
        g = plan_graph(log_n=16, kind=kind, tokens=tokens)
        meta, bundles, ops, inputs = g.export()
        assert meta.log_n == 16 and meta.tokens == tokens and meta.kind == kind
        h = graph_from_ops(meta, bundles, ops, inputs)
        a, b = tmp_path / "a.heops", tmp_path / "b.heops"
        g.dump(a)
        h.dump(b)
        assert open(a).read() == open(b).read()
        assert h.key_ids().tolist() == g.key_ids().tolist()


def test_graph_from_ops_validates(tmp_path):
    from paper_2604_03425_b200 import plan_graph
    from paper_2604_03425_b200.api import graph_from_ops
    g = plan_graph(log_n=16, kind=1, tokens=128)
    meta, bundles, ops, inputs = g.export()
    rot = next(i for i, o in enumerate(ops) if o.kind == 5)
    cases = [("bundle", lambda o: setattr(o.out, "bundle", len(bundles) + 3), "outside its bundle"),
             ("lane", lambda o: setattr(o.ins[0], "lane_count", 10_000), "outside its bundle"),
             ("level", lambda o: setattr(o, "use_level", 60), "use_level"),
             ("offset", lambda o: setattr(o, "rot_offset", -700), "offset"),
             ("kind", lambda o: setattr(o, "kind", 42), "unknown kind"),
             ("ins", lambda o: setattr(o, "in_count", 9), "too many operands")]
    for name, mutate, msg in cases:
        bad = list(ops)
        o = type(ops[rot]).from_buffer_copy(ops[rot])
        mutate(o)
        bad[rot] = o
        with pytest.raises(ValueError, match=msg):
            graph_from_ops(meta, bundles, bad, inputs)
