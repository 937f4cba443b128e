"""The Aegis execution plan (csrc/plan.cu; comm_plan.hpp:51-118 restated for this
executor): per-device compute streams, collective events with trigger/wait
positions, the per-matmul mode analysis of the reference's byte rule
(comm_plan.hpp:194-242) and the staggered diagonal order.
CPU only: planning needs no device."""
import collections

import pytest

from paper_2604_03425_b200 import plan_graph

N = 1 << 16
LIMB = 8 * N
MODES = ("local", "gather_inputs", "reduce_outputs")


def test_single_device_plan_is_the_op_list():
    g = plan_graph(log_n=16, tokens=512)
    p = g.plan(1)
    s = p.summary()
    assert s["events"] == 0 and s["executable"] == 1
    assert s["instrs_total"] == g.info()[0]
    assert [i["op"] for i in p.device(0)] == list(range(g.info()[0]))


@pytest.mark.parametrize("world", [2, 4])
def test_token_group_shards_need_no_collective(world):
    """T = 2048 has 4 token groups: G <= 4 places whole groups per device."""
    p = plan_graph(log_n=16, tokens=2048).plan(world)
    s = p.summary()
    assert s["executable"] == 1 and s["events"] == 0 and s["bytes_total"] == 0
    # every HE op's output lanes are covered exactly once across the devices
    g = plan_graph(log_n=16, tokens=2048)
    _, bundles, ops, _ = g.export()
    cover = collections.Counter()
    for d in range(world):
        for i in p.device(d):
            if ops[i["op"]].kind != 0:  # Encode weights are replicated
                cover[i["op"]] += i["lane_count"]
    for k, o in enumerate(ops):
        if o.kind != 0:
            assert cover[k] == o.out.lane_count, k


def test_eight_devices_reduce_scatter_each_pcmm_once():
    g = plan_graph(log_n=16, tokens=2048)
    p = g.plan(8, reorder=False)
    s = p.summary()
    ev = p.events()
    # qkv (3 sub-tensors) + out_proj + ffn1 + ffn2, for each of the 4 token groups
    assert s["events"] == len(ev) == 4 * (3 + 1 + 1 + 1)
    assert all(e["kind"] == 1 and e["semantic"] == 2 and e["executed"] == 1 and e["dev_count"] == 2 for e in ev)
    assert s["bytes_total"] == sum(e["bytes_total"] for e in ev) == s["bytes_ffn"]
    for e in ev:  # NCCL volume: each of the 2 ranks sends the other's half of the sub-tensor
        assert e["bytes_per_device"] == (e["lane_count"] // 2) * e["level"] * 2 * LIMB
    # trigger (last PMult) precedes the wait (the rescale over this device's share) on every device
    ops = g.export()[2]
    for d in range(8):
        instrs = p.device(d)
        waits = {i["wait_event"]: k for k, i in enumerate(instrs) if i["wait_event"] >= 0}
        mine = [e for e in ev if e["dev_lo"] <= d < e["dev_lo"] + e["dev_count"]]
        assert set(waits) == {e["id"] for e in mine}
        for e in mine:
            last_pm = max(k for k, i in enumerate(instrs)
                          if ops[i["op"]].kind == 3 and ops[i["op"]].out.bundle == e["bundle"])
            assert last_pm < waits[e["id"]]


def test_reference_rule_modes_and_send_before_boot():
    """comm_plan.hpp:226-238: gather when the (pre-boot) activation is cheaper to
    ship than the partial accumulators.  qkv (12 -> 36 lanes) and ffn1 (12 -> 48)
    gather; out_proj and ffn2 reduce.  ffn1's activation is the LayerNorm boot
    output, so the gather ships the pre-boot bundle at its lower level."""
    g = plan_graph(log_n=16, tokens=2048)
    _, bundles, _, _ = g.export()
    mm = {bundles[m["acc_bundle"]].tag.decode().split(".")[1]: m for m in g.plan(8).matmuls()}
    assert {k: MODES[v["chosen"]] for k, v in mm.items()} == {
        "qkv": "gather_inputs", "out_proj": "reduce_outputs", "ffn1": "gather_inputs", "ffn2": "reduce_outputs"}
    assert all(MODES[v["executed"]] == "reduce_outputs" for v in mm.values())
    f1 = mm["ffn1"]
    assert f1["ship_bundle"] != f1["input_bundle"]
    assert bundles[f1["ship_bundle"]].level < bundles[f1["input_bundle"]].level


def test_staggered_diagonal_order():
    """reorder: device part p starts each matmul's rotation-offset sequence at
    offset p * 64 / m; the instructions are a permutation of the
    unreordered stream and every event still triggers before it is waited on."""
    g = plan_graph(log_n=16, tokens=2048)
    a, b = g.plan(8, reorder=False), g.plan(8, reorder=True)
    _, _, ops, _ = g.export()
    for d in range(8):
        ia, ib = a.device(d), b.device(d)
        key = lambda i: (i["op"], i["lane"], i["lane_count"])
        assert sorted(map(key, ia)) == sorted(map(key, ib))
        part = d % 2
        rots = [ops[i["op"]].phase for i in ib if ops[i["op"]].kind == 5 and ops[i["op"]].phase > 0]
        assert rots and (rots[0] == 32 if part else rots[0] == 1)
    for e in b.events():
        assert e["executed"] == 1


def test_unsplittable_shape_reports_why():
    """T = 128 on 2 devices splits one token group whose score accumulator
    wraps onto fewer lanes than its readers: not executable, but the matmul
    analysis (the reference rule's bytes) is still produced."""
    p = plan_graph(log_n=16, tokens=128).plan(2)
    s = p.summary()
    assert s["executable"] == 0 and s["events"] == 0
    assert "reads lanes another rank owns" in p.note
    assert s["matmuls"] == 4 and s["bytes_reference_rule"] > 0


def test_graph_in_plan_order_is_a_permutation(tmp_path):
    """aegis_graph_from_plan: the ops of device d of a reordered plan, in that
    device's order -- a permutation of the op list that moves only the
    diagonal loops, each rotation still before its PMult."""
    g = plan_graph(log_n=16, tokens=2048)
    p = g.plan(8, reorder=True)
    h = g.in_plan_order(p, 1)
    a, b = tmp_path / "a.heops", tmp_path / "b.heops"
    g.dump(a)
    h.dump(b)
    la = [ln for ln in open(a) if ln.startswith("O ")]
    lb = [ln for ln in open(b) if ln.startswith("O ")]
    assert sorted(la) == sorted(lb) and la != lb
    ops = h.export()[2]
    rot_pos = {}
    for k, o in enumerate(ops):
        if o.kind == 5:
            rot_pos[o.out.bundle] = k
        if o.kind == 3:  # PMult reads its rotated input after the rotation produced it
            src = o.ins[0].bundle
            assert src not in rot_pos or rot_pos[src] < k


def test_reference_modes_plan_gathers_where_the_rule_says():
    """aegis_graph_set_matmul_modes(g, 1): qkv and ffn1 (activation cheaper to
    ship than the partial outputs) become one AllGather per token group, out_proj
    and ffn2 stay reduce-scatters; the plan moves fewer bytes, and every device
    computes its own output share of a gathered matmul on all the group's inputs."""
    g = plan_graph(log_n=16, tokens=2048)
    base = g.plan(8, reorder=False).summary()
    g.set_matmul_modes(True)
    p = g.plan(8, reorder=False)
    s, ev = p.summary(), p.events()
    kinds = collections.Counter(e["kind"] for e in ev)
    assert kinds[0] == 2 * 4 and kinds[1] == 2 * 4  # 8 AllGathers (qkv, ffn1) + 8 reduce-scatters
    assert all(e["executed"] for e in ev)
    assert s["bytes_total"] < base["bytes_total"]
    _, bundles, ops, _ = g.export()
    mm = {bundles[m["acc_bundle"]].tag.decode().split(".")[1]: MODES[m["executed"]] for m in p.matmuls()}
    assert mm == {"qkv": "gather_inputs", "out_proj": "reduce_outputs", "ffn1": "gather_inputs",
                  "ffn2": "reduce_outputs"}
    for e in ev:
        if e["kind"] == 0:
            assert e["bytes_per_device"] == (e["lane_count"] // 2) * e["level"] * 2 * LIMB
