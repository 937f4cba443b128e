"""Algorithmic HBM bytes of an HE-op graph.

Minimal model: every input read once, every output written once, on-chip
intermediates and twiddle / constant tables excluded, limb = 8N bytes.  Per
bundled HeOp at level l = use_level over B = out lanes:

  Rot / Relin (key switch, one key per op, d = ceil(l/4) digits):
      (B (c_in l + 2 l) + 2 d (l + 4)) 8N,  c_in = 2 (Rot) / 3 (Relin)
  PMult-acc (generated weights):  (in_lanes 2 l + out_lanes 2 2 l) 8N
  CMult 7 l 8N, CAdd 6 l 8N, Rescale (4 l - 2) 8N, Boot (2 l + 42) 8N per lane
  Encode 0 (the weights are generated inside the PMult kernel)

bench.py divides the graph total by the step time for `roofline.layer`.
"""

# HeOpKind (he_ir.hpp:21-31)
ENCODE, PADD, CADD, PMULT, CMULT, ROT, RELIN, RESCALE, BOOT = range(9)


def op_bytes(kind, level, lanes, n, in_lanes=0):
    limb = 8 * n
    lv = level
    if kind in (ROT, RELIN):
        d = -(-lv // 4)
        c_in = 2 if kind == ROT else 3
        return (lanes * (c_in * lv + 2 * lv) + 2 * d * (lv + 4)) * limb
    if kind == PMULT:
        return (in_lanes * 2 * lv + lanes * 2 * 2 * lv) * limb
    if kind == CMULT:
        return 7 * lv * limb * lanes
    if kind in (CADD, PADD):
        return 6 * lv * limb * lanes
    if kind == RESCALE:
        return (4 * lv - 2) * limb * lanes
    if kind == BOOT:
        return (2 * lv + 42) * limb * lanes
    return 0


def graph_bytes(ops, n):
    """Sum over the graph's ops (descriptors from Graph.export()); returns
    (total bytes, {kind: bytes})."""
    per = {}
    for o in ops:
        b = op_bytes(o.kind, o.use_level, o.out.lane_count, n, o.ins[0].lane_count if o.in_count else 0)
        per[o.kind] = per.get(o.kind, 0) + b
    return sum(per.values()), per
