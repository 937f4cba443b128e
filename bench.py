"""bench.py -- encrypted BERT-base layer latency on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl aegis|reference]
                    [--tokens T] [--layers L]

One step = one encrypted BERT-base encoder layer (the reference's HE-op
sequence for block 0: he_ir.hpp:683 on graph.hpp:168), N = 2^16, |Q_L| = 35,
|P| = 4, s_tok = 64, synthetic ciphertext inputs and keys.
For N > 1 (torchrun, one rank per GPU) the layer is strong-scaled: token
groups are sharded across ranks (token-coherent placement) and
`value` is the max-over-ranks device time of the whole layer.

`--impl reference` times the reference path on the host CPU: the reference has
no executor, so this is the oracle restatement (oracle/, "port")
of the reference-emitted op list, every op kind measured at the layer's own
levels on one lane per host thread and scaled by its lane count (measured
seconds and the extrapolation factor are reported), next to the reference's
own NegacyclicNtt (oracle/_ref, unmodified) timed on the same cores.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

N_LOG = 16
METRIC = "encrypted BERT layer latency @2048 tok"
L2_BYTES = 126 * 2**20


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class Clocks:
    """Sample nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, dev):
        self.dev, self.rows, self.proc = dev, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init(n_gpus):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if os.environ.get("AEGIS_BACKEND", "nccl") == "nccl" else "gloo")
        local = int(os.environ.get("LOCAL_RANK", "0"))
        # AEGIS_FORCE_DEVICE: run every rank on one GPU (multi-process path check on a 1-GPU box, gloo)
        return dist, dist.get_rank(), ws, int(os.environ.get("AEGIS_FORCE_DEVICE", local))
    return None, 0, 1, 0


def shard_range(tg_total, rank, ws):
    """Contiguous token-group chunk of this rank (placement.hpp:175-182 kLaneChunks)."""
    per = -(-tg_total // ws)
    lo = min(tg_total, rank * per)
    return lo, min(tg_total, lo + per)


# ---------------------------------------------------------------------------
def run_reference(args):
    """Reference arm: the CPU restatement (oracle) of the same layer, bounded sample."""
    dist, rank, ws, _ = dist_init(args.gpus)
    if rank != 0:
        return
    res = cpu_baseline(args, budget_s=args.cpu_budget)
    out = {
        "metric": METRIC, "value": res["value"], "unit": "s/layer", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["value"] * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 (RNS residues)", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"BERT-base encoder layer, {args.tokens} tokens, CKKS N=2^16, L=35, |P|=4",
                   "tokens": args.tokens, "layers": 1},
        "cpu_baseline": res,
        "e2e": {"value": res["value"], "unit": "s/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def _mini_graph(path, kind, level, lanes, c_in=0, c_out=0):
    """One bundled HE op at `level` over `lanes` lanes, in the heops text format
    (field order of he_ir.hpp's HeOp; the same format the reference lowering
    is dumped in).  Used only to time the CPU oracle on single ops."""
    L = ["# heops v1 calibration", "inputs 0", f"B 0 {lanes} {level} 2 0 0 0 0 in"]
    one = f"0 0 {lanes}"
    if kind == "rot":
        L += [f"B 1 {lanes} {level} 2 2 0 0 0 rot", f"O 0 5 1 1 0 {lanes} 0 0 1 0 {level} 0 0 1 {one}"]
    elif kind == "cmult":
        L += [f"B 1 {lanes} {level} 2 1 0 0 0 sq", f"O 0 4 0 1 0 {lanes} 0 0 -1 0 {level} 0 0 2 {one} {one}"]
    elif kind == "relin":  # CMult(x, x) then Relin of the product (the CMult is timed apart and subtracted)
        L += [f"B 1 {lanes} {level} 2 1 0 0 0 sq",
              f"O 0 4 0 1 0 {lanes} 0 0 -1 0 {level} 0 0 2 {one} {one}",
              f"O 1 6 0 1 0 {lanes} 0 0 -1 0 {level} 0 0 1 1 0 {lanes}"]
    elif kind == "rescale":
        L += [f"B 1 {lanes} {level - 1} 2 1 0 0 0 rs", f"O 0 7 0 1 0 {lanes} 0 0 -1 0 {level} 0 0 1 {one}"]
    elif kind == "cadd":
        L += [f"B 1 {lanes} {level} 2 1 0 0 0 sum", f"O 0 2 0 1 0 {lanes} 0 0 -1 0 {level} 0 0 2 {one} {one}"]
    elif kind == "boot":
        L += [f"B 1 {lanes} 21 2 1 0 0 0 bt", f"O 0 8 0 1 0 {lanes} 0 0 -1 0 {level} 0 0 1 {one}"]
    elif kind == "pmult":
        w = c_in * c_out
        L[2] = f"B 0 {c_in} {level} 2 0 0 0 0 in"
        L += [f"B 1 {c_out} {level} 2 1 {c_out} 0 0 acc", f"B 2 {w} {level} 1 3 0 0 0 w",
              f"O 0 0 0 2 0 {w} 0 0 -1 0 0 0 0 0",
              f"O 1 3 0 1 0 {c_out} 1 0 0 {c_in * c_out} {level} 0 0 2 0 0 {c_in} 2 0 {w}"]
    elif kind == "none":
        pass
    open(path, "w").write("\n".join(L) + "\n")


def _layer_ops(tokens):
    """The layer's op list as the UNMODIFIED reference lowering emitted it
    (tests/golden/block_n16_t<T>.heops.gz, made by tests/golden/make_golden.py
    from lower_app_to_he, he_ir.hpp:683) -- no libaegis on the reference arm."""
    import gzip
    path = os.path.join(ROOT, "tests", "golden", f"block_n16_t{tokens}.heops.gz")
    with gzip.open(path, "rt") as f:
        return [ln.split() for ln in f if ln.startswith("O ")], path


def _fit(points, degree):
    """least-squares polynomial through measured (level, seconds-per-lane) points"""
    xs = np.array([p[0] for p in points], dtype=float)
    ys = np.array([p[1] for p in points], dtype=float)
    deg = min(degree, len(xs) - 1)
    c = np.polyfit(xs, ys, deg)
    return lambda lv: max(float(np.polyval(c, lv)), 0.0)


def reference_ntt(threads, limbs=None):
    """BASELINE.md path (a): the reference's own NegacyclicNtt (rns_math.hpp:44-123,
    compiled unmodified into oracle/_ref/libheplan_ref.so) on the host cores:
    forward NTTs of N = 2^16 limbs over the 35 main primes, one limb per thread."""
    import ctypes
    from tools_params import main_primes
    so = os.path.join(ROOT, "oracle", "_ref", "libheplan_ref.so")
    if not os.path.exists(so):
        return {"unavailable": "oracle/_ref/libheplan_ref.so not built"}
    lib = ctypes.CDLL(so)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    lib.ref_ntt_set_create.restype = ctypes.c_void_p
    lib.ref_ntt_set_create.argtypes = [ctypes.c_uint32, u64p, ctypes.c_uint32]
    lib.ref_ntt_set_run.argtypes = [ctypes.c_void_p, u64p, ctypes.c_uint32, ctypes.c_int, ctypes.c_int]
    lib.ref_ntt_set_destroy.argtypes = [ctypes.c_void_p]
    n = 1 << N_LOG
    pr = np.array(main_primes()[:35], dtype=np.uint64)
    t0 = time.time()
    h = lib.ref_ntt_set_create(n, pr.ctypes.data_as(u64p), len(pr))
    t_tables = time.time() - t0
    limbs = limbs or 2 * threads
    rng = np.random.default_rng(1)
    data = np.stack([rng.integers(0, int(pr[i % len(pr)]), n, dtype=np.uint64) for i in range(limbs)])
    t0 = time.time()
    lib.ref_ntt_set_run(h, data.ctypes.data_as(u64p), limbs, 0, threads)
    dt = time.time() - t0
    lib.ref_ntt_set_destroy(h)
    return {"kind": "reference", "ns_per_limb": dt / limbs * 1e9, "limbs": limbs, "threads": threads,
            "measured_s": round(dt, 3), "table_build_s": round(t_tables, 3),
            "gbs_algorithmic": 2 * 8 * n * limbs / dt / 1e9,
            "what": "heplan::NegacyclicNtt::forward (rns_math.hpp:68-82), unmodified, N=2^16, 35 primes"}


def cpu_baseline(args, budget_s=20.0, kind=0):
    """The CPU arm.  The reference ships no executor, so the layer
    is run by the oracle (oracle/, a scalar C++ restatement of the reference's
    semantics, all host threads) op kind by op kind: every Rot / Relin / CMult /
    Rescale / CAdd / PMult / Boot op of the reference-emitted op list is costed
    at its own level from a MEASURED single-op sample at that level (one lane
    per host thread; lanes are independent, so an op's cost is per-lane cost x
    its lane count).  Levels not sampled are interpolated by a least-squares
    fit through the sampled ones (quadratic for key switching, linear for the
    element-wise kinds).  Reported: the sampled seconds, the extrapolated layer
    seconds and their ratio, plus the reference's own NTT timed beside it."""
    from oracle_py import Oracle
    threads = os.cpu_count() or 1
    ops, src = _layer_ops(args.tokens)
    o = Oracle(N_LOG, threads=threads)
    lanes = threads
    samples = {}
    measured = 0.0
    with tempfile.TemporaryDirectory() as d:
        def run(kind, level, lanes_, **kw):
            mp = os.path.join(d, f"{kind}_{level}.heops")
            _mini_graph(mp, kind, level, lanes_, **kw)
            base = os.path.join(d, f"none_{level}.heops")
            _mini_graph(base, "none", level, max(lanes_, kw.get("c_in", 0)))
            t0 = time.time()
            o.run_graph(base)  # input materialisation only
            t_in = time.time() - t0
            t0 = time.time()
            o.run_graph(mp)
            dt = time.time() - t0
            return max(dt - t_in, 1e-6), dt + t_in

        _mini_graph(os.path.join(d, "warm.heops"), "rescale", 35, 1)
        o.run_graph(os.path.join(d, "warm.heops"))  # NTT tables of the main chain (not timed)
        plan = [("rot", lv) for lv in (2, 17, 30, 34, 35)] + \
               [("relin", lv) for lv in (3, 9, 17, 25, 34)] + \
               [("cmult", lv) for lv in (3, 17, 34)] + [("rescale", lv) for lv in (3, 17, 35)] + \
               [("cadd", lv) for lv in (17, 34)] + [("boot", 1)] + [("pmult", lv) for lv in (2, 17, 35)]
        for kind_, lv in plan:
            if kind_ == "pmult":
                t, w = run("pmult", lv, 1, c_in=12, c_out=lanes)
                samples.setdefault("pmult", []).append((lv, t / (12 * lanes)))  # per lane-product
            else:
                t, w = run(kind_, lv, lanes)
                samples.setdefault(kind_, []).append((lv, t / lanes))  # per lane
            measured += w
        # relin sample = CMult + Relin: subtract the CMult at the same level
        cm = _fit(samples["cmult"], 1)
        samples["relin"] = [(lv, max(t - cm(lv), 1e-9)) for lv, t in samples["relin"]]
    fits = {"rot": _fit(samples["rot"], 2), "relin": _fit(samples["relin"], 2), "cmult": _fit(samples["cmult"], 1),
            "rescale": _fit(samples["rescale"], 1), "cadd": _fit(samples["cadd"], 1),
            "boot": _fit(samples["boot"], 0), "pmult": _fit(samples["pmult"], 1)}
    exact = {k: dict(v) for k, v in samples.items()}
    names = {2: "cadd", 3: "pmult", 4: "cmult", 5: "rot", 6: "relin", 7: "rescale", 8: "boot"}
    value = 0.0
    for f in ops:
        k, nl, work, lv = int(f[2]), int(f[6]), int(f[10]), int(f[11])
        nm = names.get(k)
        if nm is None:
            continue
        per = exact.get(nm, {}).get(lv)
        per = fits[nm](lv) if per is None else per
        value += per * (work if nm == "pmult" else nl)
    ntt = reference_ntt(threads)
    return {"value": value, "unit": "s/layer", "cores": threads, "kind": "port",
            "measured_s": round(measured, 2), "extrapolation": round(value / max(measured, 1e-9), 1),
            "sample": (f"oracle (CPU port of the reference semantics, {threads} threads, one lane per thread): "
                       f"{len(plan)} single HE ops timed at the layer's own levels (Rot l=2/17/30/34/35, Relin "
                       f"3..34, CMult, Rescale, CAdd, Boot, PMult 12x{lanes}); every op of the reference-emitted "
                       f"op list ({os.path.basename(src)}, {len(ops)} ops) costed as per-lane time at its level x "
                       f"its lanes (unsampled levels: least-squares fit)"),
            "reference_ntt": ntt}


# ---------------------------------------------------------------------------
def run_aegis(args):
    import torch
    from paper_2604_03425_b200 import Context
    dist, rank, ws, local = dist_init(args.gpus)
    torch.cuda.set_device(local)
    c = Context(log_n=N_LOG, device=local)
    g = c.graph(kind=0, tokens=args.tokens, layers=args.layers)
    tg_total = -(-args.tokens // ((1 << N_LOG) // 2 // 64))
    win = None
    if ws > 1:
        from paper_2604_03425_b200.dist import P2pReducer, attach_p2p, make_reducer, token_group_comms
        if ws > tg_total and os.environ.get("AEGIS_STAGGER", "1") == "1":
            # this rank's staggered diagonal order from the Aegis plan (bit-identical)
            g = g.in_plan_order(g.plan(ws, reorder=True), rank)
        g.set_shard(ws, rank)
        if os.environ.get("AEGIS_MATMUL_MODES") == "reference":  # gather where the reference's byte rule does
            g.set_matmul_modes(True)
        groups, m = token_group_comms(ws, tg_total)
        if m > 1:
            # default: the executor's own data plane (comm stream, peer-memory windows, device flags);
            # AEGIS_REDUCER=hook: the host-synchronised peer-memory reducer; =nccl: ncclReduceScatter
            mode = os.environ.get("AEGIS_REDUCER", "device")
            if mode == "device":
                win = attach_p2p(c, g, groups, rank % m)
            if win is None:
                g.set_reducer(make_reducer(groups, rank % m) if mode == "nccl" else P2pReducer(c, groups, rank % m))
    c.keys_generate(g.key_ids())
    c.sync()
    st = torch.cuda.ExternalStream(c.stream)

    def barrier():
        c.sync()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        g.run()
    barrier()
    l0 = c.launch_count()
    # the step's dominant kernel (cfwd_a) is timed live inside the
    # timed region: CUDA events bracket each of its launches on the library stream
    c.probe_start(TOP_KERNEL)
    with Clocks(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.steps):
            g.run()
        e1.record(st)
        e1.synchronize()
    barrier()
    probe = c.probe_read()
    c.probe_start(None)
    launches = (c.launch_count() - l0) // max(1, args.steps)
    peak_bytes = int(g.peak_bytes())
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- e2e: through the public API with host buffers (H2D input, D2H output) ----
    e2e_ms, h2d, d2h = end_to_end(c, g, args, st, barrier) if not args.no_e2e else (float("nan"), 0, 0)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- separately reported variant: dead-lane elimination (final bundle bit-identical) ----
    dce = None
    if not args.no_dce:
        try:
            g.set_dce(True)
            g.run()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.run()
            e1.record(st)
            e1.synchronize()
            dms = e0.elapsed_time(e1)
        except Exception as exc:  # the variant must never cost the headline line
            dms = float("nan")
            dce = {"error": str(exc)[:200]}
        g.set_dce(False)
        if dist:
            t = torch.tensor([dms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dms = float(t.item())
    if not args.no_dce and dce is None:
        dce = {"value": dms / 1e3, "unit": "s/layer", "steps": 1,
               "note": "variant, not the headline: output lanes no later op reads (72.9% of the rotated lanes at "
                       "T=2048, SURVEY Appendix B.5) are not computed; the layer output bundle is bit-identical "
                       "(tests/test_gpu_parity.py::test_dead_lane_elimination_keeps_final_bundle)"}

    # ---- the other single-GPU BASELINE configs (parity cases, reported for reference) ----
    others = None
    if ws == 1 and not args.no_configs:
        others = {name: time_config(c, st, kind, tokens)
                  for name, kind, tokens in (("config1_ffn_T128", 1, 128), ("config2_layer_T512", 0, 512))}

    # ---- the Aegis plan of this layer at 8 devices (host-side; events, bytes) ----
    plan = None
    try:
        ps = g.plan(max(ws, 8)).summary()
        plan = {k: ps[k] for k in ("world", "token_groups", "ranks_per_group", "events", "events_executed",
                                   "bytes_total", "bytes_ffn", "bytes_attention", "bytes_reference_rule",
                                   "matmuls_gather_chosen")}
        plan["comm_bytes_this_rank_last_run"] = g.comm_bytes()
        plan["note"] = ("PCMM reduce-scatter per sub-tensor when a token group spans several devices; attention "
                        "is lane-local under the reference's pairing (no collective); bytes_reference_rule = "
                        "the volume if each matmul used the mode comm_plan.hpp:226-238 picks")
    except Exception as exc:
        plan = {"error": str(exc)[:200]}

    # ---- stored-plaintext PCMM variant (config 2 layer; weights written to / read from HBM) ----
    stored = None
    if ws == 1 and not args.no_configs:
        stored = time_config(c, st, 0, 512, stored=True)

    # ---- roofline of the step's dominant kernel (timed live in the step) + the NTT metric ----
    roof = step_roofline(probe, ms, args.steps, g)
    roof["ntt"] = ntt_roofline(c, st)
    out = None
    if rank == 0:
        cpu = cpu_baseline(args, budget_s=args.cpu_budget) if (ws == 1 and not args.no_cpu) else None
        out = {
            "metric": METRIC, "value": ms / 1e3, "unit": "s/layer", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64 (RNS residues mod 43-48-bit primes)", "data": "synthetic",
            "config": {"workload": f"BERT-base encoder layer (block 0 of the reference op sequence), "
                                   f"{args.tokens} tokens, CKKS N=2^16, L=35, |P|=4, s_tok=64",
                       "tokens": args.tokens, "layers": args.layers, "ring_degree": 1 << N_LOG,
                       "parallelism": f"token-group shards x{ws}",
                       "l2": "inputs > L2 (working set of every op >> 126 MB)"},
            "e2e": {"value": e2e_ms / 1e3, "unit": "s/layer", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "roofline": roof,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "peak_device_bytes": peak_bytes,
            "dce_variant": dce,
            "other_configs": others,
            "stored_weights_variant": stored,
            "plan": plan,
        }
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        if win is not None:
            g.set_p2p(None)
            win.close()
        dist.destroy_process_group()


def time_config(c, st, kind, tokens, stored=False):
    """One warm + one timed run of another BASELINE config on this context
    (reported for reference; a failure here never costs the headline line).
    stored: the PCMM weights are written to HBM by the Encode ops and read by
    the PMult kernel (SURVEY §8(d) stored-plaintext variant)."""
    import torch
    try:
        go = c.graph(kind=kind, tokens=tokens, layers=1)
        go.set_stored_weights(stored)
        c.keys_generate(go.key_ids())
        go.run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        go.run()
        e1.record(st)
        e1.synchronize()
        go.free()
        r = {"value": e0.elapsed_time(e1) / 1e3, "unit": "s/layer", "steps": 1}
        if stored:
            r["workload"] = f"config-{'2' if tokens == 512 else '?'} layer, T={tokens}, stored weights"
        return r
    except Exception as exc:
        return {"error": str(exc)[:200]}


def end_to_end(c, g, args, st, barrier):
    """Same layer through the C-ABI with host buffers: pinned H2D of the input
    ciphertexts and D2H of the layer output inside the timed region."""
    import torch
    in_words, out_words = g.io_words()
    hin = torch.empty(in_words, dtype=torch.int64, pin_memory=True)
    hout = torch.empty(out_words, dtype=torch.int64, pin_memory=True)
    g.fill_host_inputs(hin)
    steps = max(1, min(args.steps, 2))
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        g.run_host(hin.data_ptr(), in_words, hout.data_ptr(), out_words)
    e1.record(st)
    e1.synchronize()
    h2d, d2h = g.io_bytes()  # bytes actually copied by the last run (owned lanes only when sharded)
    return e0.elapsed_time(e1) / steps, h2d, d2h


TOP_KERNEL = "cfwd_a"


def step_roofline(probe, ms, steps, g):
    """roofline of the step's top kernel from the live probe: algorithmic bytes
    (DESIGN.md §3 per-launch model: k prepared source limbs + the overflow row
    read once per lane, every target limb written once) / its summed device
    time, against the measured HBM copy bandwidth; `traffic` and the pipe
    utilisations come from one ncu --set full capture of the same kernel
    (profiles/r02_cfwd_a_full.json).  `layer` = SURVEY §8(d) algorithmic bytes
    of the whole replayed op list / step time."""
    from paper_2604_03425_b200.costs import graph_bytes
    pk = peaks()
    n, pms, pbytes = probe
    out = {"kernel": "cfwd_a<k,2> (exact basis conversion fused with NTT pass A; ModUp / ModDown / rescale "
                     "targets, DESIGN.md §3.3)", "bound": "hbm", "unit": "GB/s",
           "peak": pk.get("hbm_gbs"), "peak_source": "measured" if not pk.get("_fallback") else "fallback"}
    if n and pms > 0:
        ach = pbytes / (pms / 1e3) / 1e9
        out.update({"achieved": ach, "frac": ach / pk.get("hbm_gbs"), "launches_per_step": n / max(1, steps),
                    "avg_launch_us": pms * 1e3 / n, "alg_bytes_per_launch": pbytes / n,
                    "share_of_step": pms / (ms * max(1, steps))})
    else:
        out.update({"achieved": None, "frac": None})
    out["traffic"] = None
    try:
        # DRAM bytes / algorithmic bytes of every cfwd_a launch of one layer (ncu + the probe,
        # same run, profiles/r02_cfwd_a_full.json), applied to this step's per-launch bytes
        prof = json.load(open(os.path.join(ROOT, "profiles", "r02_cfwd_a_full.json")))
        if out.get("alg_bytes_per_launch"):
            out["traffic"] = prof["traffic_over_algorithmic"] * out["alg_bytes_per_launch"]
        out["traffic_over_algorithmic"] = prof["traffic_over_algorithmic"]
        out["ncu_full"] = prof["full_capture_T2048_launch_3000"]
    except Exception:
        pass
    _, _, ops, _ = g.export()
    total, _ = graph_bytes(ops, 1 << N_LOG)
    ach = total / (ms / 1e3) / 1e9
    out["layer"] = {"alg_bytes": total, "achieved": ach, "frac": ach / pk.get("hbm_gbs"),
                    "model": "SURVEY §8(d) per-op bytes summed over the replayed op list "
                             "(paper_2604_03425_b200/costs.py)"}
    return out


def ntt_roofline(c, st):
    """Forward NTT of 48 lanes x 17 limbs (the FFN1 rotation source shape) --
    the kernel class that dominates the layer's key switching."""
    import torch
    pk = peaks()
    b = c.bundle(48, 1, 17)
    b.fill_input(3)
    for _ in range(3):
        c.ntt(b)
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        c.ntt(b)
    e1.record(st)
    e1.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    limbs = 48 * 17
    alg = 2 * 8 * (1 << N_LOG) * limbs
    try:
        fp64_peak = json.load(open(os.path.join(ROOT, "profiles", "r02_pipe_peaks.json")))["dfma_tfma_s"]
    except Exception:
        fp64_peak = 148 * 64 * 1.965e9 / 1e12
    achieved = alg / t / 1e9
    b.free()
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ntt_traffic.json")))["bytes_per_launch"]
    except Exception:
        pass
    return {"kernel": "NTT v2 fwd_a + fwd_b (forward, 2 passes, 816 limbs of N=2^16)", "bound": "hbm",
            "achieved": achieved, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
            "frac": achieved / pk.get("hbm_gbs"), "traffic": traffic,
            "peak_source": "measured" if not pk.get("_fallback") else "fallback",
            "ns_per_limb": t / limbs * 1e9,
            # the binding resource of the 64-bit NTT on B200 is the FP64 pipe:
            # 8 DFMA-pipe instructions per butterfly, 16 x 32768 butterflies per limb, plus the
            # u64<->f64 conversions (~7 per coefficient); peak = 148 SMs x 64 lanes x max SM clock
            "fp64_pipe": {"achieved_tops": limbs * (16 * 32768 * 8 + 7 * 65536) / t / 1e12,
                          "peak_tops": fp64_peak,
                          "peak_source": "measured DFMA rate (tools/probe/imad_peak.cu, profiles/r02_pipe_peaks.json)",
                          "frac": limbs * (16 * 32768 * 8 + 7 * 65536) / t / (fp64_peak * 1e12)}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="aegis", choices=["aegis", "reference"])
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dce", action="store_true", help="skip the dead-lane-elimination variant")
    ap.add_argument("--no-configs", action="store_true", help="skip the config-1/2 reference timings")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer (e2e) run (profiling only)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_aegis(args)


if __name__ == "__main__":
    main()
