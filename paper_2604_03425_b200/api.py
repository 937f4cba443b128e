"""Python host API of libaegis, mirroring the reference's operator surface.

Reference mapping (proj/include/heplan/):
  Context      -- one GPU + CkksProfile (ckks.hpp:21-46) + keys/tables
  Bundle       -- CtBundle (he_ir.hpp:57-74): [lane][comp][limb][N] u64 on device
  Context.rot / relin / rescale / boot / cmult / cadd / pmult_acc
               -- HeOpKind evaluator ops (he_ir.hpp:21-31), bundled form
  Context.ntt / automorphism / basis_convert / keyswitch
               -- PolyOpKind instructions (poly_ir.hpp:23-32)
  Graph        -- HeOpGraph from lower_app_to_he (he_ir.hpp:683) + executor
                  (SPEC.md:407-415 exec_sequential)
Errors raise the reference's exception types: EINVAL -> ValueError
(std::invalid_argument), ELOGIC -> RuntimeError subclass LogicError
(std::logic_error), CUDA/NCCL/OOM -> AegisError.
"""
import ctypes

import numpy as np

from . import _lib as L

BERT_PARAMS = dict(log_n=16, chain_length=35, special_primes=4, bootstrap_level=14)
SEED_INPUT = 0xAE615
SEED_WEIGHT = 0xAE616
SEED_KEY = 0xAE617


class AegisError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"aegis error {code}: {msg}")
        self.code = code


class LogicError(AegisError):
    pass


def _raise(code, msg):
    if code == L.AEGIS_EINVAL:
        raise ValueError(msg)
    if code == L.AEGIS_ELOGIC:
        raise LogicError(code, msg)
    raise AegisError(code, msg)


def _u64p(a):
    return a.ctypes.data_as(L.u64p)


def _u32arr(xs):
    a = np.ascontiguousarray(np.asarray(xs, dtype=np.uint32))
    return a, a.ctypes.data_as(L.u32p)


class Bundle:
    def __init__(self, ctx, handle, lanes, comps, level):
        self.ctx, self.h, self.lanes, self.comps, self.level = ctx, handle, lanes, comps, level

    @property
    def shape(self):
        return (self.lanes, self.comps, self.level, self.ctx.n)

    def upload(self, arr):
        a = np.ascontiguousarray(arr, dtype=np.uint64)
        if a.shape != self.shape:
            raise ValueError(f"upload shape {a.shape} != {self.shape}")
        self.ctx._call("aegis_bundle_upload", self.h, _u64p(a), a.size)

    def download(self):
        a = np.empty(self.shape, dtype=np.uint64)
        self.ctx._call("aegis_bundle_download", self.h, _u64p(a), a.size)
        return a

    def hash(self, comps=None, level=None):
        out = ctypes.c_uint64()
        self.ctx._call("aegis_bundle_hash", self.h, self.comps if comps is None else comps,
                       self.level if level is None else level, ctypes.byref(out))
        return out.value

    def fill_input(self, bundle_id):
        self.ctx._call("aegis_bundle_fill_input", self.h, bundle_id)

    def device_ptr(self):
        p = ctypes.c_uint64()
        L.load().aegis_bundle_info(self.h, None, None, None, ctypes.byref(p))
        return p.value

    def free(self):
        if self.h:
            self.ctx._call("aegis_bundle_free", self.h)
            self.h = None


class Context:
    """One B200 running the CKKS hot path (a CkksProfile plus device state)."""

    def __init__(self, log_n=16, chain_length=35, bootstrap_level=14, device=0,
                 seed_input=SEED_INPUT, seed_weight=SEED_WEIGHT, seed_key=SEED_KEY):
        self.lib = L.load()
        self.params = L.AegisParams(log_n, chain_length, 4, bootstrap_level, seed_input,
                                    seed_weight, seed_key)
        h = ctypes.c_void_p()
        rc = self.lib.aegis_ctx_create(ctypes.byref(self.params), device, ctypes.byref(h))
        if rc != L.AEGIS_OK:
            _raise(rc, self.lib.aegis_last_error(None).decode())
        self.h = h
        self.n = 1 << log_n
        self.log_n = log_n
        self.chain = chain_length

    def _call(self, name, *args):
        rc = getattr(self.lib, name)(self.h, *args)
        if rc != L.AEGIS_OK:
            _raise(rc, self.lib.aegis_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.aegis_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- misc --
    def prime(self, ext):
        return self.lib.aegis_prime(self.h, ext)

    def sync(self):
        self._call("aegis_sync")

    @property
    def stream(self):
        return self.lib.aegis_stream_compute(self.h)

    def launch_count(self):
        return self.lib.aegis_launch_count(self.h)

    PROBE = {"cfwd_a": 1, "fwd_b_fin": 2, "fwd_b_km": 3}

    def probe_start(self, kernel):
        """Bracket every launch of `kernel` (cfwd_a | fwd_b_fin | fwd_b_km | None) with CUDA events."""
        self._call("aegis_probe_start", self.PROBE[kernel] if kernel else 0)

    def probe_read(self):
        """-> (launches, device ms summed over them, algorithmic bytes summed over them)"""
        n, ms, b = ctypes.c_uint64(), ctypes.c_double(), ctypes.c_double()
        self._call("aegis_probe_read", ctypes.byref(n), ctypes.byref(ms), ctypes.byref(b))
        return n.value, ms.value, b.value

    # -- peer-memory windows (csrc/p2p.cu) --
    def p2p_window(self, nbytes):
        """A window of `nbytes` data bytes; returns a P2pWindow (with .handle, its 64-byte IPC handle)."""
        raw = (ctypes.c_char * 64)()
        h = ctypes.c_void_p()
        self._call("aegis_p2p_create", nbytes, ctypes.cast(raw, ctypes.c_void_p), ctypes.byref(h))
        return P2pWindow(self, h, bytes(raw), nbytes)

    # -- bundles / keys --
    def bundle(self, lanes, comps, level):
        h = ctypes.c_void_p()
        self._call("aegis_bundle_alloc", lanes, comps, level, ctypes.byref(h))
        return Bundle(self, h, lanes, comps, level)

    def bundle_load(self, path):
        """A bundle from an aegis store file (csrc/store.cu), streamed to the device and hash-checked."""
        h = ctypes.c_void_p()
        self._call("aegis_bundle_load", str(path).encode(), ctypes.byref(h))
        lanes, comps, level = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        self.lib.aegis_bundle_info(h, ctypes.byref(lanes), ctypes.byref(comps), ctypes.byref(level), None)
        return Bundle(self, h, lanes.value, comps.value, level.value)

    def bundle_save(self, b, path):
        self._call("aegis_bundle_save", b.h, str(path).encode())

    def keys_save(self, key_id, path):
        self._call("aegis_keys_save", key_id, str(path).encode())

    def keys_load(self, key_id, path):
        self._call("aegis_keys_load", key_id, str(path).encode())

    def keys_generate(self, ids):
        a = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64))
        self._call("aegis_keys_generate", _u64p(a), len(a))

    def keys_upload(self, key_id, key, coeff_domain=True):
        """Caller-supplied key, uint64 [digits][2][chain + 4][N] (include/aegis.h)."""
        a = np.ascontiguousarray(key, dtype=np.uint64)
        if a.shape != self.key_shape():
            raise ValueError(f"key shape {a.shape} != {self.key_shape()}")
        self._call("aegis_keys_upload", key_id, _u64p(a), a.size, 1 if coeff_domain else 0)

    def key_shape(self):
        """(digits, 2, chain + 4, N) of one key-switching key."""
        return (-(-self.chain // 4), 2, self.chain + 4, 1 << self.log_n)

    # -- polynomial instructions --
    def ntt(self, b, lane=0, lanes=None, lo=0, hi=None, inverse=False):
        self._call("aegis_ntt", b.h, lane, b.lanes if lanes is None else lanes, lo,
                   b.level - 1 if hi is None else hi, 1 if inverse else 0)

    def automorphism(self, out, inp, galois, level=None, lane=0, lanes=None):
        self._call("aegis_automorphism", out.h, inp.h, lane, inp.lanes if lanes is None else lanes,
                   inp.level if level is None else level, galois)

    def basis_convert(self, out, inp, src_ext, src_limb, dst_ext, dst_limb):
        a, pa = _u32arr(src_ext)
        b, pb = _u32arr(src_limb)
        c, pc = _u32arr(dst_ext)
        d, pd = _u32arr(dst_limb)
        self._call("aegis_basis_convert", out.h, inp.h, pa, pb, len(a), pc, pd, len(c))

    def keyswitch(self, out, inp, comp, level, key_id):
        self._call("aegis_keyswitch", out.h, inp.h, comp, level, key_id)

    # -- HE operators --
    def rot(self, out, inp, offset, level, out_lane=0, in_lane=0, lanes=None):
        self._call("aegis_rot", out.h, out_lane, inp.h, in_lane,
                   inp.lanes if lanes is None else lanes, level, offset)

    def rot_hoisted(self, outs, inp, offsets, level, out_lanes=None, in_lane=0, lanes=None):
        """Rotations of one source by several offsets, ModUp shared (bit-identical to separate rot calls)."""
        k = len(offsets)
        hs = (ctypes.c_void_p * k)(*[o.h for o in outs])
        ol = (ctypes.c_uint32 * k)(*(out_lanes or [0] * k))
        of = (ctypes.c_int * k)(*offsets)
        self._call("aegis_rot_hoisted", hs, ol, of, k, inp.h, in_lane, inp.lanes if lanes is None else lanes, level)

    def limb_op(self, opcode, out, a=None, b=None, lo=0, hi=None, lanes=None, out_lane=0, a_slice=None,
                b_slice=None, param=0):
        """kLimbMulAdd with LimbOpcode `opcode` (_lib.LIMB_*) on limbs [lo, hi] (poly_ir.hpp:49-58, 192-213)."""
        lanes = out.lanes if lanes is None else lanes
        al, ac = a_slice or ((0, a.lanes) if a is not None else (0, 0))
        bl, bc = b_slice or ((0, b.lanes) if b is not None else (0, 0))
        self._call("aegis_limb_op", opcode, out.h, out_lane, lanes, a.h if a is not None else None, al, ac,
                   b.h if b is not None else None, bl, bc, lo, out.level - 1 if hi is None else hi, param)

    def limb_drop(self, out, inp, level, mode=0, out_lane=0, in_lane=0, lanes=None):
        """kLimbDrop (poly_ir.hpp:341-354): mode 0 truncates, 3 (kRescaleTail) rescales."""
        self._call("aegis_limb_drop", out.h, out_lane, inp.h, in_lane, inp.lanes if lanes is None else lanes,
                   level, mode)

    def padd(self, out, ct, pt, level, lanes=None, ct_slice=None, pt_slice=None, out_lane=0):
        lanes = out.lanes if lanes is None else lanes
        cl, cc = ct_slice or (0, ct.lanes)
        pl, pc = pt_slice or (0, pt.lanes)
        self._call("aegis_padd", out.h, out_lane, lanes, ct.h, cl, cc, pt.h, pl, pc, level)

    def encode(self, pt, weight_bundle, level, lane=0, lanes=None):
        """kEncode: the kGenerate weights of bundle id `weight_bundle` into a 1-component bundle."""
        self._call("aegis_encode", pt.h, lane, pt.lanes if lanes is None else lanes, level, weight_bundle)

    def relin(self, b, level, lane=0, lanes=None):
        self._call("aegis_relin", b.h, lane, b.lanes if lanes is None else lanes, level)

    def rescale(self, out, inp, level, out_lane=0, in_lane=0, lanes=None):
        self._call("aegis_rescale", out.h, out_lane, inp.h, in_lane,
                   inp.lanes if lanes is None else lanes, level)

    def boot(self, out, inp, level, out_level, out_lane=0, in_lane=0, lanes=None):
        self._call("aegis_boot", out.h, out_lane, inp.h, in_lane,
                   inp.lanes if lanes is None else lanes, level, out_level)

    def cmult(self, out, a, b, level, lanes=None, a_slice=None, b_slice=None, out_lane=0):
        lanes = out.lanes if lanes is None else lanes
        al, ac = a_slice or (0, a.lanes)
        bl, bc = b_slice or (0, b.lanes)
        self._call("aegis_cmult", out.h, out_lane, lanes, a.h, al, ac, b.h, bl, bc, level)

    def cadd(self, out, a, b, level, accumulate=False, lanes=None, a_slice=None, b_slice=None,
             out_lane=0):
        lanes = out.lanes if lanes is None else lanes
        al, ac = a_slice or (0, a.lanes)
        if b is None:
            bh, bl, bc = None, 0, 0
        else:
            bh = b.h
            bl, bc = b_slice or (0, b.lanes)
        self._call("aegis_cadd", out.h, out_lane, lanes, a.h, al, ac, bh, bl, bc, level,
                   1 if accumulate else 0)

    def pmult_acc(self, acc, x, weight_bundle, weight_lanes, level, chunk_period=0):
        self._call("aegis_pmult_acc", acc.h, 0, acc.lanes, chunk_period, x.h, 0, x.lanes,
                   weight_bundle, weight_lanes, level)

    def pmult_acc_stored(self, acc, x, w, level, chunk_period=0, w_slice=None):
        wl, wc = w_slice or (0, w.lanes)
        self._call("aegis_pmult_acc_stored", acc.h, 0, acc.lanes, chunk_period, x.h, 0, x.lanes, w.h, wl, wc, level)

    # -- graphs --
    def graph(self, kind=0, tokens=128, layers=1, model_dim=768, ffn_dim=3072, head_dim=64,
              slots_per_token=64):
        m = L.AegisModel(kind, layers, model_dim, ffn_dim, head_dim, slots_per_token, tokens)
        h = ctypes.c_void_p()
        self._call("aegis_graph_build", ctypes.byref(m), ctypes.byref(h))
        return Graph(self.lib, h, self)

    def load_graph(self, path):
        h = ctypes.c_void_p()
        self._call("aegis_graph_load", str(path).encode(), ctypes.byref(h))
        return Graph(self.lib, h, self)

    def graph_from_ops(self, meta, bundles, ops, inputs):
        """In-memory HeOpGraph ingest (aegis_graph_from_ops): see graph_from_ops()."""
        g = graph_from_ops(meta, bundles, ops, inputs)
        g.ctx = self
        return g


def graph_from_ops(meta, bundles, ops, inputs):
    """Build a graph from descriptor arrays (_lib.AegisGraphMeta, AegisBundleDesc[],
    AegisOpDesc[], bundle ids) with no text round trip; no device needed."""
    lib = L.load()
    nb, no, ni = len(bundles), len(ops), len(inputs)
    barr = (L.AegisBundleDesc * max(nb, 1))(*bundles)
    oarr = (L.AegisOpDesc * max(no, 1))(*ops)
    iarr = (ctypes.c_uint32 * max(ni, 1))(*inputs)
    h = ctypes.c_void_p()
    rc = lib.aegis_graph_from_ops(ctypes.byref(meta), barr, nb, oarr, no, iarr, ni, ctypes.byref(h))
    if rc != L.AEGIS_OK:
        _raise(rc, lib.aegis_last_error(None).decode())
    return Graph(lib, h, None)


def plan_graph(log_n=16, chain_length=35, bootstrap_level=14, kind=0, tokens=128, layers=1,
               model_dim=768, ffn_dim=3072, head_dim=64, slots_per_token=64):
    """Lower a model to its HeOpGraph without a GPU (the layer drivers are host code)."""
    lib = L.load()
    p = L.AegisParams(log_n, chain_length, 4, bootstrap_level, 0, 0, 0)
    m = L.AegisModel(kind, layers, model_dim, ffn_dim, head_dim, slots_per_token, tokens)
    h = ctypes.c_void_p()
    rc = lib.aegis_graph_build_params(ctypes.byref(p), ctypes.byref(m), ctypes.byref(h))
    if rc != L.AEGIS_OK:
        _raise(rc, lib.aegis_last_error(None).decode())
    return Graph(lib, h, None)


class Graph:
    def __init__(self, lib, h, ctx):
        self.lib, self.h, self.ctx = lib, h, ctx

    def info(self):
        o, b = ctypes.c_uint64(), ctypes.c_uint64()
        self.lib.aegis_graph_info(self.h, ctypes.byref(o), ctypes.byref(b))
        return o.value, b.value

    def export(self):
        """-> (meta, [AegisBundleDesc], [AegisOpDesc], [input bundle ids]) (aegis_graph_export)."""
        nops, nb = self.info()
        ni = ctypes.c_uint32()
        self.lib.aegis_graph_export(self.h, None, 0, None, 0, None, 0, ctypes.byref(ni), None)
        barr = (L.AegisBundleDesc * max(nb, 1))()
        oarr = (L.AegisOpDesc * max(nops, 1))()
        iarr = (ctypes.c_uint32 * max(ni.value, 1))()
        meta = L.AegisGraphMeta()
        rc = self.lib.aegis_graph_export(self.h, barr, nb, oarr, nops, iarr, ni.value, None, ctypes.byref(meta))
        if rc:
            _raise(rc, self.lib.aegis_last_error(None).decode())
        return meta, list(barr)[:nb], list(oarr)[:nops], list(iarr)[:ni.value]

    def dump(self, path):
        rc = self.lib.aegis_graph_dump(self.h, str(path).encode())
        if rc:
            raise ValueError(f"cannot dump graph to {path}")

    def key_ids(self):
        n = ctypes.c_uint32()
        self.lib.aegis_graph_key_ids(self.h, None, 0, ctypes.byref(n))
        a = np.zeros(n.value, dtype=np.uint64)
        self.lib.aegis_graph_key_ids(self.h, _u64p(a), n.value, ctypes.byref(n))
        return a

    def set_shard(self, world, rank):
        """Token-coherent lane ownership for rank `rank` of `world`."""
        rc = self.lib.aegis_graph_set_shard(self.h, world, rank)
        if rc:
            _raise(rc, self.lib.aegis_last_error(None).decode())

    def set_hash_group(self, group):
        """Unsharded run, hashes over the lanes of token group `group` only (-1: all)."""
        rc = self.lib.aegis_graph_set_hash_group(self.h, group)
        if rc:
            _raise(rc, self.lib.aegis_last_error(None).decode())

    def shard_info(self):
        v = [ctypes.c_uint32() for _ in range(5)]
        self.lib.aegis_graph_shard_info(self.h, *[ctypes.byref(x) for x in v])
        return dict(zip(["tg_total", "tg_lo", "tg_hi", "ranks_per_group", "part"], [x.value for x in v]))

    def owned_lanes(self, bundle, lanes):
        m = (ctypes.c_uint8 * lanes)()
        rc = self.lib.aegis_graph_owned_lanes(self.h, bundle, m, lanes)
        if rc:
            raise ValueError("bad bundle")
        return np.frombuffer(m, dtype=np.uint8).astype(bool)

    def set_reducer(self, fn):
        """fn(buf_ptr:int, words_per_rank:int, group:int) -> None; reduce-scatter
        (uint64 sum) of words_per_rank * m words at the device pointer."""
        def cb(user, buf, words, group):
            try:
                fn(buf, words, group)
                return 0
            except Exception as e:  # never let an exception cross the C boundary
                import sys
                print(f"aegis reducer failed: {e!r}", file=sys.stderr)
                return 1
        self._reducer = L.REDUCE_FN(cb)  # keep alive
        self.lib.aegis_graph_set_reducer(self.h, ctypes.cast(self._reducer, ctypes.c_void_p), None)

    def plan(self, world, reorder=True):
        """The Aegis execution plan on `world` devices (aegis_plan_build): a Plan."""
        h = ctypes.c_void_p()
        rc = self.lib.aegis_plan_build(self.h, world, 1 if reorder else 0, ctypes.byref(h))
        if rc:
            _raise(rc, self.lib.aegis_last_error(None).decode())
        return Plan(self.lib, h)

    def in_plan_order(self, plan, device):
        """This graph's ops in the order device `device` of `plan` runs them (bit-identical)."""
        h = ctypes.c_void_p()
        rc = self.lib.aegis_graph_from_plan(self.h, plan.h, device, ctypes.byref(h))
        if rc:
            _raise(rc, self.lib.aegis_last_error(None).decode())
        return Graph(self.lib, h, self.ctx)

    def comm_bytes(self):
        """Bytes this rank sent through PCMM exchanges in the last run."""
        v = ctypes.c_uint64()
        self.lib.aegis_graph_comm_bytes(self.h, ctypes.byref(v))
        return v.value

    def p2p_bytes(self):
        """Window bytes the device-synchronised PCMM exchange needs under the current shard (0: none)."""
        v = ctypes.c_uint64()
        rc = self.lib.aegis_graph_p2p_bytes(self.h, ctypes.byref(v))
        if rc:
            _raise(rc, self.lib.aegis_last_error(None).decode())
        return v.value

    def set_p2p(self, window):
        """Attach a p2p window (Context.p2p_window): sharded PCMM sums are exchanged on the comm
        stream with device-side flags; no reduce hook needed (None detaches)."""
        self._p2p = window  # keep alive while attached
        self.lib.aegis_graph_set_p2p(self.h, window.h if window is not None else None)

    def set_stored_weights(self, enable):
        """Stored-plaintext PCMM (weights written to HBM by the Encode ops, read by PMult)."""
        self.lib.aegis_graph_set_stored_weights(self.h, 1 if enable else 0)

    def set_matmul_modes(self, reference_rule):
        """1: each matmul gathers or reduces as the reference's byte rule picks (needs a p2p window)."""
        self.lib.aegis_graph_set_matmul_modes(self.h, 1 if reference_rule else 0)

    def set_fault(self, kind):
        """Fault injection (tests): 1 drops the PCMM exchange, 0 restores it."""
        rc = self.lib.aegis_graph_set_fault(self.h, kind)
        if rc:
            raise ValueError("bad fault kind")

    def set_hoisting(self, enable):
        self.lib.aegis_graph_set_hoisting(self.h, 1 if enable else 0)

    def set_wrap_defer(self, enable):
        """Wrapped accumulating CAdds summed at the operand width (bit-identical; default on)."""
        self.lib.aegis_graph_set_wrap_defer(self.h, 1 if enable else 0)

    def set_dce(self, enable):
        """Dead-lane elimination (separately reported variant; final bundle bit-identical)."""
        self.lib.aegis_graph_set_dce(self.h, 1 if enable else 0)

    def set_profiling(self, enable):
        self.lib.aegis_graph_set_profiling(self.h, 1 if enable else 0)

    def op_times(self):
        n = ctypes.c_uint64()
        self.lib.aegis_graph_op_times(self.h, None, 0, ctypes.byref(n))
        a = np.zeros(n.value, dtype=np.float32)
        self.lib.aegis_graph_op_times(self.h, a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), n.value,
                                      ctypes.byref(n))
        return a

    def comm_times(self):
        """Two-stream trace of the last profiled run: (start ms, end ms, bundle) per exchange."""
        n = ctypes.c_uint64()
        self.lib.aegis_graph_comm_times(self.h, None, 0, ctypes.byref(n))
        a = np.zeros(3 * max(1, n.value), dtype=np.float32)
        self.lib.aegis_graph_comm_times(self.h, a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), n.value,
                                        ctypes.byref(n))
        return [(float(a[3 * i]), float(a[3 * i + 1]), int(a[3 * i + 2])) for i in range(n.value)]

    def io_bytes(self):
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        self.lib.aegis_graph_io_bytes(self.h, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def run(self, max_ops=-1, hashes=False):
        if self.ctx is None:
            raise ValueError("graph was planned without a device context")
        nb = self.info()[1]
        if hashes:
            h = np.zeros(nb, dtype=np.uint64)
            self.ctx._call("aegis_graph_run", self.h, max_ops, _u64p(h), nb)
            return h
        self.ctx._call("aegis_graph_run", self.h, max_ops, None, 0)
        return None

    def io_words(self):
        i, o = ctypes.c_uint64(), ctypes.c_uint64()
        self.lib.aegis_graph_io_words(self.h, ctypes.byref(i), ctypes.byref(o))
        return i.value, o.value

    def fill_host_inputs(self, buf):
        """buf: any object with data_ptr() (e.g. a pinned torch tensor) or a numpy array."""
        ptr = buf.data_ptr() if hasattr(buf, "data_ptr") else buf.ctypes.data
        words = buf.numel() if hasattr(buf, "numel") else buf.size
        self.ctx._call("aegis_graph_host_inputs", self.h, ctypes.c_void_p(ptr), words)

    def run_host(self, in_ptr, in_words, out_ptr, out_words):
        """End-to-end run: inputs H2D from host memory, final bundle D2H."""
        self.ctx._call("aegis_graph_run_host", self.h, ctypes.c_void_p(in_ptr), in_words,
                       ctypes.c_void_p(out_ptr), out_words)

    def peak_bytes(self):
        return self.lib.aegis_graph_peak_bytes(self.h)

    def free(self):
        if self.h:
            self.lib.aegis_graph_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class P2pWindow:
    """A rank's peer-memory window (aegis_p2p_*); open it over its group with
    open_ipc (separate processes) or open_local (contexts of one process)."""

    def __init__(self, ctx, h, handle, nbytes):
        self.ctx, self.h, self.handle, self.nbytes = ctx, h, handle, nbytes

    def open_ipc(self, handles, self_rank):
        allh = ctypes.create_string_buffer(b"".join(handles), 64 * len(handles))
        self.ctx._call("aegis_p2p_open", self.h, ctypes.cast(allh, ctypes.c_void_p), len(handles), self_rank)

    def open_local(self, windows, self_rank):
        arr = (ctypes.c_void_p * len(windows))(*[w.h for w in windows])
        self.ctx._call("aegis_p2p_open_local", self.h, arr, len(windows), self_rank)

    def close(self):
        if self.h:
            self.ctx.lib.aegis_p2p_destroy(self.h)
            self.h = None


class Plan:
    """aegis_plan_* wrapper: summary(), events(), device(d), matmuls(), note."""
    CATEGORIES = ("ffn", "attention", "layernorm", "boot", "other")
    MODES = ("local", "gather_inputs", "reduce_outputs")

    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            if self.h:
                self.lib.aegis_plan_free(self.h)
        except Exception:
            pass

    def summary(self):
        s = L.AegisPlanSummary()
        self.lib.aegis_plan_summary_get(self.h, ctypes.byref(s))
        return {f: getattr(s, f) for f, _ in s._fields_ if f != "pad"}

    def _list(self, fn, typ, *pre):
        n = ctypes.c_uint64()
        getattr(self.lib, fn)(self.h, *pre, None, 0, ctypes.byref(n))
        arr = (typ * max(1, n.value))()
        getattr(self.lib, fn)(self.h, *pre, arr, n.value, ctypes.byref(n))
        return [{f: getattr(a, f) for f, _ in a._fields_} for a in list(arr)[:n.value]]

    def events(self):
        return self._list("aegis_plan_events", L.AegisPlanEvent)

    def device(self, d):
        return self._list("aegis_plan_device", L.AegisPlanInstr, d)

    def matmuls(self):
        return self._list("aegis_plan_matmuls", L.AegisPlanMatmul)

    @property
    def note(self):
        return (self.lib.aegis_plan_note(self.h) or b"").decode()
