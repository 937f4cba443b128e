"""ctypes binding of libaegis (include/aegis.h).

The shared library is built in-tree (paper_2604_03425_b200/libaegis.so) by
__graft_entry__.build().  There is deliberately no fallback: if the library is
missing, importing the product API raises immediately.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# AEGIS_LIB: an alternate build of the same library (dev A/B of kernel variants)
LIB_PATH = os.environ.get("AEGIS_LIB") or os.path.join(_HERE, "libaegis.so")

u32 = ctypes.c_uint32
u64 = ctypes.c_uint64
i64 = ctypes.c_int64
vp = ctypes.c_void_p
u64p = ctypes.POINTER(ctypes.c_uint64)
u32p = ctypes.POINTER(ctypes.c_uint32)

AEGIS_OK, AEGIS_EINVAL, AEGIS_ELOGIC, AEGIS_ECUDA, AEGIS_ENCCL, AEGIS_EOOM = range(6)


class AegisParams(ctypes.Structure):
    _fields_ = [("log_n", u32), ("chain_length", u32), ("special_primes", u32),
                ("bootstrap_level", u32), ("seed_input", u64), ("seed_weight", u64),
                ("seed_key", u64)]


class AegisModel(ctypes.Structure):
    _fields_ = [("kind", u32), ("layers", u32), ("model_dim", u32), ("ffn_dim", u32),
                ("head_dim", u32), ("slots_per_token", u32), ("tokens", u64)]


class AegisGraphMeta(ctypes.Structure):
    _fields_ = [("log_n", u32), ("chain_length", u32), ("bootstrap_level", u32), ("slots_per_token", u32),
                ("model_dim", u32), ("head_dim", u32), ("ffn_dim", u32), ("layers", u32), ("kind", u32),
                ("tokens", u64)]


class AegisBundleDesc(ctypes.Structure):
    _fields_ = [("lanes", u32), ("level", u32), ("components", u32), ("cls", u32), ("aggregation", u32),
                ("app_node", u32), ("chunk_period", u32), ("replicate_hint", u32), ("tag", ctypes.c_char_p)]


class AegisSlice(ctypes.Structure):
    _fields_ = [("bundle", u32), ("lane", u32), ("lane_count", u32)]


MAX_OP_INPUTS = 4


class AegisOpDesc(ctypes.Structure):
    _fields_ = [("kind", u32), ("accumulate", u32), ("aligned", u32), ("aggregation", u32),
                ("rot_offset", ctypes.c_int32), ("phase", ctypes.c_int32), ("out", AegisSlice),
                ("in_count", u32), ("ins", AegisSlice * MAX_OP_INPUTS), ("work", u64), ("use_level", u32),
                ("app_node", u32)]


class AegisPlanSummary(ctypes.Structure):
    _fields_ = [(f, u32) for f in ("world", "token_groups", "ranks_per_group", "reordered", "executable", "matmuls",
                                   "matmuls_gather_chosen", "pad")] + \
               [(f, u64) for f in ("events", "events_executed", "instrs_total", "bytes_total", "bytes_ffn",
                                   "bytes_attention", "bytes_layernorm", "bytes_boot", "bytes_other",
                                   "bytes_reference_rule")]


class AegisPlanEvent(ctypes.Structure):
    _fields_ = [(f, u32) for f in ("id", "kind", "semantic", "dev_lo", "dev_count", "bundle", "lane", "lane_count",
                                   "level", "category", "app_node", "he_op", "executed")] + \
               [("bytes_per_device", u64), ("bytes_total", u64)]


class AegisPlanInstr(ctypes.Structure):
    _fields_ = [("op", u32), ("lane", u32), ("lane_count", u32), ("flags", u32), ("wait_event", ctypes.c_int32)]


class AegisPlanMatmul(ctypes.Structure):
    _fields_ = [(f, u32) for f in ("app_node", "acc_bundle", "input_bundle", "ship_bundle", "chosen", "executed")] + \
               [("gather_bytes", u64), ("reduce_bytes", u64)]


# LimbOpcode (poly_ir.hpp:49-58) and PolyMode (:60-65) values of the C-ABI
LIMB_ADD, LIMB_SUB, LIMB_MUL, LIMB_MULACC, LIMB_ADDACC, LIMB_KEYMUL, LIMB_GENERATE = range(1, 8)
MODE_NONE, MODE_KEY_SWITCH, MODE_BOOT_RESET, MODE_RESCALE_TAIL = range(4)

# (name, restype, argtypes) for every function declared in include/aegis.h
SIGNATURES = [
    ("aegis_ctx_create", ctypes.c_int, [ctypes.POINTER(AegisParams), ctypes.c_int, ctypes.POINTER(vp)]),
    ("aegis_ctx_destroy", ctypes.c_int, [vp]),
    ("aegis_last_error", ctypes.c_char_p, [vp]),
    ("aegis_stream_compute", vp, [vp]),
    ("aegis_stream_comm", vp, [vp]),
    ("aegis_sync", ctypes.c_int, [vp]),
    ("aegis_prime", u64, [vp, u32]),
    ("aegis_launch_count", u64, [vp]),
    ("aegis_probe_start", ctypes.c_int, [vp, ctypes.c_int]),
    ("aegis_probe_read", ctypes.c_int, [vp, u64p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    ("aegis_ntt_impl", ctypes.c_int, [ctypes.c_int]),
    ("aegis_bundle_alloc", ctypes.c_int, [vp, u32, u32, u32, ctypes.POINTER(vp)]),
    ("aegis_bundle_free", ctypes.c_int, [vp, vp]),
    ("aegis_bundle_upload", ctypes.c_int, [vp, vp, u64p, u64]),
    ("aegis_bundle_download", ctypes.c_int, [vp, vp, u64p, u64]),
    ("aegis_bundle_info", ctypes.c_int, [vp, u32p, u32p, u32p, u64p]),
    ("aegis_bundle_fill_input", ctypes.c_int, [vp, vp, u32]),
    ("aegis_bundle_hash", ctypes.c_int, [vp, vp, u32, u32, u64p]),
    ("aegis_keys_generate", ctypes.c_int, [vp, u64p, u32]),
    ("aegis_keys_upload", ctypes.c_int, [vp, u64, u64p, u64, ctypes.c_int]),
    ("aegis_keys_bytes", ctypes.c_int, [vp, u64p]),
    ("aegis_bundle_save", ctypes.c_int, [vp, vp, ctypes.c_char_p]),
    ("aegis_bundle_load", ctypes.c_int, [vp, ctypes.c_char_p, ctypes.POINTER(vp)]),
    ("aegis_keys_save", ctypes.c_int, [vp, u64, ctypes.c_char_p]),
    ("aegis_keys_load", ctypes.c_int, [vp, u64, ctypes.c_char_p]),
    ("aegis_ntt", ctypes.c_int, [vp, vp, u32, u32, u32, u32, ctypes.c_int]),
    ("aegis_automorphism", ctypes.c_int, [vp, vp, vp, u32, u32, u32, u64]),
    ("aegis_basis_convert", ctypes.c_int, [vp, vp, vp, u32p, u32p, u32, u32p, u32p, u32]),
    ("aegis_keyswitch", ctypes.c_int, [vp, vp, vp, u32, u32, u64]),
    ("aegis_rot", ctypes.c_int, [vp, vp, u32, vp, u32, u32, u32, ctypes.c_int]),
    ("aegis_limb_op", ctypes.c_int, [vp, ctypes.c_int, vp, u32, u32, vp, u32, u32, vp, u32, u32, u32, u32, u64]),
    ("aegis_limb_drop", ctypes.c_int, [vp, vp, u32, vp, u32, u32, u32, ctypes.c_int]),
    ("aegis_rot_hoisted", ctypes.c_int, [vp, ctypes.POINTER(vp), u32p, ctypes.POINTER(ctypes.c_int), u32, vp, u32,
                                         u32, u32]),
    ("aegis_relin", ctypes.c_int, [vp, vp, u32, u32, u32]),
    ("aegis_padd", ctypes.c_int, [vp, vp, u32, u32, vp, u32, u32, vp, u32, u32, u32]),
    ("aegis_encode", ctypes.c_int, [vp, vp, u32, u32, u32, u32]),
    ("aegis_rescale", ctypes.c_int, [vp, vp, u32, vp, u32, u32, u32]),
    ("aegis_boot", ctypes.c_int, [vp, vp, u32, vp, u32, u32, u32, u32]),
    ("aegis_cmult", ctypes.c_int, [vp, vp, u32, u32, vp, u32, u32, vp, u32, u32, u32]),
    ("aegis_cadd", ctypes.c_int, [vp, vp, u32, u32, vp, u32, u32, vp, u32, u32, u32, ctypes.c_int]),
    ("aegis_pmult_acc", ctypes.c_int, [vp, vp, u32, u32, u32, vp, u32, u32, u32, u32, u32]),
    ("aegis_graph_build", ctypes.c_int, [vp, ctypes.POINTER(AegisModel), ctypes.POINTER(vp)]),
    ("aegis_graph_build_params", ctypes.c_int,
     [ctypes.POINTER(AegisParams), ctypes.POINTER(AegisModel), ctypes.POINTER(vp)]),
    ("aegis_graph_load", ctypes.c_int, [vp, ctypes.c_char_p, ctypes.POINTER(vp)]),
    ("aegis_graph_dump", ctypes.c_int, [vp, ctypes.c_char_p]),
    ("aegis_graph_info", ctypes.c_int, [vp, u64p, u64p]),
    ("aegis_graph_from_ops", ctypes.c_int,
     [ctypes.POINTER(AegisGraphMeta), ctypes.POINTER(AegisBundleDesc), u32, ctypes.POINTER(AegisOpDesc), u64, u32p,
      u32, ctypes.POINTER(vp)]),
    ("aegis_graph_export", ctypes.c_int,
     [vp, ctypes.POINTER(AegisBundleDesc), u32, ctypes.POINTER(AegisOpDesc), u64, u32p, u32, u32p,
      ctypes.POINTER(AegisGraphMeta)]),
    ("aegis_graph_set_shard", ctypes.c_int, [vp, u32, u32]),
    ("aegis_graph_set_hash_group", ctypes.c_int, [vp, ctypes.c_int32]),
    ("aegis_graph_set_reducer", ctypes.c_int, [vp, vp, vp]),
    ("aegis_plan_build", ctypes.c_int, [vp, u32, ctypes.c_int, ctypes.POINTER(vp)]),
    ("aegis_plan_summary_get", ctypes.c_int, [vp, ctypes.POINTER(AegisPlanSummary)]),
    ("aegis_plan_events", ctypes.c_int, [vp, ctypes.POINTER(AegisPlanEvent), u64, u64p]),
    ("aegis_plan_device", ctypes.c_int, [vp, u32, ctypes.POINTER(AegisPlanInstr), u64, u64p]),
    ("aegis_plan_matmuls", ctypes.c_int, [vp, ctypes.POINTER(AegisPlanMatmul), u64, u64p]),
    ("aegis_plan_note", ctypes.c_char_p, [vp]),
    ("aegis_graph_from_plan", ctypes.c_int, [vp, vp, u32, ctypes.POINTER(vp)]),
    ("aegis_plan_free", ctypes.c_int, [vp]),
    ("aegis_graph_comm_bytes", ctypes.c_int, [vp, u64p]),
    ("aegis_graph_owned_lanes", ctypes.c_int, [vp, u32, ctypes.POINTER(ctypes.c_uint8), u32]),
    ("aegis_graph_shard_info", ctypes.c_int, [vp, u32p, u32p, u32p, u32p, u32p]),
    ("aegis_graph_set_hoisting", ctypes.c_int, [vp, ctypes.c_int]),
    ("aegis_graph_set_dce", ctypes.c_int, [vp, ctypes.c_int]),
    ("aegis_graph_set_wrap_defer", ctypes.c_int, [vp, ctypes.c_int]),
    ("aegis_graph_set_profiling", ctypes.c_int, [vp, ctypes.c_int]),
    ("aegis_graph_op_times", ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_float), u64, u64p]),
    ("aegis_graph_comm_times", ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_float), u64, u64p]),
    ("aegis_graph_io_bytes", ctypes.c_int, [vp, u64p, u64p]),
    ("aegis_graph_run", ctypes.c_int, [vp, vp, i64, u64p, u64]),
    ("aegis_graph_io_words", ctypes.c_int, [vp, u64p, u64p]),
    ("aegis_graph_host_inputs", ctypes.c_int, [vp, vp, vp, u64]),
    ("aegis_graph_run_host", ctypes.c_int, [vp, vp, vp, u64, vp, u64]),
    ("aegis_graph_key_ids", ctypes.c_int, [vp, u64p, u32, u32p]),
    ("aegis_graph_free", ctypes.c_int, [vp]),
    ("aegis_graph_peak_bytes", u64, [vp]),
    ("aegis_p2p_create", ctypes.c_int, [vp, u64, vp, ctypes.POINTER(vp)]),
    ("aegis_p2p_open", ctypes.c_int, [vp, vp, vp, u32, u32]),
    ("aegis_p2p_open_local", ctypes.c_int, [vp, vp, ctypes.POINTER(vp), u32, u32]),
    ("aegis_p2p_stage", ctypes.c_int, [vp, vp, vp, u64]),
    ("aegis_p2p_reduce", ctypes.c_int, [vp, vp, vp, u64, u32]),
    ("aegis_p2p_destroy", ctypes.c_int, [vp]),
    ("aegis_graph_p2p_bytes", ctypes.c_int, [vp, u64p]),
    ("aegis_graph_set_p2p", ctypes.c_int, [vp, vp]),
    ("aegis_graph_set_fault", ctypes.c_int, [vp, ctypes.c_int]),
    ("aegis_graph_set_matmul_modes", ctypes.c_int, [vp, ctypes.c_int]),
    ("aegis_graph_set_stored_weights", ctypes.c_int, [vp, ctypes.c_int]),
    ("aegis_pmult_acc_stored", ctypes.c_int, [vp, vp, u32, u32, u32, vp, u32, u32, vp, u32, u32, u32]),
]

# int (*)(void* user, uint64_t* buf, uint64_t words_per_rank, uint32_t group)
REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32)

_lib = None


def load():
    """Load libaegis.so (raises OSError if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} is missing: run __graft_entry__.build() first "
                          "(there is no CPU fallback for the product path)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
