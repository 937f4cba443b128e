/* include/aegis.h -- C-ABI of libaegis, the B200-native executor of the AEGIS
 * CKKS hot path (arXiv 2604.03425).  Plain pointers and sizes only; no C++ or
 * torch types cross this boundary; no exceptions escape it.
 *
 * The reference (/root/reference/proj/include/heplan/, header-only C++20) has
 * no executor: SPEC.md:392-443 specifies one (`rns-oracle`: exec_sequential /
 * exec_plan) over the IR of poly_ir.hpp / he_ir.hpp.  Each entry point below
 * replaces the reference interface cited beside it (INTEGRATION.md shows the
 * binding a heplan maintainer would add).
 *
 * Data layout: a bundle is a [lane][comp][limb][N] array of
 * u64 residues; limb i of every bundle is modulo the main prime q_i, values
 * canonical in [0, p), polynomials in the NTT (evaluation) domain.
 *
 * Errors: every call returns 0 on success or one of the AEGIS_E* codes; the
 * message is available from aegis_last_error(ctx).  The C++ wrapper
 * (paper_2604_03425_b200/csrc/heplan_compat.hpp) rethrows them as the
 * reference's exception types: EINVAL -> std::invalid_argument,
 * ELOGIC -> std::logic_error, others -> std::runtime_error.
 * Threading: one host thread per context; all work is asynchronous on the
 * context's compute stream; errors from the device surface at aegis_sync().
 * The device-synchronised PCMM exchange (aegis_graph_set_p2p) is for one
 * process per GPU (the deployment, tested with separate processes) or one
 * process driving several GPUs (aegis_p2p_open_local).  Several contexts of
 * ONE process on ONE device share a CUDA context: a device-synchronising call
 * in one rank's thread (memory mapping, cudaFree) then waits for another
 * rank's flag-waiting kernel -- use the reduce hook there.  A waiting kernel
 * traps after 60 s, so such a misuse is an error, not a hang. 
 */
#ifndef AEGIS_H
#define AEGIS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define AEGIS_OK 0
#define AEGIS_EINVAL 1 /* std::invalid_argument in the reference (ckks.hpp:149, graph.hpp:100) */
#define AEGIS_ELOGIC 2 /* std::logic_error (he_ir.hpp:191) */
#define AEGIS_ECUDA 3
#define AEGIS_ENCCL 4
#define AEGIS_EOOM 5

typedef struct aegis_ctx aegis_ctx;
typedef struct aegis_bundle aegis_bundle;
typedef struct aegis_graph aegis_graph;
typedef struct aegis_p2p aegis_p2p;

/* CkksProfile (ckks.hpp:21-46) plus the seeds of the synthetic workload. */
typedef struct aegis_params {
  uint32_t log_n;           /* ring_degree = 2^log_n, 4..17 */
  uint32_t chain_length;    /* |Q_L| main primes (35 for BERT) */
  uint32_t special_primes;  /* |P|; must be 4 (AEGIS_SPECIAL_PRIMES) */
  uint32_t bootstrap_level; /* l_boot (14) -> post_boot_level = chain - l_boot */
  uint64_t seed_input;      /* graph-input ciphertexts (PRNG tag 1) */
  uint64_t seed_weight;     /* kGenerate weights (tag 2) */
  uint64_t seed_key;        /* key-switching keys (tag 3) */
} aegis_params;

/* ---- context (one per GPU) ----------------------------------------------- */
int aegis_ctx_create(const aegis_params* params, int device, aegis_ctx** out);
int aegis_ctx_destroy(aegis_ctx* ctx);
const char* aegis_last_error(const aegis_ctx* ctx);
void* aegis_stream_compute(aegis_ctx* ctx); /* cudaStream_t */
void* aegis_stream_comm(aegis_ctx* ctx);    /* cudaStream_t for collectives */
int aegis_sync(aegis_ctx* ctx);
uint64_t aegis_prime(const aegis_ctx* ctx, uint32_t ext_index); /* <60 main, >=60 special */
/* count of kernels this context launched (for the bench's gpu_launches claim) */
uint64_t aegis_launch_count(const aegis_ctx* ctx);
/* Kernel probe (measurement only; one probe per process): kind 1 = cfwd_a
 * (exact basis conversion fused with NTT pass A), 2 = fwd_b_fin (NTT pass B
 * with the ModDown / rescale finish), 3 = fwd_b_km (ModUp pass B fused with
 * the key inner product), 0 = off.  While on, CUDA events bracket every
 * launch of that kernel on the compute stream; aegis_probe_read returns the
 * launch count, the summed device time and the summed algorithmic bytes
 * (inputs read once, outputs written once). */
int aegis_probe_start(aegis_ctx* ctx, int kind);
int aegis_probe_read(aegis_ctx* ctx, uint64_t* launches, double* ms, double* alg_bytes);
/* NTT butterfly arithmetic: 0 = 64-bit integer Shoup, 1 = exact FP64 (default;
 * N = 2^16 uses the direct-access v2 passes), 2 = FP64 through the generic
 * passes.  impl < 0 only queries.  Returns the active implementation. */
int aegis_ntt_impl(int impl);

/* ---- bundles (CtBundle, he_ir.hpp:57-74) --------------------------------- */
int aegis_bundle_alloc(aegis_ctx* ctx, uint32_t lanes, uint32_t comps, uint32_t level,
                       aegis_bundle** out);
int aegis_bundle_free(aegis_ctx* ctx, aegis_bundle* b);
/* count must equal lanes*comps*level*N; host buffers are caller owned */
int aegis_bundle_upload(aegis_ctx* ctx, aegis_bundle* b, const uint64_t* host, uint64_t count);
int aegis_bundle_download(aegis_ctx* ctx, const aegis_bundle* b, uint64_t* host, uint64_t count);
int aegis_bundle_info(const aegis_bundle* b, uint32_t* lanes, uint32_t* comps, uint32_t* level,
                      uint64_t* device_ptr);
/* synthetic "fresh activations" (he_ir.hpp:178-188): PRNG tag 1 keyed by bundle_id */
int aegis_bundle_fill_input(aegis_ctx* ctx, aegis_bundle* b, uint32_t bundle_id);
/* DESIGN.md §2.4 content hash of the first `comps` comps and `level` limbs */
int aegis_bundle_hash(aegis_ctx* ctx, const aegis_bundle* b, uint32_t comps, uint32_t level,
                      uint64_t* out);

/* ---- keys (poly_ir.hpp:300-305: 0 = relin, 1000 + r = rotation r) -------- */
int aegis_keys_generate(aegis_ctx* ctx, const uint64_t* key_ids, uint32_t count);
/* caller-supplied key (replaces any key with this id): `words` =
 * digits x 2 x (chain + 4) x N u64, layout [digit][comp][slot][N], canonical
 * residues; slot s < chain is q_s, slot chain + i is the special prime P_i;
 * digit j = the key for the centred lift of limbs [4j, 4j + 4).  coeff_domain
 * != 0: rows are coefficient vectors (the library applies each slot's NTT),
 * else NTT (evaluation) order.  Rotation keys (id 1000 + r) are given in the
 * standard form for s(X^{5^r}) and stored pre-permuted internally.  The key
 * for digit j must carry the CRT factor P * Qhat_j * [Qhat_j^{-1}]_{Q_j}
 * (Qhat_j w.r.t. the full main chain), so one key serves every level. */
int aegis_keys_upload(aegis_ctx* ctx, uint64_t key_id, const uint64_t* host, uint64_t words, int coeff_domain);
int aegis_keys_bytes(const aegis_ctx* ctx, uint64_t* out);

/* ---- wire / disk format (csrc/store.cu) --------------
 * 128-byte header (magic "AEGS", ring, prime-chain fingerprint, shape, key id,
 * DESIGN.md §2.4 content hash) + little-endian u64 payload.  Bundles are
 * [lane][comp][limb][N] (encoded plaintexts are 1-component bundles, e.g. the
 * weights aegis_encode writes; ckks.hpp:226-283 byte model); keys are the
 * library's internal [digit][comp][slot][N] form (rotation keys
 * pre-permuted).  Transfers stream through two pinned 64 MiB buffers so file
 * I/O overlaps the DMA; a load recomputes the content hash on the device and
 * rejects torn, foreign-chain or mismatched files with EINVAL. */
int aegis_bundle_save(aegis_ctx* ctx, const aegis_bundle* b, const char* path);
int aegis_bundle_load(aegis_ctx* ctx, const char* path, aegis_bundle** out);
int aegis_keys_save(aegis_ctx* ctx, uint64_t key_id, const char* path);
int aegis_keys_load(aegis_ctx* ctx, uint64_t key_id, const char* path);

/* ---- polynomial instructions (PolyOpKind, poly_ir.hpp:23-32) -------------
 * FragSpan-style addressing (poly_ir.hpp:87-99): lanes [lane, lane+lane_count)
 * and limbs [prime_lo, prime_hi] of every component of bundle b.          */
int aegis_ntt(aegis_ctx* ctx, aegis_bundle* b, uint32_t lane, uint32_t lane_count,
              uint32_t prime_lo, uint32_t prime_hi, int inverse); /* kNtt / kIntt */
/* kAutomorphism: eval-domain x -> x^galois of the first `level` limbs */
int aegis_automorphism(aegis_ctx* ctx, aegis_bundle* out, const aegis_bundle* in, uint32_t lane,
                       uint32_t lane_count, uint32_t level, uint64_t galois);
/* exact centred basis conversion on coefficient-domain limbs (kModUp/kModDown
 * semantics): out limb dst_limb[t] of every lane/comp gets
 * lift_centered(in[src_limb[0..k)]) mod prime(dst_ext[t]).  src/dst ext indices
 * name the primes; src_limb/dst_limb the limb positions inside the bundles.  */
int aegis_basis_convert(aegis_ctx* ctx, aegis_bundle* out, const aegis_bundle* in,
                        const uint32_t* src_ext, const uint32_t* src_limb, uint32_t k,
                        const uint32_t* dst_ext, const uint32_t* dst_limb, uint32_t m);
/* hybrid key switch of component `comp` of every lane (poly_ir.hpp:219-298):
 * out (2 comps, level limbs) = KS(in[comp]) with key key_id */
int aegis_keyswitch(aegis_ctx* ctx, aegis_bundle* out, const aegis_bundle* in, uint32_t comp,
                    uint32_t level, uint64_t key_id);

/* kLimbMulAdd with its LimbOpcode payload (poly_ir.hpp:49-58), as
 * HeLowering::pointwise emits it per limb (poly_ir.hpp:192-213), on the
 * FragSpan out = lanes [out_lane, out_lane + lanes) x limbs [prime_lo,
 * prime_hi] of `out`; operand lanes follow emit_per_lane (a_count / b_count
 * lanes starting at a_lane / b_lane).  Plaintext operands are 1-component
 * bundles: they feed component 0 of Add/Sub and scale every component of
 * Mul/MulAcc; two ciphertexts Mul into the 3-component tensor ("component
 * product", poly_ir.hpp:53).  kGenerate fills `out` with the seeded fragment
 * of bundle id `param` (the executor's kEncode weights); a and b are unused.
 * kKeyMul is not a standalone instruction here: it runs inside
 * aegis_keyswitch (the IR's KeyMul has no digit split) and returns EINVAL.
 * `out` may be `a` only with identical lanes (a_lane == out_lane, a_count ==
 * lanes); results are canonical residues. */
#define AEGIS_LIMB_ADD 1      /* out = a + b   */
#define AEGIS_LIMB_SUB 2      /* out = a - b   */
#define AEGIS_LIMB_MUL 3      /* out = a * b   */
#define AEGIS_LIMB_MULACC 4   /* out += a * b  */
#define AEGIS_LIMB_ADDACC 5   /* out += a      */
#define AEGIS_LIMB_KEYMUL 6   /* out = a * key(param): inside aegis_keyswitch only */
#define AEGIS_LIMB_GENERATE 7 /* out = PRNG fragment of bundle `param` */
int aegis_limb_op(aegis_ctx* ctx, int opcode, aegis_bundle* out, uint32_t out_lane, uint32_t lanes,
                  const aegis_bundle* a, uint32_t a_lane, uint32_t a_count, const aegis_bundle* b,
                  uint32_t b_lane, uint32_t b_count, uint32_t prime_lo, uint32_t prime_hi, uint64_t param);
/* kLimbDrop (poly_ir.hpp:341-354): level -> level - 1.  mode = PolyMode:
 * 0 (kNone) keeps limbs [0, level - 1) (exact truncation, graph.hpp:106-107);
 * 3 (kRescaleTail) divides by the dropped prime q_{level-1} and rounds
 * (= aegis_rescale).  Other modes are EINVAL. */
#define AEGIS_MODE_NONE 0
#define AEGIS_MODE_KEY_SWITCH 1
#define AEGIS_MODE_BOOT_RESET 2
#define AEGIS_MODE_RESCALE_TAIL 3
int aegis_limb_drop(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, const aegis_bundle* in,
                    uint32_t in_lane, uint32_t lanes, uint32_t level, int mode);

/* ---- HE operators (HeOpKind, he_ir.hpp:21-31), one call per bundled HeOp --
 * Operand lanes follow emit_per_lane (he_ir.hpp:200-222): output lane l reads
 * operand lane  lane0 + (count == lanes ? l : l % count).                  */
int aegis_rot(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, const aegis_bundle* in,
              uint32_t in_lane, uint32_t lanes, uint32_t level, int offset);
/* Several rotations of the same source lanes (the rotation ladder of
 * lower_matmul / lower_attention_*, he_ir.hpp:224-241, 328-373): ModUp of the
 * source is computed once and shared by every offset (hoisting); rotation k
 * writes lanes [out_lanes[k], out_lanes[k] + lanes) of outs[k].  Bit-identical
 * to n_offsets separate aegis_rot calls. */
int aegis_rot_hoisted(aegis_ctx* ctx, aegis_bundle* const* outs, const uint32_t* out_lanes, const int* offsets,
                      uint32_t n_offsets, const aegis_bundle* in, uint32_t in_lane, uint32_t lanes,
                      uint32_t level);
int aegis_relin(aegis_ctx* ctx, aegis_bundle* b, uint32_t lane, uint32_t lanes, uint32_t level);
/* kPAdd (he_ir.hpp:23): out[l] = ct[..] + pt[..] (pt: 1-component bundle, added to component 0) */
int aegis_padd(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, uint32_t lanes, const aegis_bundle* ct,
               uint32_t ct_lane, uint32_t ct_count, const aegis_bundle* pt, uint32_t pt_lane, uint32_t pt_count,
               uint32_t level);
/* kEncode (he_ir.hpp:243-252, lowered to kGenerate poly_ir.hpp:310-321): lanes
 * [lane, lane + lanes) of the plaintext bundle pt (1 component) receive the
 * weights of bundle id `weight_bundle_id` -- the same words the PMult kernel
 * generates in-kernel, so a stored-plaintext PCMM reads what the fused one
 * computes. */
int aegis_encode(aegis_ctx* ctx, aegis_bundle* pt, uint32_t lane, uint32_t lanes, uint32_t level,
                 uint32_t weight_bundle_id);
int aegis_rescale(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, const aegis_bundle* in,
                  uint32_t in_lane, uint32_t lanes, uint32_t level);
int aegis_boot(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, const aegis_bundle* in,
               uint32_t in_lane, uint32_t lanes, uint32_t level, uint32_t out_level);
int aegis_cmult(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, uint32_t lanes,
                const aegis_bundle* a, uint32_t a_lane, uint32_t a_count, const aegis_bundle* b,
                uint32_t b_lane, uint32_t b_count, uint32_t level);
/* accumulate != 0: out[l] += a[..]; else out[l] = a[..] + b[..] */
int aegis_cadd(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, uint32_t lanes,
               const aegis_bundle* a, uint32_t a_lane, uint32_t a_count, const aegis_bundle* b,
               uint32_t b_lane, uint32_t b_count, uint32_t level, int accumulate);
/* bundled PMult-accumulate (he_ir.hpp:360-371) with in-kernel kGenerate
 * weights of bundle weight_bundle_id; chunk_period as in
 * CtBundle::chunk_period of the accumulator (0 = whole). */
int aegis_pmult_acc(aegis_ctx* ctx, aegis_bundle* acc, uint32_t acc_lane, uint32_t acc_lanes,
                    uint32_t chunk_period, const aegis_bundle* x, uint32_t x_lane, uint32_t x_lanes,
                    uint32_t weight_bundle_id, uint32_t weight_lanes, uint32_t level);

/* the same PCMM step with STORED plaintext weights (SURVEY §8(d) stored
 * variant; ckks.hpp:226-283 plaintext bytes): lanes [w_lane, w_lane + w_lanes)
 * of the 1-component bundle w hold W[ci * c_out + o] (e.g. written by
 * aegis_encode or aegis_bundle_load); the kernel streams them from HBM. */
int aegis_pmult_acc_stored(aegis_ctx* ctx, aegis_bundle* acc, uint32_t acc_lane, uint32_t acc_lanes,
                           uint32_t chunk_period, const aegis_bundle* x, uint32_t x_lane, uint32_t x_lanes,
                           const aegis_bundle* w, uint32_t w_lane, uint32_t w_lanes, uint32_t level);

/* ---- layer drivers + executor (he_ir.hpp:683 lower_app_to_he; SPEC exec_*) */
typedef struct aegis_model {
  uint32_t kind;        /* 0: transformer blocks (graph.hpp:168), 1: FFN only (config 1) */
  uint32_t layers;      /* TransformerConfig::layer_count */
  uint32_t model_dim, ffn_dim, head_dim, slots_per_token;
  uint64_t tokens;
} aegis_model;
int aegis_graph_build(aegis_ctx* ctx, const aegis_model* model, aegis_graph** out);
/* same, without a device (planning only): the lowering is host code */
int aegis_graph_build_params(const aegis_params* params, const aegis_model* model, aegis_graph** out);
int aegis_graph_load(aegis_ctx* ctx, const char* path, aegis_graph** out); /* heops text */
int aegis_graph_dump(const aegis_graph* g, const char* path);
int aegis_graph_info(const aegis_graph* g, uint64_t* ops, uint64_t* bundles);
/* In-memory HeOpGraph ingest (he_ir.hpp:57-120) -- no text round trip.  The
 * descriptors mirror CtBundle / LaneSlice / HeOp field for field (enum values
 * as in he_ir.hpp: HeOpKind, BundleClass, AggregationAxis); bundle ids are the
 * array indices, op ids the op positions.  `meta` carries the CkksProfile /
 * layout / model the graph was lowered for (token groups, ring degree).  The
 * graph is validated (bundle ids, lane ranges, levels) before it is accepted:
 * EINVAL with the first offending op otherwise.  heplan_compat.hpp builds
 * these arrays from a heplan::HeOpGraph. */
typedef struct aegis_graph_meta {
  uint32_t log_n, chain_length, bootstrap_level, slots_per_token;
  uint32_t model_dim, head_dim, ffn_dim, layers, kind;
  uint64_t tokens;
} aegis_graph_meta;
typedef struct aegis_bundle_desc {
  uint32_t lanes, level, components, cls, aggregation, app_node, chunk_period, replicate_hint;
  const char* tag; /* may be NULL; copied */
} aegis_bundle_desc;
typedef struct aegis_slice {
  uint32_t bundle, lane, lane_count;
} aegis_slice;
#define AEGIS_MAX_OP_INPUTS 4
typedef struct aegis_op_desc {
  uint32_t kind, accumulate, aligned, aggregation;
  int32_t rot_offset, phase;
  aegis_slice out;
  uint32_t in_count;
  aegis_slice ins[AEGIS_MAX_OP_INPUTS];
  uint64_t work;
  uint32_t use_level, app_node;
} aegis_op_desc;
int aegis_graph_from_ops(const aegis_graph_meta* meta, const aegis_bundle_desc* bundles, uint32_t n_bundles,
                         const aegis_op_desc* ops, uint64_t n_ops, const uint32_t* inputs, uint32_t n_inputs,
                         aegis_graph** out);
/* the reverse: copy a graph's bundles / ops / inputs out (caps in elements,
 * NULL arrays are skipped; *n_inputs receives the input count; tag pointers
 * stay valid while the graph lives) */
int aegis_graph_export(const aegis_graph* g, aegis_bundle_desc* bundles, uint32_t bundle_cap, aegis_op_desc* ops,
                       uint64_t op_cap, uint32_t* inputs, uint32_t input_cap, uint32_t* n_inputs,
                       aegis_graph_meta* meta);
/* Multi-GPU token-coherent placement (placement.hpp:175-182):
 * this context executes only the lanes rank `rank` of `world` owns.  With
 * world <= token groups each rank owns whole token groups (no collective);
 * with world = m * groups the m ranks of a group split its positions and each
 * PCMM is reduce-scattered once through the reducer hook.  world <= 1 clears. */
int aegis_graph_set_shard(aegis_graph* g, uint32_t world, uint32_t rank);
/* Parity of one token group inside an UNSHARDED run: every lane is still
 * computed, but bundle hashes (aegis_graph_run) cover only the lanes of token
 * group `group` (as aegis_graph_set_shard(token groups, group) would own
 * them).  group < 0 restores whole-bundle hashes. */
int aegis_graph_set_hash_group(aegis_graph* g, int32_t group);
/* reduce-scatter hook: sum words_per_rank*m u64 words at device pointer `buf`
 * over the m ranks of token group `group` (NCCL uint64 sum), leaving this
 * rank's share at buf + part*words_per_rank; return 0 on success. */
typedef int (*aegis_reduce_fn)(void* user, uint64_t* buf, uint64_t words_per_rank, uint32_t group);
int aegis_graph_set_reducer(aegis_graph* g, aegis_reduce_fn fn, void* user);
/* The same reduce-scatter over CUDA IPC / NVLink peer memory instead of a
 * library collective (csrc/p2p.cu; replaces the comm stream's kReduceOutputs
 * event, comm_plan.hpp:127, 238).  Each rank of a token group creates a window
 * (bytes >= m * words_per_rank * 8) and exports its 64-byte IPC handle; after the
 * handles are exchanged, open maps all m of them.  Per reduction the host runs
 * stage(buf, m * words) -> group barrier -> reduce(buf + part * words, words,
 * part) -> group barrier.  reduce writes the uint64 sum of the m windows'
 * share `part` (the reduce hook's semantics). */
int aegis_p2p_create(aegis_ctx* ctx, uint64_t bytes, void* handle_out, aegis_p2p** out);
int aegis_p2p_open(aegis_ctx* ctx, aegis_p2p* w, const void* handles, uint32_t m, uint32_t self);
/* same-process group (one host thread per context, or one thread driving
 * several contexts): group[r] is rank r's window, used through its device
 * pointer (no IPC mapping) */
int aegis_p2p_open_local(aegis_ctx* ctx, aegis_p2p* w, aegis_p2p* const* group, uint32_t m, uint32_t self);
int aegis_p2p_stage(aegis_ctx* ctx, aegis_p2p* w, const uint64_t* buf, uint64_t words);
int aegis_p2p_reduce(aegis_ctx* ctx, aegis_p2p* w, uint64_t* dst, uint64_t words_per_rank, uint32_t part);
int aegis_p2p_destroy(aegis_p2p* w);
/* The executor's own data plane for the sharded PCMM reduce-scatter (the
 * comm stream of PAPER.md:518 / comm_plan.hpp:88-91): with a window attached,
 * aegis_graph_run needs no reduce hook.  As soon as the last PMult of an
 * accumulator is issued, every sub-tensor is exchanged on aegis_stream_comm
 * -- pushes into the peers' windows, flags in peer memory, sums, acks -- and
 * the compute stream waits on a CUDA event only when an op touches those
 * lanes, so the rescale of one sub-tensor overlaps the exchange of the next.
 * No host barrier or callback runs inside the layer.  aegis_graph_p2p_bytes
 * gives the window size the current shard needs (call after set_shard; 0
 * when no token group spans several ranks).  The window must stay alive while
 * the graph runs; every rank of a group must attach windows of equal size. */
int aegis_graph_p2p_bytes(const aegis_graph* g, uint64_t* bytes);
int aegis_graph_set_p2p(aegis_graph* g, aegis_p2p* w);
/* stored-plaintext PCMM for the whole graph (separately reported variant):
 * every kEncode op writes its weight bundle to HBM and each PMult reads it
 * (aegis_pmult_acc_stored) instead of generating the weights in-kernel.  All
 * ciphertext bundles are bit-identical to the default; weight bundles are not
 * hashed.  Default off. */
int aegis_graph_set_stored_weights(aegis_graph* g, int enable);
/* Matmul collective modes when a token group spans m > 1 devices.  0
 * (default): every PCMM is input-stationary and reduce-scatters its partial
 * outputs (no rotation is repeated).  1: each matmul takes the mode the
 * reference's byte rule picks (comm_plan.hpp:226-238): where gathering the
 * activation moves fewer bytes than reducing the outputs, the activation is
 * all-gathered over the group on the comm stream and every rank rotates all
 * of its lanes and computes its own output share completely.  Needs a p2p
 * window (aegis_graph_set_p2p; size it with aegis_graph_p2p_bytes after this
 * call); the plan (aegis_plan_build) follows the same modes.  Bit-identical. */
int aegis_graph_set_matmul_modes(aegis_graph* g, int reference_rule);
/* fault injection for tests: kind 1 drops the PCMM exchange (every rank keeps
 * its partial sums); 0 restores normal execution */
int aegis_graph_set_fault(aegis_graph* g, int kind);
/* ---- execution plan (comm_plan.hpp:51-118 ExecutionPlan; plan.h) ---------
 * The Aegis plan of this graph on `world` devices under token-coherent
 * placement: per device the compute instructions (HeOp, owned lane run,
 * flags, the event it waits for) and the collective events (kind, semantic,
 * participants, payload, bytes, trigger/wait positions), plus, per matmul,
 * the bytes of both collective modes and the one the reference's rule picks
 * (comm_plan.hpp:226-238) next to the one this executor runs.  reorder
 * staggers the rotation-offset order per device part.  If the
 * shape cannot be split over `world` devices the plan has executable = 0, no
 * devices or events, and still the matmul analysis.  No device needed. */
typedef struct aegis_plan aegis_plan;
typedef struct aegis_plan_summary {
  uint32_t world, token_groups, ranks_per_group, reordered, executable, matmuls, matmuls_gather_chosen, pad;
  uint64_t events, events_executed, instrs_total;
  uint64_t bytes_total, bytes_ffn, bytes_attention, bytes_layernorm, bytes_boot, bytes_other;
  uint64_t bytes_reference_rule; /* total if every matmul used the mode the reference's rule picks */
} aegis_plan_summary;
typedef struct aegis_plan_event {
  uint32_t id, kind /* 0 AllGather, 1 ReduceScatter, 2 AllReduce */, semantic /* 0 Move, 1 Combine, 2 CombineScatter */;
  uint32_t dev_lo, dev_count, bundle, lane, lane_count, level, category, app_node, he_op, executed;
  uint64_t bytes_per_device, bytes_total;
} aegis_plan_event;
typedef struct aegis_plan_instr {
  uint32_t op, lane, lane_count, flags;
  int32_t wait_event;
} aegis_plan_instr;
typedef struct aegis_plan_matmul {
  uint32_t app_node, acc_bundle, input_bundle, ship_bundle, chosen, executed; /* 0 local, 1 gather, 2 reduce */
  uint64_t gather_bytes, reduce_bytes;
} aegis_plan_matmul;
int aegis_plan_build(const aegis_graph* g, uint32_t world, int reorder, aegis_plan** out);
int aegis_plan_summary_get(const aegis_plan* p, aegis_plan_summary* out);
int aegis_plan_events(const aegis_plan* p, aegis_plan_event* out, uint64_t cap, uint64_t* n);
int aegis_plan_device(const aegis_plan* p, uint32_t device, aegis_plan_instr* out, uint64_t cap, uint64_t* n);
int aegis_plan_matmuls(const aegis_plan* p, aegis_plan_matmul* out, uint64_t cap, uint64_t* n);
const char* aegis_plan_note(const aegis_plan* p);
/* The graph as device `device` of the plan executes it: the same ops in the
 * order of that device's compute stream (e.g. the staggered rotation-offset
 * order of a reordered plan).  Only the order changes, and only inside a
 * matmul's diagonal loop, whose accumulation commutes: every bundle is
 * bit-identical.  Shard the new graph like the original. */
int aegis_graph_from_plan(const aegis_graph* g, const aegis_plan* p, uint32_t device, aegis_graph** out);
int aegis_plan_free(aegis_plan* p);
/* bytes this rank sent through its PCMM exchanges in the last aegis_graph_run
 * (the executed counterpart of the plan's events) */
int aegis_graph_comm_bytes(const aegis_graph* g, uint64_t* bytes);
/* lane ownership of bundle `bundle` under the current shard (1 = owned) */
int aegis_graph_owned_lanes(const aegis_graph* g, uint32_t bundle, uint8_t* mask, uint32_t cap);
int aegis_graph_shard_info(const aegis_graph* g, uint32_t* tg_total, uint32_t* tg_lo, uint32_t* tg_hi,
                           uint32_t* ranks_per_group, uint32_t* part);
/* hoisted ModUp across the rotations of one source (bit-exact; default on) */
int aegis_graph_set_hoisting(aegis_graph* g, int enable);
/* dead-lane elimination (default off): output lanes no later op reads are not
 * computed.  The graph's final bundle is bit-identical; hashes of bundles with
 * dead lanes are not meaningful in this mode.  Reported as a separate variant. */
int aegis_graph_set_dce(aegis_graph* g, int enable);
/* wrapped accumulation (default on): accumulating CAdds whose operand is
 * narrower than the output (acc[j] += x[j mod m]) are summed at the operand's
 * width and applied to the output once, before its next reader.  Modular
 * addition is exact and associative, so every bundle any op reads -- and every
 * bundle hash -- is bit-identical to op-by-op execution. */
int aegis_graph_set_wrap_defer(aegis_graph* g, int enable);
/* per-op device times (CUDA events around every HeOp) of the next runs */
int aegis_graph_set_profiling(aegis_graph* g, int enable);
int aegis_graph_op_times(const aegis_graph* g, float* ms, uint64_t cap, uint64_t* n);
/* the two-stream trace of the last profiled run: every comm-stream exchange
 * as (start ms, end ms, bundle id) triples relative to the run's first
 * compute-stream event (op i spans [sum of op_times[<i], sum[<=i]]) */
int aegis_graph_comm_times(const aegis_graph* g, float* out, uint64_t cap, uint64_t* n);
/* bytes copied host->device / device->host by the last aegis_graph_run_host */
int aegis_graph_io_bytes(const aegis_graph* g, uint64_t* h2d, uint64_t* d2h);
/* Execute ops [0, max_ops) (all if < 0).  Bundles are allocated at first write
 * and freed after their last use.  If hashes != NULL, hashes[b] receives the
 * content hash of bundle b when it dies (0 if never materialised). */
int aegis_graph_run(aegis_ctx* ctx, aegis_graph* g, int64_t max_ops, uint64_t* hashes,
                    uint64_t nhashes);
/* Host-buffer execution (the end-to-end path): the graph inputs are read from
 * `in` (graph-input bundles concatenated in graph order, each
 * [lane][2][level][N]) and the last op's output bundle is written to `out`.
 * aegis_graph_io_words gives both sizes; aegis_graph_host_inputs fills a host
 * buffer with the same synthetic inputs aegis_graph_run generates on device. */
int aegis_graph_io_words(const aegis_graph* g, uint64_t* in_words, uint64_t* out_words);
int aegis_graph_host_inputs(aegis_ctx* ctx, const aegis_graph* g, uint64_t* in, uint64_t in_words);
int aegis_graph_run_host(aegis_ctx* ctx, aegis_graph* g, const uint64_t* in, uint64_t in_words,
                         uint64_t* out, uint64_t out_words);
/* key ids the graph needs (for aegis_keys_generate); returns count via *n */
int aegis_graph_key_ids(const aegis_graph* g, uint64_t* ids, uint32_t cap, uint32_t* n);
int aegis_graph_free(aegis_graph* g);
/* peak device bytes of the last aegis_graph_run */
uint64_t aegis_graph_peak_bytes(const aegis_graph* g);

#ifdef __cplusplus
}
#endif
#endif
