/* oracle/oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the AEGIS hot path (CKKS RNS evaluation of the
 * reference's HE-op sequence).  It is the CHECKER for libaegis: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.  The
 * product library never links or calls it.
 *
 * Every routine cites the reference file:line whose semantics it restates
 * (paths relative to /root/reference/proj/include/heplan/).  Parity of this
 * oracle is pinned against the unmodified reference (oracle/_ref, built from
 * rns_math.hpp / he_ir.hpp in place) by tests/test_oracle_golden.py and the
 * fixtures under tests/golden/.
 *
 * Conventions:
 *   - extended prime index e: e < 60 -> main prime q_e, e >= 60 -> special P_{e-60}
 *   - a bundle is [lane][comp][limb][N] u64, canonical residues in [0, p)
 *   - polynomials held by bundles are in the NTT (evaluation) domain
 */
#ifndef AEGIS_ORACLE_H
#define AEGIS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_ctx orc_ctx;

/* log_n in [3, 17]; chain = |Q_L| main primes; lboot = l_boot (ckks.hpp:31).
 * seeds: input ciphertexts, generated weights (kGenerate), keys. */
orc_ctx* orc_create(uint32_t log_n, uint32_t chain, uint32_t lboot, uint64_t seed_input,
                    uint64_t seed_weight, uint64_t seed_key, int threads);
void orc_destroy(orc_ctx* c);
uint64_t orc_prime(const orc_ctx* c, uint32_t ext_index);
uint64_t orc_psi(orc_ctx* c, uint32_t ext_index);

/* --- PRNG --------------------------------------------- */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_row_key(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b, uint64_t c, uint64_t d);
void orc_fill_uniform(uint64_t row_key, uint64_t p, uint64_t* out, uint32_t n);

/* --- L0 primitives (rns_math.hpp) --------------------------------------- */
/* nlimbs limbs of N coefficients, limb k uses ext prime ext_idx[k]. In place. */
int orc_ntt(orc_ctx* c, uint64_t* data, const uint32_t* ext_idx, uint32_t nlimbs, int inverse);
/* eval-domain automorphism x -> x^k on each limb (rns_math.hpp:127-139 restated). */
int orc_automorphism_eval(orc_ctx* c, const uint64_t* in, uint64_t* out, uint32_t nlimbs, uint64_t galois);
/* coefficient-domain automorphism exactly as rns_math.hpp:127-139 (any prime p). */
int orc_automorphism_coeff(orc_ctx* c, const uint64_t* in, uint64_t* out, uint64_t p, uint64_t galois);
/* one limb, any NTT-friendly prime p (tables built per call; for KATs). */
int orc_ntt_prime(orc_ctx* c, uint64_t* data, uint64_t p, int inverse);
uint64_t orc_galois(int offset, uint32_t n);

/* Exact centred basis conversion (rns_math.hpp:171-186 semantics at any size):
 * in: k source limbs (coefficient domain) over ext primes src[0..k), out: m
 * target limbs over ext primes dst[0..m). Coefficient j of out limb t =
 * lift_centered(in[.][j]) mod dst[t]. Returns the number of near-tie
 * fallbacks taken (>= 0). */
int64_t orc_basis_convert(orc_ctx* c, const uint64_t* in, const uint32_t* src, uint32_t k,
                          uint64_t* out, const uint32_t* dst, uint32_t m);
/* Same result computed with full multi-precision CRT for every coefficient
 * (slow, independent check of the fixed-point + fallback path). */
int orc_basis_convert_bigint(orc_ctx* c, const uint64_t* in, const uint32_t* src, uint32_t k,
                             uint64_t* out, const uint32_t* dst, uint32_t m);

/* --- HE operators on single ciphertext lanes ([comp][limb][N]) ----------- */
/* Hybrid key switch of one polynomial d (level l, NTT domain) with key_id. */
int orc_keyswitch(orc_ctx* c, const uint64_t* d, uint32_t level, uint64_t key_id,
                  uint64_t* out0, uint64_t* out1);
int orc_rotate(orc_ctx* c, const uint64_t* ct, uint32_t level, int offset, uint64_t* out);
int orc_relin(orc_ctx* c, const uint64_t* ct3, uint32_t level, uint64_t* out2);
int orc_rescale(orc_ctx* c, const uint64_t* ct, uint32_t level, uint64_t* out);
int orc_boot_reset(orc_ctx* c, const uint64_t* ct, uint32_t level, uint32_t out_level, uint64_t* out);
int orc_cmult(orc_ctx* c, const uint64_t* a, const uint64_t* b, uint32_t level, uint64_t* out3);
/* key material limb: key_id, digit, comp, ext prime -> N coefficients */
void orc_key_limb(orc_ctx* c, uint64_t key_id, uint32_t digit, uint32_t comp, uint32_t ext, uint64_t* out);
/* generated weight limb (kGenerate, poly_ir.hpp:57, 310-321): bundle, lane, limb */
void orc_weight_limb(orc_ctx* c, uint32_t bundle, uint32_t lane, uint32_t limb, uint64_t* out);
/* graph-input ciphertext limb: bundle, lane, comp, limb */
void orc_input_limb(orc_ctx* c, uint32_t bundle, uint32_t lane, uint32_t comp, uint32_t limb, uint64_t* out);

/* --- graph executor (SPEC.md:407-415 exec_sequential) ------------------- */
/* Runs the HE-op graph file (tests/golden/ heops format).  max_ops < 0 runs
 * all.  For every bundle, when it dies (after its last use) or at the end,
 * its content hash is written to hashes[bundle_id] (array
 * sized >= number of bundles; untouched bundles get 0).  Returns number of
 * bundles, or < 0 on error (message via orc_last_error). */
int64_t orc_run_graph(orc_ctx* c, const char* path, int64_t max_ops, uint64_t* hashes,
                      uint64_t nhashes);
/* Lane-subset form: computes and hashes only the lanes of token group tg_sel
 * (of tg_total), tagged by the oracle's own restatement of token-coherent
 * placement (placement.hpp:175-182).  tg_sel < 0 = every lane (orc_run_graph). */
int64_t orc_run_graph_tg(orc_ctx* c, const char* path, int64_t max_ops, uint64_t* hashes,
                         uint64_t nhashes, uint32_t tg_total, int32_t tg_sel);
uint64_t orc_hash_bundle_data(const uint64_t* data, uint32_t lanes, uint32_t comps_stride,
                              uint32_t comps, uint32_t level_stride, uint32_t level, uint32_t n);
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
