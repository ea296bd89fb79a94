/*
 * boostcom.h -- C ABI of libboostcom.so, the B200-native hot path of BoostCom
 * (arXiv 2407.07308): BGV word-wise encrypted comparison over non-power-of-two
 * cyclotomic rings, batched over RNS ciphertexts, hand-written for sm_100a.
 *
 * Citations: P:<n> = PAPER.md line n (section named alongside); R<k> = reading k
 * in DESIGN.md §3 (where the paper is silent).
 *
 * Problem statement (§1): "compares pairs of encrypted data to generate an
 * encrypted result that indicates whether they are equivalent, less than, or
 * greater than"; the result "returns encrypted '1' when a<b or encrypted '0'
 * otherwise" (§2.1).
 *
 * Conventions
 * -----------
 *  - All pointers named `d_*` or carried in bc_ct are DEVICE pointers on the
 *    context's device; `h_*` are HOST pointers.  Nothing is retained past
 *    return except by *_async calls until their event completes.
 *  - Ciphertext batches are caller-owned device memory with layout
 *    u64[batch][parts][level][n], limb-major, canonical residues in [0, q_i),
 *    in EVALUATION form: E[k] = a(omega_i^{z_k}), z_k the k-th element of Z_m^*
 *    in ascending order (§2.2, Listing 2; R3).
 *    `level` = number of ciphertext primes present (1 .. n_cipher).
 *  - Workspace: caller-owned device memory of at least bc_workspace_bytes().
 *  - Every call returns a bc_status; no partial output is valid on error;
 *    bc_last_error() gives a thread-local message.
 *  - ctx and keys are immutable after creation: concurrent calls on distinct
 *    streams with distinct workspaces are safe.
 *  - There is no CPU fallback: every arithmetic step runs in CUDA kernels.
 */
#ifndef BOOSTCOM_H
#define BOOSTCOM_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BC_OK = 0,
    BC_E_ARG = 1,       /* bad argument (null, size mismatch)                   */
    BC_E_PARAM = 2,     /* parameters unusable (NotEnoughPrimes, non-cyclic ...) */
    BC_E_RANGE = 3,     /* word out of range for (d, l, base)  (SPEC OutOfRange) */
    BC_E_LEVEL = 4,     /* level mismatch / out of levels                        */
    BC_E_KEY = 5,       /* missing Galois key                                    */
    BC_E_NOISE = 6,     /* noise budget exhausted (reported by probes)           */
    BC_E_CONSUMED = 7,  /* non-blocking handle already waited on                 */
    BC_E_CUDA = 8,      /* CUDA runtime failure                                  */
    BC_E_OOM = 9,       /* workspace too small                                   */
    BC_E_INTERNAL = 10
} bc_status;

/* Parameter set (Table 3; readings R1, R5, R6, R8).  The chain
 * q_0..q_{n_cipher-1} is the n_cipher smallest primes >= 2^(cipher_bits-1) with
 * q = 1 mod lcm(p, m, M), M = 2^ceil(log2(2m-1)); the n_special special
 * primes continue the same ascending search.  Key switching is hybrid with
 * digits of `alpha` consecutive primes (R8, R14).  circuit: 'U' univariate
 * (digits in [0,(p-1)/2], base (p+1)/2) or 'B' bivariate (digits in [0,p)).
 * d digits per F_{p^D} slot, l slots per word (Table 3 "(d l)", F1). */
typedef struct {
    uint32_t p, m;
    char circuit;
    uint32_t d, l;
    uint32_t n_cipher, cipher_bits;
    uint32_t n_special, special_bits;
    uint32_t alpha;
    uint32_t compact_span;   /* slot compaction offsets |delta| <= span blocks (0 -> 3), R17 */
    uint32_t schedule;       /* digit circuits: 0 or 16 = R16, 23 = R23 baby-step / giant-step, 26 = R26
                              * (bivariate two-dimensional Paterson-Stockmeyer, univariate as R23) (SURVEY
                              * §8(f) f2: "2p-6 (Bivariate case) and sqrt(p-3)+O(log p)
                              * (Univariate case)"), 27 = R27 (R26 with one scale-down per sum of
                              * products: §8(f) f1 lazy ModDown); anything else -> BC_E_PARAM */
    uint32_t bluestein;      /* 0: power-of-two Bluestein length; 1: mixed radix (R25, SURVEY §8(f)
                              * f3: the smallest 256 r N' or 2^k >= 2m - 1; prime m, shapes 9 x 32 and
                              * 3 x 128 -- others BC_E_PARAM) */
} bc_params;

typedef struct {
    uint32_t n, m, M, D, S, ints_per_ct, n_cipher, n_special, dnum, g;
    uint32_t base;           /* digit base: p ('B') or (p+1)/2 ('U')      */
    uint32_t n_galois;       /* number of Galois keys keygen generates    */
} bc_info;

typedef struct bc_ctx bc_ctx;     /* params + device tables; immutable after create */
typedef struct bc_keys bc_keys;   /* pk, relin key, Galois keys (device-resident)   */
typedef struct bc_sk bc_sk;       /* secret key (host copy + device eval form)      */
typedef struct { void *data; uint32_t batch, level; } bc_ct;  /* VIEW, 2 parts */
typedef struct { void *event; void *stream; int consumed; } bc_handle;

/* ---- context ------------------------------------------------------------- */
bc_status bc_ctx_create(const bc_params *prm, int device, bc_ctx **out);
void bc_ctx_destroy(bc_ctx *ctx);
bc_status bc_ctx_info(const bc_ctx *ctx, bc_info *out);
/* h_out[n_cipher + n_special] = the moduli; h_omega[...] = omega_i (R2). */
bc_status bc_ctx_moduli(const bc_ctx *ctx, uint64_t *h_out, uint64_t *h_omega);
/* slot algebra (R5): h_G[D+1] field polynomial, h_zeta[D], h_t[S] slot exponents */
bc_status bc_ctx_slots(const bc_ctx *ctx, int64_t *h_G, int64_t *h_zeta, int64_t *h_t);
/* host only (no device): the digit circuit a context with these (p, circuit, schedule) evaluates --
 * k = the R23 baby-step size (0 for R16; R26 bivariate: k1 << 8 | k2), products = ct x ct multiplications per digit (EQ
 * included), depth = its multiplicative depth (R16 / R23; P:71's 3p-5 for R16 bivariate).
 * BC_E_PARAM for p not an odd prime <= 257, circuit not 'U'/'B', schedule not 0/16/23/26/27. */
bc_status bc_circuit_plan(uint32_t p, char circuit, uint32_t schedule, uint32_t *k, uint32_t *products,
                          uint32_t *depth);
/* Galois elements keygen generates keys for (Frobenius p^k, rotations) */
bc_status bc_ctx_galois(const bc_ctx *ctx, uint32_t *h_out);
size_t bc_ct_bytes(const bc_ctx *ctx, uint32_t batch, uint32_t level);
/* device workspace needed by compare/min/max/select/compact on `batch` pairs
 * (computed by a dry run of the schedule; a smaller workspace makes the
 * library process the batch in chunks, never fail, down to 1 pair). */
size_t bc_workspace_bytes(bc_ctx *ctx, uint32_t batch);

/* ---- keys (R7, R8) --------------------------------------------------------- */
bc_status bc_keygen(bc_ctx *ctx, uint64_t seed, bc_sk **sk, bc_keys **keys);
void bc_sk_destroy(bc_sk *sk);
void bc_keys_destroy(bc_keys *keys);

/* ---- encode / encrypt / decrypt (R6, R9, R10) -------------------------------- */
/* words[batch * ints_per_ct] (little-endian digits) -> batch
 * ciphertexts at the top level.  ct_index0 = global index of the first
 * ciphertext (drives the counter-based sampler, R7).  Word j occupies the l slots
 * from floor(j / wpr) * S1 + (j mod wpr) * l, wpr = floor(S1 / l) (R6: rows of S1
 * slots for hypercube slot structures such as p10's 3470 x 2; S1 = S when cyclic). */
bc_status bc_encrypt(bc_ctx *ctx, const bc_keys *keys, const uint64_t *h_words, uint32_t batch,
                     uint64_t seed, uint64_t ct_index0, bc_ct out, void *d_ws, size_t ws_bytes,
                     void *stream);
/* slot form: h_slots[batch][S][D] F_p coefficients (int16) -> ciphertexts */
bc_status bc_encrypt_slots(bc_ctx *ctx, const bc_keys *keys, const int16_t *h_slots,
                           uint32_t batch, uint64_t seed, uint64_t ct_index0, bc_ct out,
                           void *d_ws, size_t ws_bytes, void *stream);
/* decrypt to slot values h_slots[batch][S][D] (int16, canonical in [0,p)) */
bc_status bc_decrypt_slots(bc_ctx *ctx, const bc_sk *sk, bc_ct in, int16_t *h_slots,
                           void *d_ws, size_t ws_bytes, void *stream);
/* decrypt words (as_bits = 0) or result bits from block slot 0 (as_bits = 1):
 * h_out[batch * ints_per_ct] */
bc_status bc_decrypt(bc_ctx *ctx, const bc_sk *sk, bc_ct in, uint64_t *h_out, int as_bits,
                     void *d_ws, size_t ws_bytes, void *stream);
/* plaintext polynomial (coefficients mod p) of a ciphertext: h_out[batch][n] */
bc_status bc_decrypt_poly(bc_ctx *ctx, const bc_sk *sk, bc_ct in, int64_t *h_out,
                          void *d_ws, size_t ws_bytes, void *stream);

/* ---- comparison (§8(a) a7-a9) ---------------------------------------- */
bc_status bc_compare(bc_ctx *ctx, const bc_keys *keys, bc_ct a, bc_ct b, bc_ct lt_out,
                     bc_ct eq_out, void *d_ws, size_t ws_bytes, void *stream);
bc_status bc_compare_lt(bc_ctx *ctx, const bc_keys *keys, bc_ct a, bc_ct b, bc_ct out,
                        void *d_ws, size_t ws_bytes, void *stream);
bc_status bc_compare_eq(bc_ctx *ctx, const bc_keys *keys, bc_ct a, bc_ct b, bc_ct out,
                        void *d_ws, size_t ws_bytes, void *stream);
/* out = x2 + bcast(cond) * (x1 - x2)  (Listing 4 straightlining) */
bc_status bc_select(bc_ctx *ctx, const bc_keys *keys, bc_ct cond, bc_ct x1, bc_ct x2, bc_ct out,
                    void *d_ws, size_t ws_bytes, void *stream);
bc_status bc_min(bc_ctx *ctx, const bc_keys *keys, bc_ct a, bc_ct b, bc_ct out, void *d_ws,
                 size_t ws_bytes, void *stream);
bc_status bc_max(bc_ctx *ctx, const bc_keys *keys, bc_ct a, bc_ct b, bc_ct out, void *d_ws,
                 size_t ws_bytes, void *stream);
/* output level of compare_lt / select for an input level (for sizing outputs) */
uint32_t bc_compare_out_level(bc_ctx *ctx, uint32_t level, int which /*0 lt, 1 eq, 2 min*/);
/* compare_lt on HOST buffers (the end-to-end call; P:440's host<->device staging, pipelined): h_a, h_b =
 * batch ciphertexts [batch][2][level][n] u64 in host memory (pinned for the copies to overlap), h_out =
 * [batch][2][bc_compare_out_level(level, 0)][n].  The batch runs in chunks of `chunk` pairs (0: batch / 4):
 * the host->device copy of chunk i+1 and the device->host copy of chunk i-1 run on a library copy stream
 * while chunk i is compared on `stream` (events only, the host is never blocked).  d_stage: device buffer of
 * bc_host_stage_bytes(ctx, chunk, level) bytes (two slots of inputs + output), d_ws as bc_compare_lt (per
 * chunk).  `stream` completes after the last output word has reached h_out.  Words identical to
 * bc_compare_lt.  BC_E_ARG for a short staging buffer or null pointers. */
size_t bc_host_stage_bytes(bc_ctx *ctx, uint32_t chunk, uint32_t level);
bc_status bc_compare_lt_host(bc_ctx *ctx, const bc_keys *keys, const uint64_t *h_a, const uint64_t *h_b,
                             uint32_t batch, uint32_t level, uint64_t *h_out, uint32_t chunk, void *d_stage,
                             size_t stage_bytes, void *d_ws, size_t ws_bytes, void *stream);

/* ---- vectors of ciphertexts: min/max tournament, rank sort -------------- */
/* Each element v[i] is a batch of `batch` ciphertexts (the same batch for all i); the operation
 * is slot-wise across the T elements.
 * bc_min_tree / bc_max_tree (R20): fixed tree over element indices -- round r pairs
 *   (i, i + 2^r) for i = 0 mod 2^(r+1), the lower index is `a` of min(a, b) = b + LT(a,b)(a - b)
 *   (max: a + LT(a,b)(b - a)); unpaired elements pass through.  The tree does not depend on how
 *   the elements are later sharded over GPUs.  out.level = bc_vec_out_level(ctx, 0|1, ...).
 * bc_sort (R21): out[k] = k-th smallest element (ties by index), via ranks
 *   rank_j = #{i: x_i < x_j or (x_i = x_j and i < j)} and out_k = sum_j [rank_j = k] x_j with
 *   [v = 0] = 1 - v^(p-1); needs T <= p and all inputs at one level; out[T] views at
 *   bc_vec_out_level(ctx, 2, ...).
 * Everything runs inside the caller's workspace of at least bc_vec_workspace_bytes() bytes (no
 * chunking: BC_E_OOM if smaller). */
bc_status bc_min_tree(bc_ctx *ctx, const bc_keys *keys, const bc_ct *v, uint32_t T, bc_ct out, void *d_ws,
                      size_t ws_bytes, void *stream);
bc_status bc_max_tree(bc_ctx *ctx, const bc_keys *keys, const bc_ct *v, uint32_t T, bc_ct out, void *d_ws,
                      size_t ws_bytes, void *stream);
bc_status bc_sort(bc_ctx *ctx, const bc_keys *keys, const bc_ct *v, uint32_t T, bc_ct *out, void *d_ws,
                  size_t ws_bytes, void *stream);
/* which: 0 min tree, 1 max tree, 2 sort; levels[T] = element levels.  0 on error. */
uint32_t bc_vec_out_level(bc_ctx *ctx, int which, const uint32_t *levels, uint32_t T);
size_t bc_vec_workspace_bytes(bc_ctx *ctx, int which, const uint32_t *levels, uint32_t T, uint32_t batch);

/* ---- non-blocking comparison (a11, Listing 5) -------------------------
 * enqueues compare_lt on side_stream (after whatever is already queued there: the caller orders the
 * inputs' producers before it) and records an event in h; never waits on the device (batches larger
 * than the workspace run chunk after chunk on side_stream); bc_wait makes joiner_stream wait for it. */
bc_status bc_compare_lt_async(bc_ctx *ctx, const bc_keys *keys, bc_ct a, bc_ct b, bc_ct out,
                              void *d_ws, size_t ws_bytes, void *side_stream, bc_handle *h);
bc_status bc_wait(bc_handle *h, void *joiner_stream);   /* BC_E_CONSUMED on 2nd wait */

/* ---- CUDA graphs (launch-bound schedules replayed without host work) ----------
 * capture_begin starts a thread-local capture on `stream`; every library call then issued on it (and on
 * the side streams those calls fork to and join back) is recorded instead of executed; capture_end
 * instantiates the graph.  A replay (bc_graph_launch) re-runs the recorded kernels on the same device
 * buffers (ciphertexts, workspaces), so their contents are read anew and no host work (schedule
 * planning, launches) is repeated.  Errors: BC_E_ARG (null), BC_E_CUDA (capture not allowed, e.g. a
 * call that must synchronise). */
typedef struct bc_graph bc_graph;
bc_status bc_graph_capture_begin(void *stream);
bc_status bc_graph_capture_end(void *stream, bc_graph **out);
bc_status bc_graph_launch(bc_graph *g, void *stream);
void bc_graph_destroy(bc_graph *g);

/* ---- private_q (Listings 3-5 at P:511-554, R24) ----------
 * out[i] = ((data[i] + op1) c_0 + (data[i] op1) c_1) + data[i]^e c_2, c_j = bcast(EQ(q, codes[j]))
 * (codes: add, mult, power words; q, codes: words in every integer block; op1: one ciphertext;
 * e >= 1 a plaintext exponent, left-to-right binary powering).  data: batch N; q, op1: batch 1;
 * codes: batch 3.  side == NULL: blocking (Listing 4), everything on `stream` with ws.  side != NULL:
 * non-blocking (Listing 5): the EQs and broadcasts run on `side` with ws_side, ordered after the work
 * already on `stream` and joined by an event before the combination; the host never waits.  ws and
 * ws_side must stay untouched until `stream` has passed the call.  Bits are identical either way.
 * out: batch >= N at level bc_private_query_level(...).  Errors: BC_E_ARG (shapes, e = 0, missing
 * side workspace), BC_E_LEVEL (levels), BC_E_OOM (workspace). */
uint32_t bc_private_query_level(bc_ctx *ctx, uint32_t n_data, uint32_t data_level, uint32_t q_level,
                                uint32_t op1_level, uint32_t e);
/* side = 0: whole query (blocking; also an upper bound for the main stream's share), 1: the side
 * stream's share (EQs + broadcasts) */
size_t bc_private_query_workspace_bytes(bc_ctx *ctx, uint32_t n_data, uint32_t data_level, uint32_t q_level,
                                        uint32_t op1_level, uint32_t e, int side);
bc_status bc_private_query(bc_ctx *ctx, const bc_keys *keys, bc_ct data, bc_ct q, bc_ct codes, bc_ct op1, uint32_t e,
                           bc_ct out, void *ws, size_t ws_bytes, void *ws_side, size_t ws_side_bytes, void *stream,
                           void *side);

/* ---- primitives (each a §8(a) row; used by the parity tests) ---------------------- */
/* a1/a2: batched Bluestein NTT over `npoly` polynomials of `nlimb` limbs each,
 * limb i mapped to modulus index prime0 + i; layout u64[npoly][nlimb][n]. */
bc_status bc_ntt_fwd(bc_ctx *ctx, const void *d_in, void *d_out, uint32_t npoly, uint32_t nlimb,
                     uint32_t prime0, void *d_ws, size_t ws_bytes, void *stream);
bc_status bc_ntt_inv(bc_ctx *ctx, const void *d_in, void *d_out, uint32_t npoly, uint32_t nlimb,
                     uint32_t prime0, void *d_ws, size_t ws_bytes, void *stream);
/* a3: tensor product, out = 3-part u64[batch][3][level][n] */
bc_status bc_tensor(bc_ctx *ctx, bc_ct a, bc_ct b, void *d_out, void *stream);
/* a4: automorphism sigma_t on both parts (no key switch) */
bc_status bc_automorph(bc_ctx *ctx, bc_ct a, uint32_t t, bc_ct out, void *stream);
/* a5: key switch of one polynomial batch d[batch][level][n] (eval) with the key
 * for Galois element t (t = 0: relinearisation key); out u64[batch][2][level][n] */
bc_status bc_keyswitch(bc_ctx *ctx, const bc_keys *keys, const void *d_poly, uint32_t batch,
                       uint32_t level, uint32_t t, void *d_out, void *d_ws, size_t ws_bytes,
                       void *stream);
/* a6: modulus switch of a 2-part batch from level to level-1 */
bc_status bc_modswitch(bc_ctx *ctx, bc_ct a, bc_ct out, void *d_ws, size_t ws_bytes, void *stream);
/* a3+a5+a6: out = R15 fused product: tensor, ModUp + KIP of d2, one scale-down by P q_{level-1} */
bc_status bc_mul(bc_ctx *ctx, const bc_keys *keys, bc_ct a, bc_ct b, bc_ct out, void *d_ws,
                 size_t ws_bytes, void *stream);
/* a4+a5: rotation (slot s receives slot s+k) and Frobenius sigma_{p^k} */
bc_status bc_rotate(bc_ctx *ctx, const bc_keys *keys, bc_ct a, int32_t k, bc_ct out, void *d_ws,
                    size_t ws_bytes, void *stream);
bc_status bc_frobenius(bc_ctx *ctx, const bc_keys *keys, bc_ct a, uint32_t k, bc_ct out,
                       void *d_ws, size_t ws_bytes, void *stream);
/* a8: digit extraction: out = d digit ciphertexts u64[batch][d][2][level][n] */
bc_status bc_extract(bc_ctx *ctx, const bc_keys *keys, bc_ct a, void *d_out, void *d_ws,
                     size_t ws_bytes, void *stream);

/* ---- slot compaction (a10, Fig. 7) ------------------------------------- */
/* h_useful[n_in * ints_per_ct] (1 = block holds a useful word).  The R17 greedy plan
 * packs the useful blocks into as few ciphertexts as the offsets |delta| <= compact_span
 * allow (= ceil(useful / ints_per_ct) for the Fig. 7 strided pattern), one plaintext
 * mask product + rotation per (input, output, offset) group, then one modulus switch.
 * out has capacity n_in cts at level in.level - 1; *n_out is set; h_dest[n_in * ints]
 * receives the destination block (out_ct * ints_per_ct + block) of every useful block,
 * -1 elsewhere. */
/* host only (no device): the R17 plan bc_compact uses for a usefulness pattern (nin x ints bytes, 1 =
 * useful): dest[c*ints + b] = c' * ints + b' (its output ciphertext and block) or -1; wpr = blocks per
 * row (R6).  BC_E_ARG on null pointers, ints = 0, wpr = 0 or wpr > ints. */
bc_status bc_compact_plan(uint32_t ints, uint32_t span, uint32_t wpr, const uint8_t *h_useful, uint32_t nin,
                          int32_t *h_dest, uint32_t *n_out);
bc_status bc_compact(bc_ctx *ctx, const bc_keys *keys, bc_ct in, const uint8_t *h_useful,
                     bc_ct out, uint32_t *n_out, int32_t *h_dest, void *d_ws, size_t ws_bytes,
                     void *stream);

/* NTT kernel family (results identical, a1/a2): 0 = binary64 register-blocked passes (default; the
 * persistent column passes for R = 256, mixed-radix rows for the R25 lengths), 1 = radix-2 integer
 * shared-memory passes (reference kernels for tests), 2-7 = 64-bit integer Shoup register passes,
 * 10-17 = binary64 pass-shape variants (17: non-persistent column passes), 20 = the fused
 * thread-block-cluster kernel (ntt4.cu; 256 x 256 prime-m shapes, else as 0) */
void bc_set_ntt_impl(int impl);
/* tuning knobs (benchmarks / tests): "ntt_timing" (0/1, see bc_ntt_timing), "phase_timing" (0/1, see
 * bc_phase_timing), "vec_chunk" = max ciphertext pairs per batched compare inside bc_min_tree/bc_max_tree/
 * bc_sort (0 = one batch per round; bounds the workspace, never changes bits), "ntt_group_bytes" = transform
 * scratch per launch group (default: the whole batch in one group; smaller groups measured slower on B200),
 * "kip_blocked" (1: batch-blocked key inner product), "f64_elem" (1: binary64 element-wise kernels),
 * "nttc_variant" / "nttc_clusters" (the fused cluster transform of bc_set_ntt_impl(20); nttc_clusters
 * returns the occupancy query's cluster count), "ntt_epi" (1: the modulus-switch / ModDown scale-sub
 * and the fused ModDown epilogue run inside pass C of the forward transform of delta; 0, default: separate
 * kernels -- measured faster on B200), "ntt_lean" (4 default: pass-C staging tile as exchange buffer, 3 CTAs per SM; 0: round-2 passes; 1-3:
 * tables read through L2 and / or the staging tile as exchange buffer), "ntt_persist_occ" (cap of the persistent passes' CTAs per SM),
 * "ntt_split" (two-stream transform calls), "axpy" (1, default: a + c x of the digit circuits' linear
 * combinations in one kernel), "ptsum" (1, default: each extracted digit's kappa-weighted sum in one kernel),
 * "lift_blocks" (row-block cap of the binary64 lifts, default 16).  None changes a result bit.  Returns 0 if
 * known (-1 if not). */
int bc_tune(const char *key, int64_t value);
/* live NTT timing: after bc_tune("ntt_timing", 1) every forward/inverse Bluestein NTT call records
 * a CUDA event pair on its stream.  bc_ntt_timing synchronises those events and returns (then
 * clears) the summed duration in ms, the number of limb-transforms and of calls.  0 on success. */
int bc_ntt_timing(double *ms, uint64_t *limb_transforms, uint64_t *calls);
/* the same, also returning how many of the limb-transforms were inverse ones (composite m: those include
 * the Barrett division by Phi_m, which the roofline counts as extra work) */
int bc_ntt_timing_split(double *ms, uint64_t *limb_transforms, uint64_t *inverse_limb_transforms, uint64_t *calls);
/* with bc_tune("phase_timing", 1): an event pair (and an NVTX range of the same name) around each
 * leaf phase of the comparison schedule on its stream -- 0 extract (a8), 1 digit_circuit (a7),
 * 2 lexicographic (a9), 3 broadcast_select (R17), 4 compaction (a10), 5 private_query_main (R24);
 * bc_phase_timing synchronises them and returns ms[6] and calls[6] since the last call (0, or -1
 * on a CUDA error).  The NVTX ranges are always emitted. */
int bc_phase_timing(double *ms, uint64_t *calls);
/* number of CUDA kernel launches issued by this thread since the last reset */
uint64_t bc_launch_count(int reset);
const char *bc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
