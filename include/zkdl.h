/*
 * zkdl.h — C ABI of libzkdl: the B200 (sm_100a) prover hot path of zkDL
 * (arXiv 2307.16273).  Citations: P:Lnnn = PAPER.md line; Dn = DESIGN.md §3.
 *
 * Conventions for every entry point
 *  - Field elements crossing the ABI are zk_fr: 32-byte little-endian canonical
 *    integers < p (D1).  A non-canonical input returns ZK_ERR_NONCANONICAL.
 *  - "d_" pointers are DEVICE pointers, borrowed: the library never frees them,
 *    they must stay valid until the context stream has executed the call.
 *    Int32 tensors are contiguous row-major; Fr tables are contiguous arrays of
 *    32-byte elements in the library's internal Montgomery form (produced by
 *    zk_embed_i32 / zk_eq_table; convert with zk_fr_table_to_canonical).
 *    Device buffers must be 16-byte aligned (torch allocations are 256-B aligned).
 *  - Host pointers ("out", "proof", "point_out", ...) are caller-allocated.
 *    Calls that return host values enqueue their work on the context stream and
 *    synchronise that stream once before returning.  Calls without host
 *    outputs are asynchronous (stream-ordered).
 *  - Sizes are powers of two given as log2 ("zero-padding may be
 *    applied"); the Python layer pads.  Variables are bound LSB-first (D2).
 *  - Every call returns a zk_status; zk_last_error(ctx) describes the last
 *    failure.  There is no CPU fallback: without a CUDA device, calls return
 *    ZK_ERR_CUDA.
 *  - One context per host thread.  Scratch memory comes from the stream-ordered
 *    CUDA memory pool of the context's device.
 */
#ifndef ZKDL_H
#define ZKDL_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct zk_ctx zk_ctx;
typedef struct zk_transcript zk_transcript;
typedef struct { uint8_t b[32]; } zk_fr;

typedef enum {
    ZK_OK = 0,
    ZK_ERR_ARG = -1,            /* bad size / null pointer / non power of two */
    ZK_ERR_RANGE = -2,          /* input outside the (Q+R)-bit range */
    ZK_ERR_NONCANONICAL = -3,   /* field element >= p */
    ZK_ERR_OOM = -4,
    ZK_ERR_CUDA = -5,
    ZK_ERR_NCCL = -6,
    ZK_ERR_UNIMPLEMENTED = -7,
    ZK_ERR_INTERNAL = -8,
    ZK_REJECT = 1               /* host verifiers: a well-formed proof that does not verify */
} zk_status;

/* ------------------------------------------------------------------ context */
/* device: CUDA ordinal; cuda_stream: a cudaStream_t (NULL = the legacy default stream). */
zk_status zk_ctx_create(int device, void* cuda_stream, zk_ctx** out);
void zk_ctx_destroy(zk_ctx* ctx);
const char* zk_last_error(const zk_ctx* ctx);
/* Library version string and the number of kernel launches issued by this context so far. */
const char* zk_version(void);
uint64_t zk_ctx_launch_count(const zk_ctx* ctx);
zk_status zk_ctx_synchronize(zk_ctx* ctx);
/* Cap the grid of the context's persistent kernels (the one-launch small-statement sumcheck) at
 * `sms` CTAs, at most one per SM (0 = every SM, the default).  Several contexts on several streams
 * with budgets that add up to the SM count prove independent statements side by side instead of
 * each latency-bound statement spreading thinly over the whole GPU.  Never changes any output. */
zk_status zk_ctx_set_sm_budget(zk_ctx* ctx, uint32_t sms);
/* Allow (1, the default) or forbid (0) the context's persistent spin-waiting kernels (the one-launch
 * small-statement sumcheck and its continuation): with 0 every sumcheck round is its own launch, so work on
 * this context never holds SMs while waiting for CTAs that other streams keep from being scheduled (the
 * co-residency a cooperative grid assumes).  For work proved beside another stream's persistent kernels.
 * Never changes any output. */
zk_status zk_ctx_set_persistent(zk_ctx* ctx, int allow);
/* Per-launch profiling: while enabled, every kernel launch of the context is bracketed by two
 * CUDA events on the context stream.  zk_ctx_profile_read synchronises, writes one line per kernel
 * "name<TAB>launches<TAB>total_ms\n" (NUL-terminated, cap bytes max) and clears the records. */
zk_status zk_ctx_profile(zk_ctx* ctx, int enable);
/* Restrict profiling to one kernel: name is a kernel's base name (every template instantiation
 * "name<...>" matches); NULL or "" = every kernel.  Lets one kernel be timed inside a region
 * without bracketing all the others. */
zk_status zk_ctx_profile_filter(zk_ctx* ctx, const char* name);
zk_status zk_ctx_profile_read(zk_ctx* ctx, char* out, uint64_t cap);

/* --------------------------------------------------- Fiat-Shamir transcript (D3)
 * The 32-byte state lives in device memory; absorb/challenge run on the device.
 * zk_transcript_absorb: tag is a NUL-terminated ASCII string of <= 255 bytes,
 *   msg a HOST buffer of len bytes (asynchronous; msg may be reused on return).
 * zk_transcript_challenges: n challenges with the same tag, returned to the host
 *   (synchronises).  zk_transcript_state copies the 32-byte state to the host. */
zk_status zk_transcript_new(zk_ctx* ctx, const uint8_t seed[32], zk_transcript** out);
zk_status zk_transcript_absorb(zk_transcript* tr, const char* tag, const void* msg, uint64_t len);
zk_status zk_transcript_challenges(zk_transcript* tr, const char* tag, uint32_t n, zk_fr* out);
zk_status zk_transcript_state(zk_transcript* tr, uint8_t out[32]);
/* Fork / join (D3d: independent statements get independent transcripts, so they can be proved
 * concurrently).  zk_transcript_fork: the parent draws challenge `tag` (one field element x) and *out
 * is a new transcript seeded with the canonical 32 bytes of x (as zk_transcript_new(x) would be);
 * it runs on child_ctx's stream (NULL: the parent's).  The fork kernel runs on the parent's stream:
 * order the child's first use after it (cudaEvent) when the streams differ.
 * zk_transcript_absorb_state: absorb(tag, <32-byte state of other>) on tr's stream; other's work must
 * be ordered before it.  Free a transcript only after every use on every stream is ordered before
 * its own stream's free (zk_transcript_free is stream-ordered on its ctx's stream). */
zk_status zk_transcript_fork(zk_transcript* parent, const char* tag, zk_ctx* child_ctx, zk_transcript** out);
zk_status zk_transcript_absorb_state(zk_transcript* tr, const char* tag, const zk_transcript* other);
void zk_transcript_free(zk_transcript* tr);

/* ------------------------------------------------------------ tables (rows a1, a2)
 * zk_embed_i32 (row a1): d_out[i] = v mod p (negatives -> p - |v|), Montgomery form.
 * zk_eq_table  (row a2):   d_out[b] = scale * prod_t (u_t b_t + (1-u_t)(1-b_t)),
 *   b in [0, 2^k), u_t <-> bit t of b (D2); scale NULL means 1.  k <= 32.
 * zk_mle_eval_* (P:L146 Eq. multilinear-extension): out = sum_b T[b] beta(u, b), m = log2 |T|.
 * zk_fr_table_to_canonical: d_out[i] = canonical 32-byte encoding of d_in[i] (may alias).
 * zk_fr_table_from_canonical: the inverse; returns ZK_ERR_NONCANONICAL if any input >= p. */
zk_status zk_embed_i32(zk_ctx* ctx, const int32_t* d_in, uint64_t n, void* d_out);
/* zk_widen_i16: d_out[i] = d_in[i] (int16 -> int32, sign-extended), asynchronous; both 16-byte aligned.
 *   The end-to-end transport of stacks whose entries fit 16 bits (the matmul operands of the FCN trace):
 *   half the host-to-device bytes, the int32 tensor the provers read is rebuilt on the device. */
zk_status zk_widen_i16(zk_ctx* ctx, const int16_t* d_in, uint64_t n, int32_t* d_out);
/* zk_undelta_i8: rebuild an int32 stack of n_slots slices of slot_elems entries from its first L slices (int16,
 *   d_base, [L][slot_elems]) and the int8 differences of every later slice to the slice L before it (d_delta,
 *   [n_slots - L][slot_elems]):  out[s] = base[s] (s < L),  out[s] = out[s - L] + delta[s - L] (s >= L).
 *   The end-to-end transport of the weight stacks (a weight changes by a few quantisation steps per SGD update,
 *   so the slice of the same layer one training step earlier, L slices back, differs by int8 values): ~1 byte
 *   per entry over PCIe instead of 2; the provers read the same int32 tensor.  slot_elems a multiple of 4;
 *   d_out 16-, d_base 8-, d_delta 4-byte aligned; asynchronous on the context stream. */
zk_status zk_undelta_i8(zk_ctx* ctx, const int16_t* d_base, const int8_t* d_delta, uint64_t slot_elems, uint32_t L,
                        uint32_t n_slots, int32_t* d_out);
zk_status zk_eq_table(zk_ctx* ctx, const zk_fr* point, uint32_t k, const zk_fr* scale, void* d_out);
zk_status zk_mle_eval_i32(zk_ctx* ctx, const int32_t* d_tab, uint32_t m, const zk_fr* point, zk_fr* out);
zk_status zk_mle_eval_fr(zk_ctx* ctx, const void* d_tab, uint32_t m, const zk_fr* point, zk_fr* out);
zk_status zk_fr_table_to_canonical(zk_ctx* ctx, const void* d_in, uint64_t n, void* d_out);
zk_status zk_fr_table_from_canonical(zk_ctx* ctx, const void* d_in, uint64_t n, void* d_out);

/* ------------------------------------------- matmul -> sumcheck (row a3)
 * Stacked product Y[n] = A[n] B[n], n < N.  A is stored [N][D1][D2] (trans_a = 0) or
 * [N][D2][D1] (trans_a = 1); B is stored [N][D2][D3] (trans_b = 0) or [N][D3][D2].
 * Transcript (D3a): absorb "mm/hdr" (logN, logD1, logD2, logD3 as u32le), draw
 * w ("mm/w" x logN), u1 ("mm/u1" x logD1), u3 ("mm/u3" x logD3).
 * Writes the restricted tables (Fr, Montgomery, flat index k*N + n, n minor):
 *     d_At[k][n] = sum_a beta(u1, a) A[n][a][k]     d_Bt[k][n] = sum_c B[n][k][c] beta(u3, c)
 * and returns (host) the point w||u1||u3 (logN + logD1 + logD3 elements) and the claim
 *     claim = Y~(w, u1, u3) = sum_{k,n} beta(w, n) At[k][n] Bt[k][n].
 * Follow with zk_sumcheck_prove(m = logN + logD2, n_eq = logN, K = 2, w, claim). */
typedef struct { uint32_t logN, logD1, logD2, logD3; uint32_t trans_a, trans_b; } zk_mm_shape;
zk_status zk_matmul_reduce(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_A, const int32_t* d_B, zk_mm_shape shape,
                           void* d_At, void* d_Bt, zk_fr* point_out, zk_fr* claim_out);

/* ------------------------------------- aggregated product sumcheck (rows a4-a6; Prot. 3 P:L504-527)
 * Proves  claim = sum_{x in {0,1}^m} beta(w, x_{<n_eq}) * prod_{k<K} T_k(x),  1 <= K <= 3.
 * d_tables[k]: Fr tables of 2^m elements (Montgomery), or int32 tables if bit k of i32_mask
 * is set (embedded on the fly).  The tables are NOT modified.  w: host, n_eq elements.
 * claim: host pointer, or NULL to let the prover compute it (it is then absorbed and
 * returned in claim_out).  Transcript (D3c): "sc/hdr" (m, n_eq, K) | "sc/claim" | per round
 * "sc/msg" (K+1 evaluations at X = 0..K: f_t for t < n_eq, g_t otherwise, D4) then
 * challenge "sc/r" | "sc/final" (T_k~(r)).
 * proof (host): u32le m, n_eq, K | claim | m*(K+1) evaluations | K finals; *proof_len is in/out.
 * proof == NULL with proof_len != NULL is a size query (nothing is proved, transcript untouched);
 * a too-small buffer returns ZK_ERR_ARG with the required size; proof == proof_len == NULL proves
 * without returning the proof bytes.
 * point_out (host, m elements) and finals_out (host, K elements) may be NULL. */
typedef struct { uint32_t m, n_eq, n_tables, i32_mask; const zk_fr* w; } zk_prod_stmt;
zk_status zk_sumcheck_prove(zk_ctx* ctx, zk_transcript* tr, const zk_prod_stmt* st, void* const* d_tables,
                            const zk_fr* claim, zk_fr* claim_out, uint8_t* proof, uint64_t* proof_len,
                            zk_fr* point_out, zk_fr* finals_out);

/* ------------------------------------------- claim reductions after the hot path
 * zk_reindex_prove — the re-indexing sumcheck, Eq. (sc-reindex) P:L262-270 (D20).
 *   d_X: int32 stack of N = 2^n slices of D = 2^d entries, row-major [N][D] (device, borrowed).  A
 *   point on X is (u over the D bits, then the N bits) (D2).  views[k]: N_k = 2^{logN} slots; slot j
 *   holds slice map[j] (host array, injective into [0, N); 0xffffffff = an all-zero slot), with the
 *   point u_k (host, logN elements); claims[k] = X_k~(u, u_k) (host, K <= 32); u: host, d elements.
 *   Transcript: "rx/hdr" (n, d, K, logN_0..logN_{K-1} as u32le) | "rx/claims" (K) | r_k = "rx/r" x K |
 *   the product sumcheck (D3c) over n variables of C(i) = sum_k r_k sum_j beta(u_k, j) [map_k[j] = i]
 *   and X~(u, i), n_eq = 0, claim sum_k r_k claims[k] given.  proof / proof_len / point_out (n) as in
 *   zk_sumcheck_prove; finals_out (host, 2): C~(r) (the verifier recomputes it from the maps) and
 *   X~(u, r), the single output claim on the stack.  Errors: ZK_ERR_RANGE (slot outside the stack),
 *   ZK_ERR_ARG (non-injective map, bad shape).  Synchronises the ctx stream once.
 * zk_relu_merge — the zkReLU aux-claim merge, P:L470 (D21), on the transcript
 *   that just proved zk_relu_prove: point = its final point (logB + logD: the j-bits w then the
 *   i-bits v), finals = its three finals aux~(0, v, w), aux~(1, v, w), aux~(0, v, Q+R-1).
 *   Transcript: rho = "relu/merge" | the product sumcheck (D3c) over (j, s) (logB + 1 variables, j
 *   first) of T(s, j) = sum_i beta(v, i) bit_j(word_s[i]) (s = 0: Z, s = 1: G_A) and W(s, j) =
 *   [s=0](beta(w, j) + rho^2 [j = Q+R-1]) + [s=1] rho beta(w, j), claim f0 + rho f1 + rho^2 f2.
 *   merged_out (host, 2): aux~(r_s, v, r_j) — the single merged claim — and W~(r); point_out:
 *   logB + 1 elements (r_j, then r_s).  Synchronises the ctx stream once. */
typedef struct { uint32_t logN; const uint32_t* map; const zk_fr* u; } zk_view;
zk_status zk_reindex_prove(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_X, uint32_t n, uint32_t d, uint32_t K,
                           const zk_view* views, const zk_fr* u, const zk_fr* claims, uint8_t* proof,
                           uint64_t* proof_len, zk_fr* point_out, zk_fr* finals_out);
zk_status zk_relu_merge(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA, uint32_t logD,
                        uint32_t Q, uint32_t R, const zk_fr* point, const zk_fr* finals, uint8_t* proof,
                        uint64_t* proof_len, zk_fr* point_out, zk_fr* merged_out);
/* zk_relu_merge_dev: the same merge, asynchronous, reading the point and finals from d_relu_out (the
 * zk_relu_prove_dev output of the same statement, device) and writing d_out = merge sumcheck proof
 * (zk_sumcheck_prove layout; finals = merged claim, W~(r)) | pad to 16 bytes | point (logB + 1
 * elements, canonical); d_out 16-byte aligned; d_out == NULL with out_len != NULL is a size query. */
zk_status zk_relu_merge_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA, uint32_t logD,
                            uint32_t Q, uint32_t R, const uint8_t* d_relu_out, uint8_t* d_out, uint64_t* out_len);

/* zk_hadamard_zero_prove — SURVEY §8(f) N2: Protocol 2's zero form (Eq. tensor-op-aggr P:L229-234,
 *   Protocol 2 P:L476-502) for the aggregated Hadamard product Y = A (.) B, D22:
 *     0 = sum_x beta(w, x) (Y(x) - A(x) B(x)),  x over m variables (the stack and the output index).
 *   d_Y, d_A, d_B: int32 tables of 2^m entries (device, borrowed; embedded mod p).  Transcript: "hd/hdr"
 *   (m as u32le) | w = "hd/w" x m | per round "sc/msg" (f_t at 0, 1, 2; beta(w_{<=t}) divided out, D4)
 *   then "sc/r" | "sc/final" (Y~(r), A~(r), B~(r)).  proof (host): u32le m | m x 3 evaluations |
 *   3 finals; proof_len in/out (proof == NULL: size query).  w_out (m), point_out (m), finals_out (3):
 *   host, may be NULL.  A false statement is not an error: the proof simply fails verification
 *   ((1 - w_0) f_0(0) + w_0 f_0(1) != 0).  Synchronises the ctx stream once. */
zk_status zk_hadamard_zero_prove(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Y, const int32_t* d_A,
                                 const int32_t* d_B, uint32_t m, uint8_t* proof, uint64_t* proof_len, zk_fr* w_out,
                                 zk_fr* point_out, zk_fr* finals_out);

/* zk_loss_grad_prove — SURVEY §8(f) N2: the loss-gradient family, Eq. (fcnn-GZ-last) P:L299-302,
 *   G_Z^(L) = Z^(L) - Y over the stacked instances (D24).  The relation is linear, so no
 *   sumcheck: at the verifier's point u the claims G_Z~(u), Z~(u), Y~(u) satisfy G_Z~(u) = Z~(u) - Y~(u)
 *   (linearity of the MLE); the three claims go to the commitments.  d_GZ, d_Z, d_Y: int32
 *   tables of 2^m entries (device, borrowed).  Transcript: "lg/hdr" (m as u32le) | u = "lg/u" x m |
 *   "lg/claims" (3 canonical values).  point_out (m) and claims_out (3): host, may be NULL.  A false
 *   statement is not an error: the claims simply fail the identity.  Synchronises the ctx stream once. */
zk_status zk_loss_grad_prove(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_GZ, const int32_t* d_Z,
                             const int32_t* d_Y, uint32_t m, zk_fr* point_out, zk_fr* claims_out);

/* ------------------------------------------- sharded product sumcheck (SURVEY §8(e), G = 2^s devices)
 * Rank g (of world = G, a power of two) holds entries [g 2^L, (g+1) 2^L) of every table, L = m - s:
 * the top s index bits (the last-bound variables, D2) are the rank id, so every round pair is local.
 * Protocol per round, driven by the caller:
 *   zk_sc_shard_partial(sh, d_part)  — this rank's K+1 partial evaluations (32-byte internal-form
 *                                      elements, already scaled by the rank's eq factor) into d_part;
 *   caller all-gathers the G partials in rank order into d_all (NCCL all_gather, G*(K+1)*32 bytes);
 *   zk_sc_shard_finish(sh, d_all)    — adds them mod p and runs the transcript step (identical on
 *                                      every rank, so no broadcast of challenges is needed).
 * When zk_sc_shard_local_log(sh) reaches the caller's threshold (or right away), zk_sc_shard_export
 * writes the K folded local tables ([K][2^local_log] elements), the caller all-gathers them
 * ([G][K][2^local_log]) and zk_sc_shard_adopt finishes every remaining round and the finals on each rank.
 * The transcript, proof bytes and point equal zk_sumcheck_prove's on the full tables for every G
 * (D3c).  zk_sc_shard_result copies them out (synchronises); all other calls are asynchronous.
 * d_local_tables follow zk_prod_stmt's i32_mask convention; claim as in zk_sumcheck_prove. */
typedef struct zk_sc_shard zk_sc_shard;
zk_status zk_sc_shard_create(zk_ctx* ctx, zk_transcript* tr, const zk_prod_stmt* st, void* const* d_local_tables,
                             const zk_fr* claim, uint32_t rank, uint32_t world, zk_sc_shard** out);
zk_status zk_sc_shard_partial(zk_sc_shard* sh, void* d_part);
zk_status zk_sc_shard_finish(zk_sc_shard* sh, const void* d_all);
uint32_t zk_sc_shard_rounds_done(const zk_sc_shard* sh);
uint32_t zk_sc_shard_local_log(const zk_sc_shard* sh);
zk_status zk_sc_shard_export(zk_sc_shard* sh, void* d_out);
zk_status zk_sc_shard_adopt(zk_sc_shard* sh, const void* d_full);
/* The exchange owned by the library (the context's NCCL communicator):
 * zk_nccl_unique_id: rank 0 creates the 128-byte communicator id (the caller broadcasts it, e.g. through
 *   torch.distributed); ZK_ERR_NCCL when libnccl.so.2 cannot be loaded.
 * zk_ctx_attach_nccl: every rank creates the communicator of `world` ranks (a power of two) on the
 *   context's device (collective: all ranks call it); the context owns it (zk_ctx_detach_nccl or
 *   zk_ctx_destroy frees it).
 * zk_sc_shard_prove_nccl: every remaining round of a shard created on an attached context with the same
 *   rank / world: per round this rank's K+1 partials are all-gathered as (K+1)*32 raw bytes (ncclUint8)
 *   on the context stream, added mod p and put through the transcript step on the device; below
 *   2^switch_log local entries the folded tables are all-gathered and every rank finishes alone.
 *   Asynchronous (no host synchronisation); then zk_sc_shard_result. */
zk_status zk_nccl_unique_id(uint8_t out[128]);
zk_status zk_ctx_attach_nccl(zk_ctx* ctx, const uint8_t id[128], int rank, int world);
zk_status zk_ctx_detach_nccl(zk_ctx* ctx);
zk_status zk_sc_shard_prove_nccl(zk_sc_shard* sh, uint32_t switch_log);
zk_status zk_sc_shard_result(zk_sc_shard* sh, uint8_t* proof, uint64_t* proof_len, zk_fr* point_out, zk_fr* finals_out,
                             zk_fr* claim_out);
void zk_sc_shard_free(zk_sc_shard* sh);

/* ----------------------------------------------------- zkReLU (rows a7, a8; Sec. 3, App. A)
 * zk_relu_tables (row a7): from Z, G_A (int32, D entries, Q+R <= 32 bits) writes
 *   sign = 1{Z < 0} (u8, D10), A = (1 - sign) Z', G_Z = (1 - sign) G_A' with Z' = round(Z / 2^R),
 *   G_A' = round(G_A / 2^R) half-up (D9), and optionally Z', G_A', R_Z = Z - 2^R Z',
 *   R_GA = G_A - 2^R G_A' (NULL to skip).  Returns ZK_ERR_RANGE (synchronising) if any
 *   input leaves [-2^{Q+R-1}, 2^{Q+R-1}).
 * zk_relu_prove (row a8): transcript (D3b): "relu/hdr" (logD, Q, R) | u_Z, u_A,
 *   u_GA, u_GZ | "relu/claims" (Z~(u_Z), A~(u_A), G_A~(u_GA), G_Z~(u_GZ)) | r, r', u_bin |
 *   logB + logD rounds of 4 evaluations (j bits first) | "relu/final" (aux~(0,v,w),
 *   aux~(1,v,w), aux~(0,v,Q+R-1)), with logB = ceil(log2(Q+R)).
 *   proof (host): u32le logD, Q, R | 4 claims | rounds x 4 evaluations | 3 finals; proof / proof_len
 *   follow zk_sumcheck_prove's size-query convention.
 *   claims_out (4), point_out (logB + logD) and finals_out (3) may be NULL. */
zk_status zk_relu_tables(zk_ctx* ctx, const int32_t* d_Z, const int32_t* d_GA, uint64_t D, uint32_t Q, uint32_t R,
                         uint8_t* d_sign, int32_t* d_A, int32_t* d_GZ, int32_t* d_Zp, int32_t* d_GAp, int32_t* d_RZ,
                         int32_t* d_RGA);
zk_status zk_relu_prove(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA, uint32_t logD,
                        uint32_t Q, uint32_t R, uint8_t* proof, uint64_t* proof_len, zk_fr* claims_out,
                        zk_fr* point_out, zk_fr* finals_out);

/* ------------------------------------------------ device-output provers (asynchronous)
 * The same proofs with every output written to caller-provided DEVICE memory.  These calls only
 * enqueue work on the context stream -- no host synchronisation, no pageable copies -- so a proving
 * window of families runs back to back and the caller synchronises once (zk_ctx_synchronize).
 * Kernel faults surface at that synchronisation.  d_out == NULL with out_len != NULL is a size query.
 * zk_matmul_prove (rows a3-a6): zk_matmul_reduce then zk_sumcheck_prove(m = logN + logD2,
 *   n_eq = logN, K = 2, w, claim) on the same transcript, identical bytes.  d_out layout:
 *   point w||u1||u3 (np = logN+logD1+logD3 elements, canonical) | claim (32 B) |
 *   sumcheck proof (zk_sumcheck_prove layout) | zero to 15 pad bytes to a 16-byte offset |
 *   sumcheck point r (m elements, canonical).  d_out must be 16-byte aligned.
 *   d_At, d_Bt: 2^(logN+logD2) Fr elements each (they hold the restricted tables on return), or
 *   NULL to use stream-ordered scratch.
 * zk_relu_prove_dev (rows a7, a8): zk_relu_prove with d_out = proof | pad to a 16-byte offset |
 *   point (logB + logD elements); d_out 16-byte aligned.
 *   Bit 0 of *d_range_flag (device u32, never cleared by the library) is set when an input leaves
 *   the (Q+R)-bit range; the caller checks it after synchronising (the proof is then meaningless).
 * zk_transcript_state_dev: copies the 32-byte state to device memory (stream-ordered). */
zk_status zk_matmul_prove(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_A, const int32_t* d_B, zk_mm_shape shape,
                          void* d_At, void* d_Bt, uint8_t* d_out, uint64_t* out_len);
zk_status zk_relu_prove_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA, uint32_t logD,
                            uint32_t Q, uint32_t R, uint8_t* d_out, uint64_t* out_len, uint32_t* d_range_flag);
zk_status zk_transcript_state_dev(zk_transcript* tr, void* d_out);
/* zk_relu_prove_chained_dev: zk_relu_prove_dev in the chained window (N3, D25): the points
 *   u_Z, u_A, u_GA, u_GZ are NOT drawn — they are given (d_pts: device, 4 x logD canonical elements, in
 *   that order), the points of the single claims the window's claim merges left on the Z, A, G_A, G_Z
 *   stacks.  The transcript is D3b without the four point draws; the proof's claims are the
 *   MLEs at the given points (the verifier checks them against the merged claims). */
zk_status zk_relu_prove_chained_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, const int32_t* d_GA,
                                    uint32_t logD, uint32_t Q, uint32_t R, const uint8_t* d_pts, uint8_t* d_out,
                                    uint64_t* out_len, uint32_t* d_range_flag);

/* ------------------------------------------- the claim merge (D25)
 * zk_claim_merge_dev — Protocol 1 line 8: the claims a window's operation families leave on
 *   views of one tensor family are reduced to ONE claim on its stack by Eq. (sc-reindex) in
 *   its general form (every claim with its own inner point).  The stack: N = 2^n slices of
 *   2^log_rows x 2^log_cols int32 entries, row-major (a point on it: col bits, row bits, slice bits; D2),
 *   read through `source`: 0 = d_X itself, 1 = A = 1{Z >= 0} round(Z / 2^R) formed from d_X = the Z
 *   words, 2 = G_Z = 1{Z >= 0} round(G_A / 2^R) from d_X = Z and d_X2 = G_A (Lemma 1; the
 *   tensors anchored by aux), 3 = the bits of d_X (aux(i, j) = bit j of X[i], j < R = the bit
 *   count, 2^log_cols columns, n = 0: the rescale's aux, D26).  views[k] (host): 2^logN slots, map[j] = the slice slot j holds
 *   (0xffffffff: an all-zero slot; injective).  d_pts (device, canonical): per claim, in order, its inner
 *   point v_k (log_rows + log_cols elements) then its slot point u_k (logN elements); d_claims (device,
 *   canonical): c_k = X_k~(v_k, u_k).  Transcript: "cm/hdr" (n, d, K, logN_k... u32le) | "cm/claims" |
 *   rho = "cm/rho" x K | phase A product sumcheck (D3c) over n + kappa variables (kappa = ceil log2 K)
 *   of P(i, k) = rho_k sum_j beta(u_k, j) [map_k[j] = i] and Rt(i, k) = X_i~(v_k), claim sum rho_k c_k |
 *   phase B product sumcheck over d = log_rows + log_cols variables of Wy(y) = sum_k beta(r_k, k)
 *   beta(v_k, y) and Xr(y) = sum_i beta(r_i, i) X(i, y), claim Rt~(r_i, r_k).
 *   d_out (device, 16-byte aligned, *out_len = capacity in / size out; NULL: size query): proof A |
 *   proof B (zk_sumcheck_prove layout each) | pad to 16 | point A (n + kappa) | point B (d) | the stack
 *   point (point B, then point A's first n elements) | the claim X~(stack point) (32 B).  Asynchronous.
 *   Errors: ZK_ERR_ARG (shape: K <= 8, n <= 16, log_rows, log_cols <= 16, d <= 30, at most 2048 view
 *   slots in all, n + kappa >= 1; map not injective), ZK_ERR_RANGE (slot outside the stack). */
typedef struct { uint32_t logN; const uint32_t* map; } zk_cm_view;
zk_status zk_claim_merge_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_X, const int32_t* d_X2, uint32_t source,
                             uint32_t R, uint32_t n, uint32_t log_rows, uint32_t log_cols, uint32_t K,
                             const zk_cm_view* views, const uint8_t* d_pts, const uint8_t* d_claims, uint8_t* d_out,
                             uint64_t* out_len);

/* ------------------------------------------- host verifiers (D23)
 * Verification replays the same sequence of rounds as proving with O(degree) field
 * operations per round: plain host code (verify.cu), no device, no context, callable anywhere.
 * st: a 32-byte transcript state (D3), in/out: the verifier's copy of the transcript before the
 * proof; on return the state after it (on accept equal to the prover's zk_transcript_state).
 * zk_htr_*: the D3 transcript on such a state (init from a seed, absorb, n challenges).
 * Every verifier returns ZK_OK (accept), ZK_REJECT with *fail = the failing 1-based round, -100 (final
 * identity), -1 (claim mismatch) or -101 (merge weight final), ZK_ERR_ARG (malformed proof bytes) or
 * ZK_ERR_NONCANONICAL.  The finals in the proof are claims on the committed tensors: the caller checks
 * them against the commitments (out of scope) or against the tensors themselves.
 * The statement's shape is the verifier's: every verifier takes the expected header (expect = (m, n_eq,
 *   K), (logD, Q, R), or m) and rejects a proof whose header differs (fail = -2) before reading further.
 * zk_verify_sumcheck: a zk_sumcheck_prove proof (Protocol 3, D3c transcript, D4 messages); w: the
 *   statement's n_eq = expect[1] eq point (host); claim: the claim the verifier expects, or NULL to take
 *   the proof's; point_out: m elements (host, may be NULL).
 * zk_verify_hadamard_zero: a zk_hadamard_zero_prove proof (Protocol 2 zero form, D22): round identities
 *   from c_0 = 0, final Y~(r) - A~(r) B~(r); w_out, point_out: m elements (may be NULL).
 * zk_verify_relu: a zk_relu_prove proof (App. A, D3b): the final identity of the six statements at the
 *   final point with the verifier's own beta, s, s' evaluations; point_out: logB + logD elements.
 *   pts: NULL (the points are drawn, D3b) or the chained form's given points (4 x logD, D25).
 * zk_verify_claim_merge: a zk_claim_merge_dev proof (proof A | proof B bytes, D25) for the verifier's own
 *   statement: n, d, the views (maps), per claim its point (v_k then u_k, host) and claimed value; checks
 *   both phases, P~ (fail -101) and Wy~ (fail -102) from the maps and points; point_out (d + n) and
 *   claim_out (1): the one claim left on the stack.
 * zk_verify_loss_grad: the loss-gradient claims (D24): replays "lg/hdr", u, "lg/claims" and checks
 *   G_Z~(u) = Z~(u) - Y~(u) (fail = -100); point_out: m elements.
 * zk_verify_relu_merge: a zk_relu_merge proof (D21) following the zkReLU proof whose point and finals
 *   are given: the verifier forms the claim and checks the weight final W~(r); point_out: logB + 1. */
zk_status zk_htr_init(const uint8_t seed[32], uint8_t st[32]);
zk_status zk_htr_absorb(uint8_t st[32], const char* tag, const void* msg, uint64_t len);
zk_status zk_htr_challenges(uint8_t st[32], const char* tag, uint32_t n, zk_fr* out);
zk_status zk_verify_sumcheck(uint8_t st[32], const uint8_t* proof, uint64_t proof_len, const uint32_t expect[3],
                             const zk_fr* w, const zk_fr* claim, zk_fr* point_out, int32_t* fail);
zk_status zk_verify_hadamard_zero(uint8_t st[32], const uint8_t* proof, uint64_t proof_len, uint32_t expect_m,
                                  zk_fr* w_out, zk_fr* point_out, int32_t* fail);
zk_status zk_verify_relu(uint8_t st[32], const uint8_t* proof, uint64_t proof_len, const uint32_t expect[3],
                         const zk_fr* pts, zk_fr* point_out, int32_t* fail);
zk_status zk_verify_loss_grad(uint8_t st[32], uint32_t m, const zk_fr* claims, zk_fr* point_out, int32_t* fail);
zk_status zk_verify_claim_merge(uint8_t st[32], uint32_t n, uint32_t d, uint32_t K, const zk_cm_view* views,
                                const zk_fr* pts, const zk_fr* claims, const uint8_t* proof, uint64_t proof_len,
                                zk_fr* point_out, zk_fr* claim_out, int32_t* fail);
zk_status zk_verify_relu_merge(uint8_t st[32], uint32_t logD, uint32_t Q, uint32_t R, const zk_fr* relu_point,
                               const zk_fr* relu_finals, const uint8_t* proof, uint64_t proof_len, zk_fr* point_out,
                               int32_t* fail);

/* ------------------------------------------- the top layer (D24, D26)
 * zk_loss_grad_prove_dev: zk_loss_grad_prove with device outputs, d_out = u (m canonical) | G_Z~(u),
 *   Z~(u), Y~(u) (canonical); asynchronous (the chained window's loss family).
 * zk_rescale_prove_dev — the top layer's rescale Z = 2^R Z' + R_Z, Z' = round(Z / 2^R) (half-up, D9),
 *   through the bits of Z (Eqs. aux-Z, zkrelu-Z and the Z' relation), at given points
 *   (d_pts: device, u_Z then u_P, logD canonical elements each: the window's claims on Z and Z', D25).
 *   Transcript (D26): "rs/hdr" (logD, Q, R) | "rs/claims" (Z~(u_Z), Z'~(u_P)) | r = "rs/r" | product
 *   sumcheck A (D3c, m = logB + logD, n_eq = 0, K = 2: W(i, j) = r beta(u_Z, i) s(j) + beta(u_P, i) s'(j)
 *   and aux(i, j), claim r Z~ + Z'~) | w = "rs/w" x m | product sumcheck B (D3c, n_eq = m, K = 2: aux and
 *   aux - 1, claim 0).  d_out (16-byte aligned): proof = u32le logD, Q, R | 2 claims | proof A | proof B,
 *   then pad to 16 | point A (m) | point B (m).  Bit 0 of *d_range_flag is set when Z leaves Q+R bits. */
zk_status zk_loss_grad_prove_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_GZ, const int32_t* d_Z,
                                 const int32_t* d_Y, uint32_t m, uint8_t* d_out, uint64_t* out_len);
zk_status zk_rescale_prove_dev(zk_ctx* ctx, zk_transcript* tr, const int32_t* d_Z, uint32_t logD, uint32_t Q,
                               uint32_t R, const uint8_t* d_pts, uint8_t* d_out, uint64_t* out_len,
                               uint32_t* d_range_flag);
/* zk_verify_rescale: a zk_rescale_prove_dev proof for expect = (logD, Q, R) at the given points (pts: u_Z then
 *   u_P, host): A's round identities from r Z~ + Z'~ and its weight final W~(r_A) (fail -101), B's from 0 in
 *   the eq form and its second final = first - 1 (fail -102).  claims_out (2): the proof's Z~(u_Z),
 *   Z'~(u_P); aux_out (2): aux~(r_A), aux~(r_B); point_out (2m): r_A then r_B. */
zk_status zk_verify_rescale(uint8_t st[32], const uint8_t* proof, uint64_t proof_len, const uint32_t expect[3],
                            const zk_fr* pts, zk_fr* claims_out, zk_fr* aux_out, zk_fr* point_out, int32_t* fail);

/* ----------------------------------------------------------------- diagnostics
 * zk_diag_fr_op: element-wise d_out[i] = op(d_a[i], d_b[i]) on Montgomery tables, op 0 add, 1 sub,
 *   2 mul, 3 inverse (Fermat), 4 negate, 5 square, 6 inverse (binary extended Euclid) (d_b may be NULL for 3-6).
 *   Used by the parity tests.
 * zk_diag_mul_bench: blocks x 256 threads each run 4 independent chains of `iters` Montgomery
 *   products on register-resident values (d_seed: 1024 elements; d_out: blocks*256 elements);
 *   bench.py times it to measure this implementation's sustained Fr-mul rate. */
zk_status zk_diag_fr_op(zk_ctx* ctx, int op, const void* d_a, const void* d_b, uint64_t n, void* d_out);
/* zk_diag_rowdot: out[r] = sum_c M[r][c] beta(point, c) (Montgomery, d_out: nrows Fr) through the CUDA-core
 * (use_tc = 0) or the tensor-core row-dot kernel of the matmul restriction with its cp.async producer
 * (use_tc = 1) or its TMA producer (use_tc = 2, the default path); cols a power of two. */
zk_status zk_diag_rowdot(zk_ctx* ctx, const int32_t* d_M, uint64_t nrows, uint32_t cols, const zk_fr* point,
                         void* d_out, int use_tc);
zk_status zk_diag_mul_bench(zk_ctx* ctx, const void* d_seed, uint32_t iters, uint32_t blocks, void* d_out);
/* zk_diag_fs_bench: n sequential transcript steps on one warp (mode 0: absorb 3 elements + squeeze,
 * 1: transcript-hash (BLAKE2s) compressions only, 2: out-of-line Montgomery products); d_out receives one element. */
zk_status zk_diag_fs_bench(zk_transcript* tr, uint32_t n, int mode, void* d_out);

#ifdef __cplusplus
}
#endif
#endif /* ZKDL_H */
