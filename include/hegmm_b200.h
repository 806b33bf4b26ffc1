/*
 * hegmm_b200.h -- C ABI of the B200 HE-primitive library (libhegmm_b200.so).
 *
 * This is the drop-in boundary for the reference's backend contract
 * `hegmm::Backend` (/root/reference/proj/include/hegmm/backend.hpp:107-127).
 * Each entry point replaces one virtual of that interface; a C++ adapter that
 * implements `hegmm::Backend` on top of these calls is given in
 * integration/bfv_gpu_backend.cpp and INTEGRATION.md.
 *
 *   hgm_ctx            <- one backend session (SlotBackend ctor, backend.cpp:114-116)
 *   hgm_encrypt        <- Backend::encrypt   (backend.hpp:113, backend.cpp:118-134)
 *   hgm_decrypt        <- Backend::decrypt   (backend.hpp:114, backend.cpp:136-139)
 *   hgm_add            <- Backend::he_add    (backend.hpp:116, backend.cpp:141-153)
 *   hgm_mul            <- Backend::he_mult   (backend.hpp:117, backend.cpp:155-167)
 *   hgm_cmul           <- Backend::he_cmult  (backend.hpp:118, backend.cpp:169-183)
 *   hgm_rot            <- Backend::he_rot    (backend.hpp:119, backend.cpp:185-197)
 *   hgm_stats / hgm_reset_stats / hgm_peak_live / hgm_set_phase / hgm_phase
 *                      <- Backend::stats/reset_stats/peak_live_ciphertexts/
 *                         set_phase/phase   (backend.hpp:121-126)
 *   hgm_apply_plan     <- apply_plan (lintrans.hpp:161-165, lintrans.cpp:433-461):
 *                         sum_z mask_z .* Rot(ct, z) with one hoisted ModUp
 *   hgm_matmul_batch   <- basic_mm / enhanced_mm (algorithms.hpp:59-66) over a
 *                         batch of independent instances in lockstep
 *
 * Conventions: every call returns HGM_OK (0) or an error code and never throws
 * across the ABI; hgm_last_error() gives the thread-local message.  Error codes
 * map to the reference exception types (errors.hpp:17-37):
 *   HGM_EDIM -> DimensionError, HGM_ECAP -> CapacityError,
 *   HGM_EOVERFLOW -> OverflowError, anything else -> Error.
 * Ciphertexts are immutable, reference counted handles owned by the caller
 * (hgm_ct_release).  Operations are recorded and executed lazily on the GPU;
 * hgm_decrypt / hgm_ct_export / hgm_flush force execution.
 * Slot semantics: slot_count = N/2 values per ciphertext row, values mod
 * t = 65537, decrypted values canonical in [0, t); rotation is cyclic over the
 * full N/2-slot row ("Row semantics").
 */
#ifndef HEGMM_B200_H
#define HEGMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    HGM_OK = 0,
    HGM_EDIM = 1,
    HGM_ECAP = 2,
    HGM_EINTERNAL = 3,
    HGM_EOVERFLOW = 4,
    HGM_ECUDA = 5,
    HGM_EARG = 6
};

enum { HGM_PHASE_CLIENT = 0, HGM_PHASE_CLOUD = 1 };

/* Parameter sets: 0 = N 8192 / 3x60-bit Q / 1 special prime / dnum 3 (configs 1-4),
 * 1 = N 32768 / 8x55-bit Q / 4 special primes / dnum 2 (config 5),
 * 2 = N 4096 small test set. */
typedef struct hgm_ctx hgm_ctx;
typedef struct hgm_ct hgm_ct;

/* Sessions are reference counted: every live handle and batch keeps its
 * context alive, so hgm_ctx_destroy with handles outstanding only drops the
 * creator's reference (the device memory goes with the last handle).  Every
 * entry point makes the context's device current for its duration and
 * restores the caller's current device.
 *
 * Randomness.  Keys and encryption noise come from a counter-based generator
 * keyed by `seed` (splitmix64 finalisers, shared bit for bit with the CPU
 * oracle).  A caller-chosen seed is a TEST / PARITY mode: anyone who knows
 * the seed can regenerate the secret key (and since that generator is a public
 * bijection chain, one sample such as a public key's uniform `a` gives the seed
 * back).  HGM_CTX_OS_SEED sessions draw every key and noise sample from ChaCha12
 * keyed with 256 bits from the OS CSPRNG instead, never exported (hgm_ctx_info
 * reports seed 0);
 * for keys held outside the library, create the cloud context with
 * HGM_CTX_KEYLESS and upload them (hgm_key_upload), and encrypt with
 * host-sampled noise (hgm_encrypt_noise). */
#define HGM_CTX_KEYLESS 1 /* no keys are generated: upload sk / pk / switching keys */
#define HGM_CTX_OS_SEED 2 /* seed from /dev/urandom, not exported */
hgm_ctx* hgm_ctx_create(int param_id, uint64_t seed, int device);
hgm_ctx* hgm_ctx_create_ex(int param_id, uint64_t seed, int device, int flags);
void hgm_ctx_destroy(hgm_ctx* ctx);
const char* hgm_last_error(void);

/* info[0]=N [1]=L [2]=K [3]=nB [4]=dnum [5]=t [6]=alpha [7]=seed (0 if OS seeded), then primes */
int hgm_ctx_info(const hgm_ctx* ctx, uint64_t* info, size_t cap);
size_t hgm_slot_count(const hgm_ctx* ctx);
size_t hgm_ct_words(const hgm_ctx* ctx);

/* Key material (SURVEY.md 8b hgm_keys_upload), canonical residues in the NTT
 * domain, words = hgm_key_words(kind):
 *   kind 0 secret key [R][N] (s over Q ++ P, R = L + K primes)
 *   kind 1 public key [2][L][N] (pk0 = -a s + e, pk1 = a)
 *   kind 2 switching key of Galois element `elt` (0 = relinearisation, s^2)
 *          [dnum][2][R][N] (row dg: -a s + e + [r in digit dg] P s', a)
 * Upload replaces the context's copy; export of a switching key the context
 * lacks generates it (needs the secret key).  A context without the secret
 * key cannot decrypt (HGM_EARG) and fails on a rotation / product whose key was
 * not uploaded (HGM_EARG, naming the Galois element). */
size_t hgm_key_words(const hgm_ctx* ctx, int kind);
int hgm_key_export(hgm_ctx* ctx, int kind, uint32_t elt, uint64_t* words, size_t n);
int hgm_key_upload(hgm_ctx* ctx, int kind, uint32_t elt, const uint64_t* words, size_t n);
int hgm_key_drop_secret(hgm_ctx* ctx);
int hgm_key_has(const hgm_ctx* ctx, int kind); /* kind 0 / 1 */
/* Galois element of a left rotation by `offset` slots: 3^(offset mod N/2) mod 2N */
uint32_t hgm_galois_element(const hgm_ctx* ctx, int64_t offset);

/* encrypt reserves (atomically) and uses the next session encryption counter;
 * the _at variant takes it explicitly (the counter selects u, e0, e1). */
int hgm_encrypt(hgm_ctx* ctx, const int64_t* values, size_t S, hgm_ct** out);
int hgm_encrypt_at(hgm_ctx* ctx, const int64_t* values, size_t S, uint64_t counter, hgm_ct** out);
/* Encryption with host-sampled randomness: u (ternary), e0, e1 are N signed
 * coefficients each (SURVEY.md 8b hgm_rand).  Counts as one encrypt. */
int hgm_encrypt_noise(hgm_ctx* ctx, const int64_t* values, size_t S, const int64_t* u, const int64_t* e0,
                      const int64_t* e1, hgm_ct** out);
/* Reserves n consecutive session counters; returns the first. */
uint64_t hgm_reserve_counters(hgm_ctx* ctx, uint64_t n);
/* counter0 value for the batch entry points: take count * E counters from the
 * session (hgm_reserve_counters) instead of an explicit range */
#define HGM_COUNTER_AUTO UINT64_MAX
int hgm_decrypt(hgm_ctx* ctx, const hgm_ct* ct, int64_t* out, size_t cap);
int hgm_add(hgm_ctx* ctx, const hgm_ct* x, const hgm_ct* y, hgm_ct** out);
/* he_mult's result is a pending product: hgm_add over products sums their
 * unscaled tensors; scale-and-round and relinearisation run once, when any
 * other op, decrypt or export reads the value (same slots, counters, depth). */
int hgm_mul(hgm_ctx* ctx, const hgm_ct* x, const hgm_ct* y, hgm_ct** out);
int hgm_cmul(hgm_ctx* ctx, const hgm_ct* x, const int64_t* mask, size_t S, hgm_ct** out);
/* he_rot's result is a pending key switch (the accumulator over Q and the
 * special primes): hgm_cmul / hgm_add of rotations work on it and ModDown runs
 * once, when any other op, decrypt or export reads the value. */
int hgm_rot(hgm_ctx* ctx, const hgm_ct* x, int64_t offset, hgm_ct** out);
/* offsets[n], masks[n][S] (row-major); counts n cmult, n-1 add and one rot
 * per non-zero offset, as apply_plan does. */
int hgm_apply_plan(hgm_ctx* ctx, const hgm_ct* x, size_t n, const int64_t* offsets,
                   const int64_t* masks, size_t S, hgm_ct** out);

/* Executes every pending operation whose result a pinned handle still
 * refers to (unpinned handles stay lazy); synchronous. */
int hgm_flush(hgm_ctx* ctx);
int hgm_ct_export(hgm_ctx* ctx, const hgm_ct* ct, uint64_t* words);
int hgm_ct_import(hgm_ctx* ctx, const uint64_t* words, size_t S, size_t depth, hgm_ct** out);

/* Ciphertext wire format (client <-> cloud transport; new): a 48-byte header
 * { "HGMC", u32 version = 1, u64 key-set fingerprint (primes + key seed),
 *   u32 N, u32 L, u32 segment, u32 depth, u32 phase, u32 reserved,
 *   u64 FNV-1a checksum of the payload } followed by the 2*L*N residues
 * (c0 limbs then c1 limbs, NTT domain, canonical), little endian.
 * hgm_ct_serialize writes hgm_ct_wire_size() bytes; hgm_ct_deserialize
 * rejects (HGM_EARG) a wrong magic/version/size, another parameter or key set,
 * a checksum mismatch or a non-canonical residue, and S > slot_count
 * (HGM_ECAP) as hgm_encrypt does. */
size_t hgm_ct_wire_size(const hgm_ctx* ctx);
int hgm_ct_serialize(hgm_ctx* ctx, const hgm_ct* ct, void* buf, size_t cap);
int hgm_ct_deserialize(hgm_ctx* ctx, const void* buf, size_t len, hgm_ct** out);
size_t hgm_ct_segment(const hgm_ct* ct);
size_t hgm_ct_depth(const hgm_ct* ct);
int hgm_ct_phase(const hgm_ct* ct);
hgm_ct* hgm_ct_retain(hgm_ct* ct);
void hgm_ct_release(hgm_ct* ct);
/* A pinned handle (the default) keeps its ciphertext materialised after a
 * flush.  An unpinned handle only keeps the recipe: the value is recomputed
 * (bit-identically) if it is needed again, and it never blocks the fusion of
 * its node into a consumer.  Adapters that cannot observe when the caller
 * drops a handle (integration/bfv_gpu_backend.cpp) unpin everything. */
int hgm_ct_set_pinned(hgm_ct* ct, int pinned);

/* stats[2*k + {0: client, 1: cloud}] for k = add, mult_cc, mult_cp, rot,
 * encrypt, decrypt (OpStats field order, backend.hpp:50-57). */
int hgm_stats(const hgm_ctx* ctx, uint64_t stats[12]);
int hgm_reset_stats(hgm_ctx* ctx);
size_t hgm_peak_live(const hgm_ctx* ctx);
int hgm_set_phase(hgm_ctx* ctx, int phase);
int hgm_phase(const hgm_ctx* ctx);

/* Batched HEGMM: `count` independent products C_i = A_i B_i (A_i m x l, B_i
 * l x n, row-major int64) through basic_mm (algo 0), enhanced_mm (algo 1) or
 * square_pad_mm (algo 2) (algorithms.hpp:59-71); order -1 auto / 0 column-major /
 * 1 row-major; flags bit 0 = MultiplyOptions::encrypted_client_transforms
 * (algorithms.hpp:21).  Inputs and outputs are host buffers; outputs canonical
 * mod t.  Instance i encrypts with counters counter0 + i * E, E = encryptions
 * per instance (3 basic, 2 enhanced).  stats (optional) receives one
 * instance's counts (identical for all). */
#define HGM_FLAG_ENCRYPTED_CLIENT_TRANSFORMS 1
int hgm_matmul_batch(hgm_ctx* ctx, int algo, int order, int flags, size_t m, size_t l, size_t n,
                     size_t count, const int64_t* A, const int64_t* B, int64_t* C,
                     uint64_t counter0, uint64_t* stats);
/* same, also exporting every instance's final (pre-decrypt) ciphertext */
int hgm_matmul_batch_export(hgm_ctx* ctx, int algo, int order, int flags, size_t m, size_t l, size_t n,
                            size_t count, const int64_t* A, const int64_t* B, int64_t* C,
                            uint64_t counter0, uint64_t* final_words);
/* blocked_mm (algorithms.hpp:97-98, algorithms.cpp:434-498): the product tiled by
 * the row / mid / col partitions; every block product runs (the independent
 * ones in lockstep batches) with `algo`, falling back from enhanced (1) to
 * basic (0) when a block's working set exceeds the slots, and the decrypted
 * blocks are accumulated mod t.  log (optional, 4 int32 per block in the
 * reference loop order bi, bj, bk): algo used, fell_back, block m, l.
 * Block b encrypts with counters counter0 + (encryptions of blocks before b). */
int hgm_blocked_mm(hgm_ctx* ctx, int algo, size_t m, size_t l, size_t n, const size_t* row_blocks,
                   size_t n_row, const size_t* mid_blocks, size_t n_mid, const size_t* col_blocks,
                   size_t n_col, const int64_t* A, const int64_t* B, int64_t* C, uint64_t counter0,
                   int32_t* log);

/* blocked_mm with ENCRYPTED accumulation (new): every block
 * product of an output block stays a ciphertext on the GPU; the products of
 * one output block that share a slot layout (working rows / cols and flatten
 * order -- all of them unless the enhanced -> basic fallback mixes layouts)
 * are summed over the mid dimension (mod q, one add launch per depth level),
 * and each sum is decrypted ONCE -- where the reference decrypts every block
 * product and adds in cleartext (algorithms.cpp:485-490), so the decrypt
 * count differs (n_decrypts).  Products, log and encryption counters are those
 * of hgm_blocked_mm; a sum decrypts to the sum of its products mod t.
 *   out_first / out_count  output blocks (row-major bi * n_col + bj) this call
 *                          computes -- a shard for multi-GPU; C entries of other
 *                          blocks are left untouched; counters stay those of the
 *                          whole product, so shards are bit-identical to one run
 *   acc_words / acc_meta   optional host outputs, acc_cap entries: each summed
 *                          ciphertext ([ct_words]) and its meta (8 int64: output
 *                          block, algo used, block m, l, n, flatten order, terms,
 *                          segment); *n_acc = number of sums
 * flags 0 gives hgm_blocked_mm exactly (out range must then cover all blocks). */
#define HGM_BLOCKED_ENCRYPTED_ACCUMULATION 1
/* with it: export the sums only, decrypt nothing (the decrypting rank gathers them) */
#define HGM_BLOCKED_NO_DECRYPT 2
int hgm_blocked_mm_ex(hgm_ctx* ctx, int algo, size_t m, size_t l, size_t n, const size_t* row_blocks,
                      size_t n_row, const size_t* mid_blocks, size_t n_mid, const size_t* col_blocks,
                      size_t n_col, const int64_t* A, const int64_t* B, int64_t* C, uint64_t counter0, int flags,
                      size_t out_first, size_t out_count, int32_t* log, uint64_t* acc_words, int64_t* acc_meta,
                      size_t acc_cap, size_t* n_acc, size_t* n_decrypts);

/* The same pipeline split at the reference's phase boundaries
 * (algorithms.cpp:216-247: Client encrypt / Cloud loop / Client decrypt):
 *   hgm_batch_encrypt  packs and encrypts `count` instances (ciphertexts stay in HBM)
 *   hgm_batch_cloud    runs the cloud program on them; *device_ms = CUDA-event time
 *   hgm_batch_output   device pointer of instance i's result ciphertext (for gathers)
 *   hgm_batch_decrypt  decrypts and unpacks every result into host C */
typedef struct hgm_batch hgm_batch;
int hgm_batch_encrypt(hgm_ctx* ctx, int algo, int order, int flags, size_t m, size_t l, size_t n,
                      size_t count, const int64_t* A, const int64_t* B, uint64_t counter0,
                      hgm_batch** out);
int hgm_batch_cloud(hgm_ctx* ctx, hgm_batch* b, float* device_ms);
uint64_t* hgm_batch_output(hgm_batch* b, size_t i);
int hgm_batch_decrypt(hgm_ctx* ctx, hgm_batch* b, int64_t* C);
int hgm_batch_decrypt_words(hgm_ctx* ctx, const uint64_t* dev_words, size_t count, size_t S,
                            int64_t* out);
void hgm_batch_free(hgm_batch* b);
/* Decrypts and unpacks `count` result ciphertexts of a product shape held in
 * device (or host) memory (e.g. gathered from other ranks by hgm_comm_gather_batch) into
 * host C[count][m][n]: the client-side decrypt of algorithms.cpp:244-247. */
int hgm_decrypt_products(hgm_ctx* ctx, int algo, int order, int flags, size_t m, size_t l, size_t n,
                         const uint64_t* dev_words, size_t count, int64_t* C);

/* Multi-GPU (reference analogue: the std::async pool over
 * independent cases, costmodel.cpp:273-296).  One process per GPU, one NCCL
 * communicator per session over NVLink / NVSwitch.  Work shards by independent
 * products or output blocks with keys replicated per GPU; the communicator
 * only MOVES result ciphertexts (never reduces them: NCCL sums wrap mod 2^64,
 * not mod q) and carries control values.  Every call is collective over the
 * communicator and stream-ordered after the session's queued work.
 *   hgm_comm_unique_id / hgm_comm_init   NCCL bootstrap with a caller-distributed id
 *   hgm_comm_init_file                   the same, rank 0 publishing the id at `path`
 *                                        (atomic rename; other ranks poll, timeout_s)
 *   hgm_comm_barrier                     after every rank's queued work
 *   hgm_comm_max                         host double, max over ranks (timings)
 *   hgm_comm_gather                      variable-size gather of words to `root` (rank
 *                                        order); recv / recv_cap_words used on root; host
 *                                        buffers are staged through device memory
 *   hgm_comm_gather_batch                every rank's batch results to `root`, in rank
 *                                        order, into a device buffer the library allocates
 *                                        (free with hgm_comm_buffer_free); b may be NULL
 *                                        on a rank without instances */
typedef struct hgm_comm hgm_comm;
#define HGM_COMM_ID_BYTES 128
int hgm_comm_unique_id(uint8_t* id);
int hgm_comm_init(hgm_ctx* ctx, int rank, int world, const uint8_t* id, hgm_comm** out);
int hgm_comm_init_file(hgm_ctx* ctx, int rank, int world, const char* path, double timeout_s, hgm_comm** out);
void hgm_comm_destroy(hgm_comm* comm);
int hgm_comm_rank(const hgm_comm* comm);
int hgm_comm_size(const hgm_comm* comm);
int hgm_comm_barrier(hgm_comm* comm);
int hgm_comm_max(hgm_comm* comm, double* value);
int hgm_comm_gather(hgm_comm* comm, const uint64_t* send, size_t send_words, uint64_t* recv,
                    size_t recv_cap_words, int root, size_t* recv_words);
int hgm_comm_gather_batch(hgm_comm* comm, hgm_batch* b, int root, uint64_t** dev_out, size_t* total_count);
int hgm_comm_buffer_free(hgm_comm* comm, uint64_t* p);

/* Program facts of a product shape (no GPU needed): stats[12] as hgm_stats,
 * facts[0]=segment [1]=encryptions [2]=rotations after CSE [3]=masked sums
 * [4]=CC-mults [5]=levels [6]=flatten order used [7]=ModDowns (values with a
 * pending key switch read) [8]=scale-and-round + relinearisations (values with
 * a pending product read) [9]=rows [10]=cols of the product's slot layout
 * (entry (r, c) at r + c rows column-major / r cols + c row-major, by [6]);
 * facts holds 11 entries. */
int hgm_program_info(int algo, int order, int flags, size_t m, size_t l, size_t n, size_t slots,
                     uint32_t N, uint64_t* stats, uint64_t* facts);
/* Switching keys a product shape needs (no GPU): sorted Galois elements, 0
 * (relinearisation) first when it multiplies; returns the count (or -error). */
long hgm_program_keys(int algo, int order, int flags, size_t m, size_t l, size_t n, size_t slots, uint32_t N,
                      uint32_t* elements, size_t cap);
/* Op stream of a product shape in call order (no GPU needed), same layout as
 * the reference trace: hdr[3*i] = kind (0 enc 1 dec 2 add 3 mult 4 cmult 5 rot),
 * hdr[3*i+1] = rotation offset / segment, hdr[3*i+2] = data length; data = the
 * cmult masks concatenated.  Returns the op count (or -error). */
long hgm_program_stream(int algo, int order, int flags, size_t m, size_t l, size_t n, size_t slots,
                        uint32_t N, int64_t* hdr, size_t hdr_cap, int64_t* data, size_t data_cap,
                        size_t* data_len);

/* Diagonal plan introspection (no GPU): kind 0 = eps_k (a=m, b=l, c=n),
 * 1 = omega_k (a=l, b=m, c=n) embedded in `segment`; 4 / 5 = the shaped
 * eps / omega plans of enhanced_mm (a=rows, b=cols, c=period).  Writes up to
 * cap (offset, weight) pairs; returns the entry count or -error. */
long hgm_plan_info(int kind, size_t k, size_t a, size_t b, size_t c, int order, size_t segment,
                   int64_t* offsets, uint64_t* weights, size_t cap);

/* Kernel-level timing hooks for bench.py (CUDA events on the library stream). */
int hgm_bench_ntt(hgm_ctx* ctx, int forward, size_t limbs, int iters, float* ms_per_iter);
/* Test hook (no GPU): the ChaCha block function of OS-seeded sessions (key 8
 * words, 64-bit nonce and block counter, `rounds` rounds) into out[16]. */
int hgm_test_chacha(const uint32_t* key, uint64_t nonce, uint64_t counter, int rounds, uint32_t* out);
/* key-switch inner product (k_ks_inner) over `items` rotations, 8 per Galois key */
int hgm_bench_keyswitch(hgm_ctx* ctx, size_t items, int iters, float* ms_per_iter);
/* masked sums of rotations straight from the ModUp digits (k_ks_plan), laid out as
 * the cloud step launches them: tiles of `tile` instances, `sums` sums of `terms`
 * rotations per instance, all reading that instance's digits */
int hgm_bench_keyswitch_plan(hgm_ctx* ctx, size_t instances, size_t sums, size_t terms, size_t tile, int iters,
                             float* ms_per_iter);
int hgm_device_sync(hgm_ctx* ctx);
/* Test hook: in-place NTT of `count` host limbs (count*N words) under one
 * prime (index into Q ++ P ++ B, or -1 for t). */
int hgm_test_ntt(hgm_ctx* ctx, int forward, int prime, uint64_t* data, size_t count);
/* Number of this library's kernels launched on the context so far. */
uint64_t hgm_launch_count(const hgm_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
