// context.hpp -- per-device BFV context: tables and keys resident in HBM, the
// content-addressed plaintext-mask cache, pinned staging, and the batched
// primitive launchers that every higher layer (C ABI, lazy engine) calls.
//
// Every primitive works on a batch of independent items given as arrays of
// device pointers, so one launch sequence serves many ciphertexts (many
// rotations of one HEGMM call, or the same op of many lockstep instances).
// Ciphertexts are 2*L*N words, c0 limbs then c1 limbs, NTT domain, canonical.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "ntt.cuh"
#include "params.hpp"

namespace hgm {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
void cuda_check(cudaError_t e, const char* what);
#define HGM_CUDA(x) ::hgm::cuda_check((x), #x)

// Host-pinned ring for uploads of small argument tables and input values.
class PinnedRing {
  public:
    explicit PinnedRing(size_t bytes);
    ~PinnedRing();
    // Copies `bytes` from host `src` to the returned device pointer,
    // asynchronously on `s` (the device copy lives in `dev_` ring).
    void* upload(const void* src, size_t bytes, cudaStream_t s);
    // Two-step form: reserve() returns the pinned host range to fill, commit()
    // issues its copy and returns the device pointer.
    char* reserve(size_t bytes);
    void* commit(char* host, size_t bytes, cudaStream_t s);

  private:
    size_t cap_;
    char* host_ = nullptr;
    char* dev_ = nullptr;
    size_t head_ = 0;
    struct Mark {
        size_t end;
        cudaEvent_t ev;
    };
    std::vector<Mark> marks_;
    std::vector<cudaEvent_t> free_events_;
};

// One group of k_ks_plan (a masked sum of rotations computed straight from the
// ModUp digits): a tile of lockstep instances of one sum, sharing its masked keys.
struct PlanGroup {
    u32 item0, cnt;     // outputs item0 .. item0 + cnt - 1
    u32 term0, nterms;  // masked keys / Galois elements term0 .. term0 + nterms - 1
    u32 dbase, pad;     // digits / c0 of instance u, term t at dbase + u * nterms + t
};

class Context {
  public:
    // keyless: no secret, public or switching keys are generated; they must be
    // uploaded (upload_key) before the operations that need them
    // csprng_key (optional, 8 words from the OS CSPRNG): keys and noise from ChaCha12
    // instead of the seeded parity PRF (HGM_CTX_OS_SEED sessions)
    Context(int param_id, u64 seed, int device, bool keyless = false, const u32* csprng_key = nullptr);
    ~Context();
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    const HostParams& host() const { return hp_; }
    const DevParams& hdev() const { return hp_.dev; }
    const DevParams* dparams() const { return dp_; }
    cudaStream_t stream() const { return stream_; }
    int device() const { return device_; }
    size_t ct_words() const { return (size_t)2 * hp_.L * hp_.N; }
    size_t slots() const { return hp_.N / 2; }

    u64* alloc(size_t words);
    void release(void* p);
    void sync();
    template <typename T>
    T* upload(const std::vector<T>& v) {
        return static_cast<T*>(ring_->upload(v.data(), v.size() * sizeof(T), stream_));
    }
    // pinned host buffer for result downloads (grown on demand, reused)
    void* download_buffer(size_t bytes);
    // pinned double buffers of the pipelined batch decrypt (grown on demand, reused:
    // cudaMallocHost / cudaFreeHost per call cost milliseconds)
    u32* pinned_slot(int i, size_t bytes);

    // ---------------------------------------------------------------- keys
    const u64* ks_key(u32 kid);  // [dnum][2][R][N]; kid = Galois element, 0 = relin
    void ensure_galois_keys(const std::vector<u32>& elements);
    size_t key_count() const;
    // Key material at the boundary (canonical residues, NTT domain):
    //   kind 0 secret key   [R][N]  (s over Q ++ P)
    //   kind 1 public key   [2][L][N]
    //   kind 2 switching key for Galois element `elt` (0 = relinearisation)
    //                       [dnum][2][R][N]
    size_t key_words(int kind) const;
    void upload_key(int kind, u32 elt, const u64* host, size_t words);
    void export_key(int kind, u32 elt, u64* host);
    // Forget the secret key (a cloud context keeps only evaluation keys):
    // decryption and generation of new switching keys then fail.
    void drop_secret();
    bool has_secret() const { return d_sk_ != nullptr; }
    bool has_public() const { return d_pk_ != nullptr; }
    static u32 galois_of(i64 z, u32 N);  // 3^(z mod N/2) mod 2N; 1 for z = 0

    // ---------------------------------------------------------------- masks
    // NTT-domain centred lift of the batch-encoded mask over Q: [L][N].
    const u64* mask_plain(const i64* mask, size_t S, u64 stable_id = 0);
    // Bounds the device mask cache (least recently used first) to mask_budget()
    // bytes; called between programs (execute()), never while one holds mask
    // pointers -- frees are stream-ordered behind the launches that used them.
    void trim_mask_cache();
    size_t mask_budget() const;

    // ---------------------------------------------------------------- primitives
    // host_vals[i] holds S[i] values; counters[i] is the encryption counter.
    void encrypt(int n, const i64* const* host_vals, const size_t* S, const u64* counters,
                 u64* const* out);
    // Same with host-sampled randomness: noise = n x [u | e0 | e1] x N signed
    // coefficients (u ternary, e0 / e1 small), instead of the counter PRNG.
    void encrypt_noise(int n, const i64* const* host_vals, const size_t* S, const i64* noise,
                       u64* const* out);
    // Decrypts n ciphertexts into host buffers (synchronises the stream).
    void decrypt(int n, const u64* const* in, const size_t* S, i64* const* host_out);
    // Enqueues the decryption of n ciphertexts into pinned host memory (N/2 u32
    // slots per ciphertext, values in [0, t)); valid once the stream reaches it.
    void decrypt_to(int n, const u64* const* in, const size_t* S, u32* pinned_host);
    void add(int n, const u64* const* a, const u64* const* b, u64* const* out);
    // out[o] = sum over terms t in [off[o], off[o+1]) of in[t] (.* mask[t] if set)
    void lincomb(int n_out, const u32* off, const u64* const* in, const u64* const* mask,
                 u64* const* out);
    // Hoisted half of key switching: digits of c1, lifted to Q++P, NTT domain.
    size_t modup_words() const { return (size_t)hp_.dnum * hp_.R * hp_.N; }
    void modup(int n, const u64* const* ct, u64* const* out);
    // out = Rot(ct, g) from ct's ModUp image.
    void rotate(int n, const u64* const* modup, const u64* const* ct, const u32* g,
                u64* const* out);
    void mult(int n, const u64* const* a, const u64* const* b, u64* const* out);
    // Pending key switches (oracle rot_x): acc [2][R][N] over Q ++ P, NTT domain,
    // P phi_g(c0) folded in; their plain value is ModDown(acc).
    size_t ks_words() const { return (size_t)2 * hp_.R * hp_.N; }
    void rotate_acc(int n, const u64* const* modup, const u64* const* ct, const u32* g, u64* const* acc);
    // out = ModDown(acc) (acc is left intact)
    void moddown(int n, const u64* const* acc, u64* const* out, bool prescaled = false);
    // Masked sums of rotations straight from the ModUp digits (k_ks_plan).
    // masked_key: key_g (.) (sum of the masks) over Q ++ P followed by (P mod q) (.)
    // (that sum) over Q, packed digits, cached per (g, mask ids) -- the ids are the
    // stable ids of cached programs' masks, mask_dev their device lifts
    // (mask_plain; null = look up only); nullptr when absent / the cache budget
    // cannot take another entry.
    size_t masked_key_words() const { return ((size_t)hp_.dnum * 2 * hp_.R + hp_.L) * hp_.N; }
    // prescaled: the Q limbs' masks carry P^-1, so the sum over Q is P^-1 (acc + P phi(c0))
    // and moddown(..., prescaled) adds it without the Shoup product (can_prescale())
    const u64* masked_key(u32 g, const std::vector<u64>& ids, const std::vector<const u64*>* mask_dev,
                          bool prescaled = false);
    bool can_prescale() const;
    size_t masked_key_budget() const;
    bool masked_keys_fit(size_t count) const { return count * masked_key_words() * 8 <= masked_key_budget(); }
    void trim_masked_keys(size_t needed);  // between programs: room for `needed` more entries
    void drop_masked_keys();               // keys changed
    // out[i] = sum over the terms of i's group of mask (.) RotAcc: mkey / g per
    // term, digits / c0 per (instance, term) as PlanGroup lays them out
    void rotate_plan(const std::vector<PlanGroup>& groups, const std::vector<const u64*>& mkey,
                     const std::vector<u32>& g, const std::vector<const u64*>& digits,
                     const std::vector<const u64*>& c0, const std::vector<u64*>& out);
    // lincomb over pending key switches ([2][R][N] inputs, masks over Q ++ P)
    void lincomb_qp(int n_out, const u32* off, const u64* const* in, const u64* const* mask, u64* const* out);
    // Pending products (oracle XCt): a pending value is [T: 3 (L+nB) N][addend: 2 L N],
    // T the unscaled tensor sum over Q ++ B in the NTT domain.
    size_t pending_words() const { return (size_t)3 * (hp_.L + hp_.nB) * hp_.N + ct_words(); }
    size_t tensor_words() const { return (size_t)3 * (hp_.L + hp_.nB) * hp_.N; }
    // T[d] (+= if init[d]) sum of tensor(a[i], b[i]) over i in [off[d], off[d+1])
    void tensor_acc(int n_dest, const u32* off, const u64* const* a, const u64* const* b, u64* const* T,
                    const unsigned char* init);
    // T regions: out[o] (+= if init[o]) sum of in[t], t in [off[o], off[o+1])
    void tsum(int n_out, const u32* off, const u64* const* in, u64* const* out, const unsigned char* init);
    // out[i] = scale-and-round + relinearisation of T[i], + addend[i] (optional)
    void materialize(int n, const u64* const* T, const u64* const* addend, u64* const* out);
    void copy(int n, const u64* const* in, u64* const* out);

    // batched NTT helpers (exposed for tests / micro-benchmarks)
    void ntt(bool forward, const NttJobs& jobs);
    // micro-benchmark inputs: limb l gets pseudo-random residues of prime
    // first_prime + l % period (canonical, so the kernels see real operands)
    void fill_residues(u64* p, u32 limbs, u32 first_prime, u32 period, u64 seed);
    // micro-benchmark of the key-switch inner product (k_ks_inner) over `items`
    // rotations in groups of 8 sharing a Galois key, as the engine orders them;
    // returns ms per launch (CUDA events on the library stream)
    float bench_inner_product(int items, int iters);
    float bench_plan(int instances, int sums, int terms, int tile, int iters);  // k_ks_plan, ms per launch
    u64 launches() const { return launches_.load(); }

  private:
    void build_keys();
    void encrypt_impl(int n, const i64* const* host_vals, const size_t* S, const u64* counters,
                      const i64* noise, u64* const* out);
    u64* b_extend(int n, const u64* const* a, const u64* const* b);
    void scale_relin(int n, u64* T, u64* const* out);
    void key_switch_tail(int n, u64* const* acc, const u64* const* ecoef, const u64* const* addn,
                         const u32* g, u64* const* out, bool prescaled = false);
    bool tail_keeps_acc() const;
    void inner_product(int n, const u64* const* digits, const u64* const* keys, const u32* g,
                       u64* const* acc, const u64* const* c0 = nullptr);

    HostParams hp_;
    std::atomic<u64> launches_{0};
    int device_ = 0;
    bool keyless_ = false;
    cudaStream_t stream_ = nullptr;
    DevParams* dp_ = nullptr;
    DevCtx cx_{};
    u64* d_tw_ = nullptr;
    u32* d_slot_ = nullptr;
    u64* d_cdt_ = nullptr;
    u64* d_sk_ = nullptr;  // [R][N]
    u64* d_pk_ = nullptr;  // [2][L][N]
    std::unique_ptr<PinnedRing> ring_;
    void* dl_host_ = nullptr;
    size_t dl_cap_ = 0;
    u32* slot_host_[2] = {nullptr, nullptr};
    size_t slot_cap_[2] = {0, 0};
    mutable std::mutex key_mu_;
    std::unordered_map<u32, u64*> keys_;
    std::mutex mask_mu_;
    struct MaskEntry {
        std::vector<i64> content;
        u64* dev;
        u64 tick = 0;            // last use (LRU)
        std::vector<u64> ids;    // stable ids aliasing this entry
    };
    std::unordered_map<u64, std::list<MaskEntry>> masks_;
    std::unordered_map<u64, MaskEntry*> masks_by_id_;  // stable MaskData ids
    struct MaskedKey {
        u64* dev;
        u64 tick;
    };
    std::map<std::vector<u64>, MaskedKey> mkeys_;  // {g, sorted mask ids} -> masked key
    u64 mask_tick_ = 0;
    size_t mask_bytes_ = 0;
    mutable size_t mask_budget_ = 0;
};

}  // namespace hgm
