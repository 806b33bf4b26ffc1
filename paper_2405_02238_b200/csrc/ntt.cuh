// ntt.cuh -- batched negacyclic NTT / INTT over 64-bit primes.
//
// One CTA transforms one block of NB = 2^LB residues (one limb for N <= 8192,
// a quarter limb for N = 32768) entirely in shared memory:
//   coalesced 16-byte loads -> smem -> 3 register rounds of up to 5 radix-2
//   stages each (Cooley-Tukey forward / Gentleman-Sande inverse) -> smem ->
//   coalesced stores.
// The smem image is padded one word per 16 (pad()) so that the stride-16 and
// contiguous-16 access patterns of the three rounds are bank-conflict free.
// Twiddles are Shoup pairs read through the read-only path; every twiddle is
// loaded once per group and stage.  For N = 2^15 a limb is held by a cluster of
// four CTAs that exchange the two outermost stages through distributed shared
// memory, one HBM pass per limb (k_ntt_fwd_c4 / k_ntt_inv_c4); HGM_NTT_CLUSTER=0
// runs those two stages as a separate coalesced pass instead.  The forward
// transform's fused last stage canonicalises through a 16-entry k*q table in
// shared memory (Canon, ntt.cu).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace hgm {

// A batch of in-place transforms.  Job j works on ptrs[j] if ptrs is set,
// else on base + j*N; its prime is prime[j % period] (index into DevParams::pr,
// kTIndex for the plaintext modulus).
struct NttJobs {
    u64* base = nullptr;
    u64* const* ptrs = nullptr;
    // optional out-of-place source: job j reads src[j] and writes its ptr/base
    // slot (whole-limb transforms only, N <= 8192)
    const u64* const* src = nullptr;
    u32 count = 0;
    u32 period = 1;
    // inverse only: leave out the N^-1 scaling (the output is N * INTT(x)); for
    // consumers whose first step multiplies by a constant that has N^-1 folded in.
    // 1: canonical residues; 2 (kLazyOut): residues in [0, 4q), not reduced
    // (whole-limb transforms; for consumers whose Shoup product takes any
    // 64-bit input -- others get canonical output)
    u32 unscaled = 0;
    // inverse only: the first Gentleman-Sande stage (t = 1) was applied by the
    // producer (k_tensor); only honoured where ntt_inverse_takes_first_stage()
    u32 first_done = 0;
    // set by the launcher: CTA x also prefetches job x + ahead's block into L2
    // (the CTA that will take its slot one wave later); 0 = off
    u32 ahead = 0;
    unsigned char prime[32] = {0};  // host-side pattern
    u64 packed[4] = {0, 0, 0, 0};   // the same pattern, packed for the kernel
    void pack() {
        for (int w = 0; w < 4; ++w) {
            packed[w] = 0;
            for (int b = 0; b < 8; ++b) packed[w] |= (u64)prime[8 * w + b] << (8 * b);
        }
    }
};

void ntt_forward(const DevCtx& cx, const DevParams& hp, const NttJobs& jobs, cudaStream_t s);
void ntt_inverse(const DevCtx& cx, const DevParams& hp, const NttJobs& jobs, cudaStream_t s);
// Forward NTTs with fused base conversions (whole-limb transforms, N <= 8192):
//  * ModUp: D[item][dg][r] = NTT_r(digit dg of C[item] lifted to prime r), C
//    holding L coefficient-domain limbs per item (stride c_stride words);
//  * ModDown: out[item] = (acc - NTT(conv(P-part))) P^-1 (+ NTT(addc)) (+ addn[galois]),
//    acc's P limbs already inverse-transformed.  Pointer arrays live on the device.
constexpr int kFuseModUp = 1, kFuseModDown = 2;
bool ntt_fusable(const DevParams& hp, int which);
// whole-limb transforms (N <= 8192): out-of-place jobs allowed
// (N = 32768 too while its transforms run as 4-CTA clusters, which read any source)
bool ntt_out_of_place_ok(const DevParams& hp);
inline bool ntt_fusable_size(const DevParams& hp) { return ntt_out_of_place_ok(hp); }
void ntt_modup_fused(const DevCtx& cx, const DevParams& hp, int n, const u64* C, size_t c_stride, u64* D,
                     cudaStream_t s);
void ntt_moddown_fused(const DevCtx& cx, const DevParams& hp, int n, u64* const* acc, const u64* const* addc,
                       const u64* const* addn, const u32* g, u64* const* out, cudaStream_t s);
// ModDown's forward NTT of V (k_moddown_conv's output, [n][2][L][N]) with the
// finishing pass (P^-1 acc + phi_g(addn)) fused into the store; default on
// (HGM_FUSED_FINISH=0 disables) for whole-limb transforms.
bool ntt_finish_fusable(const DevParams& hp);
void ntt_finish_fused(const DevCtx& cx, const DevParams& hp, int n, const u64* V, u64* const* acc,
                      const u64* const* addn, const u32* g, u64* const* out, cudaStream_t s,
                      bool prescaled = false);  // prescaled: acc's Q limbs hold P^-1 acc already
// INTT of acc's P limb with k_moddown_conv fused into its store (K = 1, whole
// limbs; default on, HGM_FUSED_CONV=0 disables): writes V = ecoef - P^-1 conv.
bool ntt_conv_fusable(const DevParams& hp);
void ntt_moddown_conv_fused(const DevCtx& cx, const DevParams& hp, int n, u64* const* acc, const u64* const* ecoef,
                            u64* V, cudaStream_t s);
// The tensor product over Q ++ B fused into its INTT (whole limbs; opt-in,
// HGM_FUSED_TENSOR=1): T[item][p][d] = N * INTT(tensor_p) in [0, 4q),
// A/B per item NTT-domain ciphertexts, XB [n][4][nB][N] their B extension.
bool ntt_tensor_fusable(const DevParams& hp);
void ntt_tensor_fused(const DevCtx& cx, const DevParams& hp, int n, const u64* const* A, const u64* const* B,
                      const u64* XB, u64* T, cudaStream_t s);
// copies a parameter set's constants into this translation unit's __constant__ slot
void ntt_upload_params(int pid, const DevParams& p);

constexpr u32 kLazyOut = 2;
// whether ntt_inverse honours NttJobs::first_done for this parameter set
bool ntt_inverse_takes_first_stage(const DevParams& hp);

inline NttJobs jobs_contig(u64* base, u32 count, u32 first_prime, u32 period) {
    NttJobs j;
    j.base = base;
    j.count = count;
    j.period = period;
    for (u32 i = 0; i < period && i < 32; ++i) j.prime[i] = (unsigned char)(first_prime + i);
    return j;
}

}  // namespace hgm
