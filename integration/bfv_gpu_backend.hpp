// bfv_gpu_backend.hpp -- the reference-side binding: a `hegmm::Backend`
// (/root/reference/proj/include/hegmm/backend.hpp:107-127) implemented on the
// C ABI of libhegmm_b200.so (include/hegmm_b200.h).  It compiles against the
// reference's header UNMODIFIED, so the reference's own basic_mm / enhanced_mm /
// square_pad_mm / blocked_mm / apply_plan run on the B200 with no source change:
//
//     hegmm::BfvGpuBackend gpu(/*param_id=*/0, /*seed=*/1, /*device=*/0);
//     hegmm::Matrix c = hegmm::basic_mm(a, b, gpu);       // encrypted on the GPU
//
// config().slot_count is N/2 (4096 at N = 8192) and config().plaintext_modulus
// is 65537, so decrypted products equal naive_matmul_mod(a, b, 65537).
//
// Minting.  `Ciphertext` can only be constructed by SlotBackend
// (backend.hpp:97-102).  This adapter mints its handles through an inner,
// modulus-free SlotBackend: slot 0 of the minted value carries the GPU handle
// id, depth is raised by he_mult with an all-ones vector, and the phase tag is
// the adapter's phase.  The GPU ciphertext itself never leaves HBM.  A
// maintainer who can touch backend.hpp would instead add one protected factory
// (see INTEGRATION.md); the arithmetic is unaffected either way.
#pragma once

#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "hegmm/backend.hpp"
#include "hegmm_b200.h"

namespace hegmm {

class BfvGpuBackend final : public Backend {
  public:
    BfvGpuBackend(int param_id = 0, std::uint64_t seed = 1, int device = 0);
    ~BfvGpuBackend() override;
    BfvGpuBackend(const BfvGpuBackend&) = delete;
    BfvGpuBackend& operator=(const BfvGpuBackend&) = delete;

    const BackendConfig& config() const override { return cfg_; }

    Ciphertext encrypt(std::span<const value_t> values) override;
    std::vector<value_t> decrypt(const Ciphertext& ct) override;
    Ciphertext he_add(const Ciphertext& x, const Ciphertext& y) override;
    Ciphertext he_mult(const Ciphertext& x, const Ciphertext& y) override;
    Ciphertext he_cmult(const Ciphertext& x, std::span<const value_t> mask) override;
    Ciphertext he_rot(const Ciphertext& x, std::ptrdiff_t offset) override;

    OpStats stats() const override;
    void reset_stats() override;
    std::size_t peak_live_ciphertexts() const override;
    void set_phase(Phase p) override;
    Phase phase() const override;

    // GPU words (2*L*N, NTT domain) of a ciphertext produced by this backend
    std::vector<std::uint64_t> export_words(const Ciphertext& ct);
    hgm_ctx* raw() const { return ctx_; }
    // GPU handles currently held / handle sets released (no minted ciphertext alive)
    std::size_t held_handles() const {
        std::lock_guard<std::mutex> lk(mu_);
        return handles_.size();
    }
    std::size_t epochs() const {
        std::lock_guard<std::mutex> lk(mu_);
        return epoch_;
    }

  private:
    Ciphertext wrap(hgm_ct* h, std::size_t segment, std::size_t depth);
    hgm_ct* handle(const Ciphertext& ct) const;
    static void check(int rc);

    hgm_ctx* ctx_ = nullptr;
    BackendConfig cfg_;
    SlotBackend minter_;
    mutable std::mutex mu_;
    std::vector<hgm_ct*> handles_;                 // id -> GPU handle (this epoch)
    std::size_t epoch_ = 0;                        // handle sets released so far
    std::map<std::size_t, Ciphertext> ones_;       // per segment, for depth minting
};

}  // namespace hegmm
