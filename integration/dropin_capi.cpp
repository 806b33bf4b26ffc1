// dropin_capi.cpp -- test entry: the REFERENCE's own algorithms (compiled from
// /root/reference sources into oracle/_ref/libhegmm_ref.so) driving the B200
// through hegmm::BfvGpuBackend.  Used by tests/test_gpu_dropin.py.
#include <algorithm>
#include <cstring>
#include <optional>

#include "bfv_gpu_backend.hpp"
#include "hegmm/algorithms.hpp"

using namespace hegmm;

namespace {

thread_local std::string g_err;

// Forwards to the GPU backend and remembers the last decrypted ciphertext.
class Recording final : public Backend {
  public:
    explicit Recording(BfvGpuBackend& be) : be_(be) {}
    const BackendConfig& config() const override { return be_.config(); }
    Ciphertext encrypt(std::span<const value_t> v) override { return be_.encrypt(v); }
    std::vector<value_t> decrypt(const Ciphertext& ct) override {
        last_ = ct;
        return be_.decrypt(ct);
    }
    Ciphertext he_add(const Ciphertext& x, const Ciphertext& y) override { return be_.he_add(x, y); }
    Ciphertext he_mult(const Ciphertext& x, const Ciphertext& y) override { return be_.he_mult(x, y); }
    Ciphertext he_cmult(const Ciphertext& x, std::span<const value_t> m) override { return be_.he_cmult(x, m); }
    Ciphertext he_rot(const Ciphertext& x, std::ptrdiff_t z) override { return be_.he_rot(x, z); }
    OpStats stats() const override { return be_.stats(); }
    void reset_stats() override { be_.reset_stats(); }
    std::size_t peak_live_ciphertexts() const override { return be_.peak_live_ciphertexts(); }
    void set_phase(Phase p) override { be_.set_phase(p); }
    Phase phase() const override { return be_.phase(); }
    std::optional<Ciphertext> last_;

  private:
    BfvGpuBackend& be_;
};

}  // namespace

extern "C" {

const char* dropin_last_error(void) { return g_err.c_str(); }

int dropin_mm(int param_id, std::uint64_t seed, int algo, int order, const std::int64_t* A, std::size_t m,
              std::size_t l, const std::int64_t* B, std::size_t n, std::int64_t* C, std::uint64_t* stats,
              std::uint64_t* final_words) {
    try {
        BfvGpuBackend gpu(param_id, seed, 0);
        Recording be(gpu);
        Matrix a(m, l, std::vector<value_t>(A, A + m * l));
        Matrix b(l, n, std::vector<value_t>(B, B + l * n));
        MultiplyOptions opts;
        if (order == 0) opts.order = FlattenOrder::ColumnMajor;
        if (order == 1) opts.order = FlattenOrder::RowMajor;
        Matrix c = algo == 0 ? basic_mm(a, b, be, opts) : algo == 1 ? enhanced_mm(a, b, be, opts)
                                                                    : square_pad_mm(a, b, be, opts);
        std::memcpy(C, c.data().data(), m * n * 8);
        if (stats) {
            const OpStats s = be.stats();
            const PhaseCounts* f[6] = {&s.n_add, &s.n_mult_cc, &s.n_mult_cp, &s.n_rot, &s.n_encrypt, &s.n_decrypt};
            for (int k = 0; k < 6; ++k) { stats[2 * k] = f[k]->client; stats[2 * k + 1] = f[k]->cloud; }
            stats[12] = be.peak_live_ciphertexts();
        }
        if (final_words && be.last_) {
            const auto w = gpu.export_words(*be.last_);
            std::memcpy(final_words, w.data(), w.size() * 8);
        }
        return 0;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return 1;
    } catch (const CapacityError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// `reps` products on ONE long-lived backend session (the handle table must
// not grow across products): info[0] = handle sets released, info[1] = handles
// held at the end, info[2] = most handles held at once.
int dropin_repeat(int param_id, int algo, const std::int64_t* A, std::size_t m, std::size_t l,
                  const std::int64_t* B, std::size_t n, int reps, std::int64_t* C, std::uint64_t* info) {
    try {
        BfvGpuBackend gpu(param_id, 1, 0);
        Matrix a(m, l, std::vector<value_t>(A, A + m * l));
        Matrix b(l, n, std::vector<value_t>(B, B + l * n));
        std::size_t most = 0;
        for (int r = 0; r < reps; ++r) {
            Matrix c = algo == 0 ? basic_mm(a, b, gpu) : enhanced_mm(a, b, gpu);
            std::memcpy(C + (std::size_t)r * m * n, c.data().data(), m * n * 8);
            most = std::max(most, gpu.held_handles());
        }
        info[0] = gpu.epochs();
        info[1] = gpu.held_handles();
        info[2] = most;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

}  // extern "C"
