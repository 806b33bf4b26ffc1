// bfv_gpu_backend.cpp -- see bfv_gpu_backend.hpp.  Every override forwards to
// one C-ABI entry point and keeps the reference's contract: argument checks and
// exception types (backend.cpp:118-197), one counter bump per call by phase
// (the library counts), and immutable value semantics for Ciphertext.
#include "bfv_gpu_backend.hpp"

#include <string>

namespace hegmm {

namespace {

BackendConfig config_of(hgm_ctx* ctx) {
    std::uint64_t info[64];
    hgm_ctx_info(ctx, info, 64);
    return BackendConfig{static_cast<std::size_t>(info[0] / 2), static_cast<value_t>(info[5])};
}

}  // namespace

void BfvGpuBackend::check(int rc) {
    switch (rc) {
        case HGM_OK: return;
        case HGM_EDIM: throw DimensionError(hgm_last_error());
        case HGM_ECAP: throw CapacityError(hgm_last_error());
        case HGM_EOVERFLOW: throw OverflowError(hgm_last_error());
        default: throw Error(std::string("libhegmm_b200: ") + hgm_last_error());
    }
}

static hgm_ctx* create_or_throw(int param_id, std::uint64_t seed, int device) {
    hgm_ctx* c = hgm_ctx_create(param_id, seed, device);
    if (!c) throw Error(std::string("libhegmm_b200: ") + hgm_last_error());
    return c;
}

BfvGpuBackend::BfvGpuBackend(int param_id, std::uint64_t seed, int device)
    : ctx_(create_or_throw(param_id, seed, device)),
      cfg_(config_of(ctx_)),
      minter_(BackendConfig{cfg_.slot_count, std::nullopt}) {}

BfvGpuBackend::~BfvGpuBackend() {
    ones_.clear();
    for (hgm_ct* h : handles_) hgm_ct_release(h);
    hgm_ctx_destroy(ctx_);
}

Ciphertext BfvGpuBackend::wrap(hgm_ct* h, std::size_t segment, std::size_t depth) {
    // the caller's Ciphertext lifetime is not observable per handle: keep the recipe only
    hgm_ct_set_pinned(h, 0);
    std::lock_guard<std::mutex> lk(mu_);
    // ... but the minter's live count is (LiveTracker, backend.cpp:50-90; reset_stats
    // sets peak = current): when no ciphertext this backend handed out is alive any
    // more -- e.g. between two basic_mm calls on one session -- every GPU handle is
    // dead and is released, so a long-lived backend does not grow without bound.
    minter_.reset_stats();
    if (minter_.peak_live_ciphertexts() <= ones_.size() && !handles_.empty()) {
        for (hgm_ct* old : handles_) hgm_ct_release(old);
        handles_.clear();
        ++epoch_;
    }
    const std::uint64_t id = handles_.size();
    handles_.push_back(h);
    minter_.set_phase(phase());
    std::vector<value_t> v(segment, 0);
    v[0] = static_cast<value_t>(id);
    Ciphertext ct = minter_.encrypt(v);
    if (depth > 0) {
        auto it = ones_.find(segment);
        if (it == ones_.end())
            it = ones_.emplace(segment, minter_.encrypt(std::vector<value_t>(segment, 1))).first;
        for (std::size_t d = 0; d < depth; ++d) ct = minter_.he_mult(ct, it->second);
    }
    return ct;
}

hgm_ct* BfvGpuBackend::handle(const Ciphertext& ct) const {
    if (ct.segment_length() == 0) throw DimensionError("empty ciphertext handle");
    const auto id = static_cast<std::size_t>(ct.slots()[0]);
    std::lock_guard<std::mutex> lk(mu_);
    if (id >= handles_.size()) throw Error("ciphertext does not belong to this backend");
    return handles_[id];
}

Ciphertext BfvGpuBackend::encrypt(std::span<const value_t> values) {
    hgm_ct* out = nullptr;
    check(hgm_encrypt(ctx_, values.data(), values.size(), &out));
    return wrap(out, values.size(), 0);
}

std::vector<value_t> BfvGpuBackend::decrypt(const Ciphertext& ct) {
    std::vector<value_t> out(ct.segment_length());
    check(hgm_decrypt(ctx_, handle(ct), out.data(), out.size()));
    return out;
}

Ciphertext BfvGpuBackend::he_add(const Ciphertext& x, const Ciphertext& y) {
    hgm_ct* out = nullptr;
    check(hgm_add(ctx_, handle(x), handle(y), &out));
    return wrap(out, x.segment_length(), std::max(x.depth(), y.depth()));
}

Ciphertext BfvGpuBackend::he_mult(const Ciphertext& x, const Ciphertext& y) {
    hgm_ct* out = nullptr;
    check(hgm_mul(ctx_, handle(x), handle(y), &out));
    return wrap(out, x.segment_length(), std::max(x.depth(), y.depth()) + 1);
}

Ciphertext BfvGpuBackend::he_cmult(const Ciphertext& x, std::span<const value_t> mask) {
    hgm_ct* out = nullptr;
    check(hgm_cmul(ctx_, handle(x), mask.data(), mask.size(), &out));
    return wrap(out, x.segment_length(), x.depth());
}

Ciphertext BfvGpuBackend::he_rot(const Ciphertext& x, std::ptrdiff_t offset) {
    hgm_ct* out = nullptr;
    check(hgm_rot(ctx_, handle(x), static_cast<std::int64_t>(offset), &out));
    return wrap(out, x.segment_length(), x.depth());
}

OpStats BfvGpuBackend::stats() const {
    std::uint64_t s[12];
    hgm_stats(ctx_, s);
    OpStats o;
    PhaseCounts* f[6] = {&o.n_add, &o.n_mult_cc, &o.n_mult_cp, &o.n_rot, &o.n_encrypt, &o.n_decrypt};
    for (int k = 0; k < 6; ++k) *f[k] = PhaseCounts{s[2 * k], s[2 * k + 1]};
    return o;
}

void BfvGpuBackend::reset_stats() {
    hgm_reset_stats(ctx_);
    minter_.reset_stats();
}

std::size_t BfvGpuBackend::peak_live_ciphertexts() const {
    // live minted values, minus the cached all-ones helpers
    const std::size_t p = minter_.peak_live_ciphertexts();
    std::lock_guard<std::mutex> lk(mu_);
    return p > ones_.size() ? p - ones_.size() : 0;
}

void BfvGpuBackend::set_phase(Phase p) { hgm_set_phase(ctx_, p == Phase::Client ? HGM_PHASE_CLIENT : HGM_PHASE_CLOUD); }
Phase BfvGpuBackend::phase() const { return hgm_phase(ctx_) == HGM_PHASE_CLIENT ? Phase::Client : Phase::Cloud; }

std::vector<std::uint64_t> BfvGpuBackend::export_words(const Ciphertext& ct) {
    std::vector<std::uint64_t> w(hgm_ct_words(ctx_));
    check(hgm_ct_export(ctx_, handle(ct), w.data()));
    return w;
}

}  // namespace hegmm
