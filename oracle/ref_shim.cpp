// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.  Compiled against the UNMODIFIED
// reference headers (/root/reference/proj/include) and linked with the
// reference's own hot-path sources (matrix/backend/lintrans/algorithms.cpp),
// built in place by oracle/ref.mk into oracle/_ref/.  Exposes, to pytest and
// bench.py's reference arm, a C ABI over:
//   * the reference algorithms over the reference SlotBackend (the literal
//     reference CPU path; cleartext slot emulation), and
//   * the reference algorithms over the CPU BFV oracle (bfv_oracle.cpp),
//     plugged in through `hegmm::Backend` (backend.hpp:107-127) exactly the
//     way the GPU backend is (see integration/bfv_gpu_backend.cpp).
//
// Minting: `Ciphertext`'s fields are private and only SlotBackend may build
// one (backend.hpp:97-102).  A third-party backend therefore mints its handles
// through an inner SlotBackend without a modulus: slot 0 carries the handle id,
// depth is raised with he_mult by an all-ones vector, and the phase tag follows
// the minter's phase.  All of this is host bookkeeping, O(segment) per op.
#include <atomic>
#include <map>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "bfv_oracle.h"
#include "hegmm/algorithms.hpp"
#include "hegmm/costmodel.hpp"
#include "hegmm/backend.hpp"
#include "hegmm/lintrans.hpp"
#include "hegmm/matrix.hpp"

using namespace hegmm;

namespace {

thread_local std::string g_err;

class Minter {
  public:
    explicit Minter(std::size_t slots) : be_(BackendConfig{slots, std::nullopt}) {}
    Ciphertext mint(std::size_t segment, std::size_t depth, std::uint64_t id, Phase ph) {
        be_.set_phase(ph);
        std::vector<value_t> v(segment, 0);
        v[0] = static_cast<value_t>(id);
        Ciphertext ct = be_.encrypt(v);
        if (depth > 0) {
            const Ciphertext ones = be_.encrypt(std::vector<value_t>(segment, 1));
            for (std::size_t d = 0; d < depth; ++d) ct = be_.he_mult(ct, ones);
        }
        return ct;
    }
    static std::uint64_t id_of(const Ciphertext& ct) {
        return static_cast<std::uint64_t>(ct.slots()[0]);
    }
    std::size_t peak() const { return be_.peak_live_ciphertexts(); }
    void reset_peak() { be_.reset_stats(); }

  private:
    SlotBackend be_;
};

// hegmm::Backend over the CPU BFV oracle.
class OracleBackend final : public Backend {
  public:
    OracleBackend(orc_ctx* ctx, std::uint64_t enc_counter)
        : ctx_(ctx), cfg_(config_of(ctx)), minter_(cfg_.slot_count), counter_(enc_counter) {
        words_ = orc_ct_words(ctx);
        pwords_ = orc_pending_words(ctx);
    }
    static BackendConfig config_of(orc_ctx* ctx) {
        std::uint64_t info[64];
        orc_info(ctx, info, 64);
        return BackendConfig{info[0] / 2, static_cast<value_t>(info[5])};
    }
    const BackendConfig& config() const override { return cfg_; }

    Ciphertext encrypt(std::span<const value_t> values) override {
        if (values.empty()) throw DimensionError("cannot encrypt an empty vector");
        if (values.size() > cfg_.slot_count)
            throw CapacityError("vector of length " + std::to_string(values.size()) +
                                " exceeds " + std::to_string(cfg_.slot_count) + " slots");
        std::vector<std::uint64_t> buf(words_);
        check(orc_encrypt(ctx_, values.data(), values.size(), counter_++, buf.data()));
        count(&OpStats::n_encrypt);
        return keep(std::move(buf), 0, values.size(), 0);
    }
    std::vector<value_t> decrypt(const Ciphertext& ct) override {
        count(&OpStats::n_decrypt);
        std::vector<value_t> out(ct.segment_length());
        last_decrypted_ = Minter::id_of(ct);
        check(orc_decrypt(ctx_, buf(ct), out.size(), out.data()));
        return out;
    }
    // Values carry parts (bfv_oracle.cpp XCt): he_mult yields a pending product,
    // he_rot a pending key switch, he_cmult masks a value's plain and key-switch
    // parts, he_add sums parts; every other reader uses the materialised value.
    Ciphertext he_add(const Ciphertext& x, const Ciphertext& y) override {
        same_segment(x, y, "he_add");
        const int kx = kind(x), ky = kind(y);
        std::vector<std::uint64_t> o(orc_kind_words(ctx_, kx | ky));
        check(orc_add_any(ctx_, raw(x), kx, raw(y), ky, o.data()));
        count(&OpStats::n_add);
        return keep(std::move(o), kx | ky, x.segment_length(), std::max(x.depth(), y.depth()));
    }
    Ciphertext he_mult(const Ciphertext& x, const Ciphertext& y) override {
        same_segment(x, y, "he_mult");
        std::vector<std::uint64_t> o(orc_kind_words(ctx_, 1));
        check(orc_mult_pending(ctx_, buf(x), buf(y), o.data()));
        count(&OpStats::n_mult_cc);
        return keep(std::move(o), 1, x.segment_length(), std::max(x.depth(), y.depth()) + 1);
    }
    Ciphertext he_cmult(const Ciphertext& x, std::span<const value_t> mask) override {
        if (mask.size() != x.segment_length())
            throw DimensionError("he_cmult mask length " + std::to_string(mask.size()) +
                                 " does not match segment " +
                                 std::to_string(x.segment_length()));
        std::vector<std::uint64_t> o(orc_kind_words(ctx_, kind(x) & 2));
        int k = 0;
        check(orc_cmult_x(ctx_, raw(x), kind(x), mask.data(), mask.size(), o.data(), &k));
        o.resize(orc_kind_words(ctx_, k));
        count(&OpStats::n_mult_cp);
        return keep(std::move(o), k, x.segment_length(), x.depth());
    }
    Ciphertext he_rot(const Ciphertext& x, std::ptrdiff_t offset) override {
        std::vector<std::uint64_t> o(orc_kind_words(ctx_, 2));
        int k = 0;
        check(orc_rot_x(ctx_, buf(x), offset, o.data(), &k));
        o.resize(orc_kind_words(ctx_, k));
        count(&OpStats::n_rot);
        return keep(std::move(o), k, x.segment_length(), x.depth());
    }
    OpStats stats() const override {
        std::lock_guard<std::mutex> lk(mu_);
        return stats_;
    }
    void reset_stats() override {
        std::lock_guard<std::mutex> lk(mu_);
        stats_ = OpStats{};
        minter_.reset_peak();
    }
    std::size_t peak_live_ciphertexts() const override { return minter_.peak(); }
    void set_phase(Phase p) override { phase_.store(p); }
    Phase phase() const override { return phase_.load(); }

    // the (materialised) ciphertext words of handle id
    const std::vector<std::uint64_t>& ct_words(std::uint64_t id) { return plain(id); }
    std::uint64_t last_decrypted() const { return last_decrypted_; }
    std::uint64_t counter() const { return counter_; }

  private:
    static void check(int rc) {
        if (rc != 0) throw Error(std::string("oracle: ") + orc_last_error());
    }
    static void same_segment(const Ciphertext& x, const Ciphertext& y, const char* what) {
        if (x.segment_length() != y.segment_length())
            throw DimensionError(std::string(what) + " segment mismatch: " +
                                 std::to_string(x.segment_length()) + " vs " +
                                 std::to_string(y.segment_length()));
    }
    void count(PhaseCounts OpStats::*c) {
        const Phase p = phase();
        std::lock_guard<std::mutex> lk(mu_);
        (stats_.*c).bump(p);
    }
    int kind(const Ciphertext& ct) const { return kinds_.at(Minter::id_of(ct)); }
    const std::uint64_t* raw(const Ciphertext& ct) const { return store_.at(Minter::id_of(ct)).data(); }
    // plain value of handle id: a pending product is materialised once, cached
    const std::vector<std::uint64_t>& plain(std::uint64_t id) {
        const std::vector<std::uint64_t>& w = store_.at(id);
        if (kinds_.at(id) == 0) return w;
        auto it = plain_.find(id);
        if (it == plain_.end()) {
            std::vector<std::uint64_t> o(words_);
            check(orc_materialize_kind(ctx_, w.data(), kinds_.at(id), o.data()));
            it = plain_.emplace(id, std::move(o)).first;
        }
        return it->second;
    }
    const std::uint64_t* buf(const Ciphertext& ct) { return plain(Minter::id_of(ct)).data(); }
    Ciphertext keep(std::vector<std::uint64_t> words, int kind, std::size_t seg, std::size_t depth) {
        const std::uint64_t id = store_.size();
        store_.push_back(std::move(words));
        kinds_.push_back(kind);
        return minter_.mint(seg, depth, id, phase());
    }

    orc_ctx* ctx_;
    BackendConfig cfg_;
    Minter minter_;
    std::size_t words_ = 0, pwords_ = 0;
    std::map<std::uint64_t, std::vector<std::uint64_t>> plain_;
    std::uint64_t counter_;
    std::uint64_t last_decrypted_ = 0;
    std::vector<std::vector<std::uint64_t>> store_;
    std::vector<int> kinds_;
    mutable std::mutex mu_;
    OpStats stats_;
    std::atomic<Phase> phase_{Phase::Client};
};

// Records the op stream (kind, offset, mask) while delegating to SlotBackend.
class TraceBackend final : public Backend {
  public:
    explicit TraceBackend(BackendConfig cfg) : inner_(cfg) {}
    struct Op {
        int kind;  // 0 enc 1 dec 2 add 3 mult 4 cmult 5 rot
        std::int64_t arg;  // rot offset / segment
        std::vector<value_t> data;  // cmult mask / encrypt values
    };
    std::vector<Op> ops;
    const BackendConfig& config() const override { return inner_.config(); }
    Ciphertext encrypt(std::span<const value_t> v) override {
        ops.push_back({0, (std::int64_t)v.size(), {v.begin(), v.end()}});
        return inner_.encrypt(v);
    }
    std::vector<value_t> decrypt(const Ciphertext& ct) override {
        ops.push_back({1, (std::int64_t)ct.segment_length(), {}});
        return inner_.decrypt(ct);
    }
    Ciphertext he_add(const Ciphertext& x, const Ciphertext& y) override {
        ops.push_back({2, (std::int64_t)x.segment_length(), {}});
        return inner_.he_add(x, y);
    }
    Ciphertext he_mult(const Ciphertext& x, const Ciphertext& y) override {
        ops.push_back({3, (std::int64_t)x.segment_length(), {}});
        return inner_.he_mult(x, y);
    }
    Ciphertext he_cmult(const Ciphertext& x, std::span<const value_t> m) override {
        ops.push_back({4, (std::int64_t)m.size(), {m.begin(), m.end()}});
        return inner_.he_cmult(x, m);
    }
    Ciphertext he_rot(const Ciphertext& x, std::ptrdiff_t z) override {
        ops.push_back({5, (std::int64_t)z, {}});
        return inner_.he_rot(x, z);
    }
    OpStats stats() const override { return inner_.stats(); }
    void reset_stats() override { inner_.reset_stats(); }
    std::size_t peak_live_ciphertexts() const override { return inner_.peak_live_ciphertexts(); }
    void set_phase(Phase p) override { inner_.set_phase(p); }
    Phase phase() const override { return inner_.phase(); }

  private:
    SlotBackend inner_;
};

Matrix run(int algo, int order, const Matrix& a, const Matrix& b, Backend& be, int flags = 0) {
    MultiplyOptions opts;
    opts.encrypted_client_transforms = (flags & 1) != 0;
    if (order == 0) opts.order = FlattenOrder::ColumnMajor;
    if (order == 1) opts.order = FlattenOrder::RowMajor;
    switch (algo) {
        case 0: return basic_mm(a, b, be, opts);
        case 1: return enhanced_mm(a, b, be, opts);
        case 2: return square_pad_mm(a, b, be, opts);
        default: throw DimensionError("unknown algorithm id");
    }
}

void put_stats(const Backend& be, std::uint64_t* st) {
    if (!st) return;
    const OpStats s = be.stats();
    const PhaseCounts* pc[6] = {&s.n_add, &s.n_mult_cc, &s.n_mult_cp, &s.n_rot, &s.n_encrypt,
                                &s.n_decrypt};
    for (int i = 0; i < 6; ++i) { st[2 * i] = pc[i]->client; st[2 * i + 1] = pc[i]->cloud; }
    st[12] = be.peak_live_ciphertexts();
}

int rc_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const DimensionError*>(&e)) return 1;
    if (dynamic_cast<const CapacityError*>(&e)) return 2;
    if (dynamic_cast<const OverflowError*>(&e)) return 4;
    return 3;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// The reference's own run_campaign (costmodel.cpp:266-314) over SlotBackend{slots, modulus}:
// shapes[c*3 + {0,1,2}] = m, l, n; per (case, algo) in algos_mask bit order (0 hegmm,
// 1 hegmm-en, 2 square-pad): costs[2*k] client_ms, costs[2*k+1] cloud_ms, exact[k],
// stats[12*k + 2*op + phase].
int ref_campaign(std::size_t cases, std::size_t lo, std::size_t hi, std::uint64_t seed, int algos_mask,
                 std::size_t slots, std::int64_t modulus, std::uint64_t* shapes, double* costs,
                 std::uint8_t* exact, std::uint64_t* stats, std::uint64_t* resampled) {
    try {
        CampaignConfig cfg;
        cfg.cases = cases;
        cfg.dim_lo = lo;
        cfg.dim_hi = hi;
        cfg.seed = seed;
        cfg.algos.clear();
        const Algo all[3] = {Algo::Hegmm, Algo::HegmmEn, Algo::SquarePad};
        for (int i = 0; i < 3; ++i)
            if (algos_mask & (1 << i)) cfg.algos.push_back(all[i]);
        cfg.slot_count = slots;
        if (modulus > 0) cfg.plaintext_modulus = modulus;
        const CampaignResult r = run_campaign(cfg);
        std::size_t k = 0;
        for (const CaseReport& c : r.cases) {
            shapes[3 * c.index] = c.m;
            shapes[3 * c.index + 1] = c.l;
            shapes[3 * c.index + 2] = c.n;
            for (const AlgoResult& a : c.results) {
                costs[2 * k] = a.cost.client_ms;
                costs[2 * k + 1] = a.cost.cloud_ms;
                exact[k] = a.exact ? 1 : 0;
                const PhaseCounts* pc[6] = {&a.stats.n_add, &a.stats.n_mult_cc, &a.stats.n_mult_cp,
                                            &a.stats.n_rot, &a.stats.n_encrypt, &a.stats.n_decrypt};
                for (int i = 0; i < 6; ++i) {
                    stats[12 * k + 2 * i] = pc[i]->client;
                    stats[12 * k + 2 * i + 1] = pc[i]->cloud;
                }
                ++k;
            }
        }
        *resampled = r.resampled;
        return 0;
    } catch (const std::exception& e) {
        return rc_of(e);
    }
}

// Reference algorithm over the reference SlotBackend. modulus <= 0: none.
int ref_mm(int algo, int order, const std::int64_t* A, std::size_t m, std::size_t l,
           const std::int64_t* B, std::size_t n, std::size_t slots, std::int64_t modulus,
           std::int64_t* C, std::uint64_t* stats) {
    try {
        Matrix a(m, l, std::vector<value_t>(A, A + m * l));
        Matrix b(l, n, std::vector<value_t>(B, B + l * n));
        BackendConfig cfg{slots, modulus > 0 ? std::optional<value_t>(modulus) : std::nullopt};
        SlotBackend be(cfg);
        const Matrix c = run(algo, order, a, b, be);
        std::memcpy(C, c.data().data(), m * n * 8);
        put_stats(be, stats);
        return 0;
    } catch (const std::exception& e) {
        return rc_of(e);
    }
}

// Same with MultiplyOptions flags (bit 0: encrypted_client_transforms).
int ref_mm2(int algo, int order, int flags, const std::int64_t* A, std::size_t m, std::size_t l,
            const std::int64_t* B, std::size_t n, std::size_t slots, std::int64_t modulus, std::int64_t* C,
            std::uint64_t* stats) {
    try {
        Matrix a(m, l, std::vector<value_t>(A, A + m * l));
        Matrix b(l, n, std::vector<value_t>(B, B + l * n));
        BackendConfig cfg{slots, modulus > 0 ? std::optional<value_t>(modulus) : std::nullopt};
        SlotBackend be(cfg);
        const Matrix c = run(algo, order, a, b, be, flags);
        std::memcpy(C, c.data().data(), m * n * 8);
        put_stats(be, stats);
        return 0;
    } catch (const std::exception& e) {
        return rc_of(e);
    }
}

long ref_trace2(int algo, int order, int flags, const std::int64_t* A, std::size_t m, std::size_t l,
                const std::int64_t* B, std::size_t n, std::size_t slots, std::int64_t* hdr, std::size_t hdr_cap,
                std::int64_t* data, std::size_t data_cap, std::size_t* data_len) {
    try {
        Matrix a(m, l, std::vector<value_t>(A, A + m * l));
        Matrix b(l, n, std::vector<value_t>(B, B + l * n));
        TraceBackend be(BackendConfig{slots, value_t{65537}});
        run(algo, order, a, b, be, flags);
        std::size_t dl = 0;
        for (const auto& op : be.ops) dl += op.data.size();
        if (data_len) *data_len = dl;
        if (hdr) {
            if (hdr_cap < be.ops.size() * 3 || data_cap < dl) return -5;
            std::size_t off = 0;
            for (std::size_t i = 0; i < be.ops.size(); ++i) {
                hdr[3 * i] = be.ops[i].kind;
                hdr[3 * i + 1] = be.ops[i].arg;
                hdr[3 * i + 2] = (std::int64_t)be.ops[i].data.size();
                std::memcpy(data + off, be.ops[i].data.data(), be.ops[i].data.size() * 8);
                off += be.ops[i].data.size();
            }
        }
        return (long)be.ops.size();
    } catch (const std::exception& e) {
        return -rc_of(e);
    }
}

// Reference blocked_mm (algorithms.cpp:434-498) over SlotBackend; log: 4 ints per block
int ref_blocked(int algo, const std::size_t* rows, std::size_t nr, const std::size_t* mids, std::size_t nm,
                const std::size_t* cols, std::size_t nc, const std::int64_t* A, std::size_t m, std::size_t l,
                const std::int64_t* B, std::size_t n, std::size_t slots, std::int64_t modulus, std::int64_t* C,
                std::int32_t* log) {
    try {
        Matrix a(m, l, std::vector<value_t>(A, A + m * l));
        Matrix b(l, n, std::vector<value_t>(B, B + l * n));
        BlockPlan plan{std::vector<std::size_t>(rows, rows + nr), std::vector<std::size_t>(mids, mids + nm),
                       std::vector<std::size_t>(cols, cols + nc)};
        BackendConfig cfg{slots, modulus > 0 ? std::optional<value_t>(modulus) : std::nullopt};
        SlotBackend be(cfg);
        std::vector<BlockRun> runs;
        const Algo al = algo == 0 ? Algo::Hegmm : algo == 1 ? Algo::HegmmEn : Algo::SquarePad;
        const Matrix c = blocked_mm(a, b, plan, al, be, &runs);
        std::memcpy(C, c.data().data(), m * n * 8);
        for (std::size_t i = 0; log && i < runs.size(); ++i) {
            log[4 * i] = runs[i].used == Algo::Hegmm ? 0 : runs[i].used == Algo::HegmmEn ? 1 : 2;
            log[4 * i + 1] = runs[i].fell_back ? 1 : 0;
            log[4 * i + 2] = (std::int32_t)runs[i].m;
            log[4 * i + 3] = (std::int32_t)runs[i].l;
        }
        return 0;
    } catch (const std::exception& e) {
        return rc_of(e);
    }
}

// Reference naive_matmul_mod (matrix.cpp:223-239).
int ref_naive_mod(const std::int64_t* A, std::size_t m, std::size_t l, const std::int64_t* B,
                  std::size_t n, std::int64_t q, std::int64_t* C) {
    try {
        Matrix a(m, l, std::vector<value_t>(A, A + m * l));
        Matrix b(l, n, std::vector<value_t>(B, B + l * n));
        const Matrix c = naive_matmul_mod(a, b, q);
        std::memcpy(C, c.data().data(), m * n * 8);
        return 0;
    } catch (const std::exception& e) {
        return rc_of(e);
    }
}

// Op stream of a reference run: per op (kind, arg, data_len) into `hdr` (3
// words each) and the concatenated data into `data`.  Returns the op count, or
// a negative error code; counts only when the buffers are null.
long ref_trace(int algo, int order, const std::int64_t* A, std::size_t m, std::size_t l,
               const std::int64_t* B, std::size_t n, std::size_t slots, std::int64_t* hdr,
               std::size_t hdr_cap, std::int64_t* data, std::size_t data_cap,
               std::size_t* data_len) {
    try {
        Matrix a(m, l, std::vector<value_t>(A, A + m * l));
        Matrix b(l, n, std::vector<value_t>(B, B + l * n));
        TraceBackend be(BackendConfig{slots, value_t{65537}});
        run(algo, order, a, b, be);
        std::size_t dl = 0;
        for (const auto& op : be.ops) dl += op.data.size();
        if (data_len) *data_len = dl;
        if (hdr) {
            if (hdr_cap < be.ops.size() * 3 || data_cap < dl) return -5;
            std::size_t off = 0;
            for (std::size_t i = 0; i < be.ops.size(); ++i) {
                hdr[3 * i] = be.ops[i].kind;
                hdr[3 * i + 1] = be.ops[i].arg;
                hdr[3 * i + 2] = (std::int64_t)be.ops[i].data.size();
                std::memcpy(data + off, be.ops[i].data.data(), be.ops[i].data.size() * 8);
                off += be.ops[i].data.size();
            }
        }
        return (long)be.ops.size();
    } catch (const std::exception& e) {
        return -rc_of(e);
    }
}

// Reference algorithm over the CPU BFV oracle.  Writes the decrypted product,
// the words of the ciphertext that was decrypted, the stats, and returns the
// encryption counter after the run (the next free counter).
long ref_mm_oracle(int param_id, std::uint64_t seed, std::uint64_t counter0, int algo, int order,
                   const std::int64_t* A, std::size_t m, std::size_t l, const std::int64_t* B,
                   std::size_t n, std::int64_t* C, std::uint64_t* final_ct,
                   std::uint64_t* stats) {
    orc_ctx* ctx = orc_create(param_id, seed);
    if (!ctx) { g_err = orc_last_error(); return -3; }
    try {
        Matrix a(m, l, std::vector<value_t>(A, A + m * l));
        Matrix b(l, n, std::vector<value_t>(B, B + l * n));
        OracleBackend be(ctx, counter0);
        const Matrix c = run(algo, order, a, b, be);
        std::memcpy(C, c.data().data(), m * n * 8);
        if (final_ct) {
            const auto& w = be.ct_words(be.last_decrypted());
            std::memcpy(final_ct, w.data(), w.size() * 8);
        }
        put_stats(be, stats);
        const long next = (long)be.counter();
        orc_destroy(ctx);
        return next;
    } catch (const std::exception& e) {
        orc_destroy(ctx);
        return -rc_of(e);
    }
}

// Persistent oracle session (keys and tables built once, reused across products);
// one session per thread.
void* ref_oracle_session_create(int param_id, std::uint64_t seed) {
    orc_ctx* ctx = orc_create(param_id, seed);
    if (!ctx) g_err = orc_last_error();
    return ctx;
}
void ref_oracle_session_destroy(void* s) { orc_destroy(static_cast<orc_ctx*>(s)); }
long ref_oracle_session_mm(void* s, std::uint64_t counter0, int algo, int order, const std::int64_t* A,
                           std::size_t m, std::size_t l, const std::int64_t* B, std::size_t n,
                           std::int64_t* C) {
    try {
        Matrix a(m, l, std::vector<value_t>(A, A + m * l));
        Matrix b(l, n, std::vector<value_t>(B, B + l * n));
        OracleBackend be(static_cast<orc_ctx*>(s), counter0);
        const Matrix c = run(algo, order, a, b, be);
        std::memcpy(C, c.data().data(), m * n * 8);
        return (long)be.counter();
    } catch (const std::exception& e) {
        return -rc_of(e);
    }
}

}  // extern "C"
