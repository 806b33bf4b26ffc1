// hegmm_algos.hpp -- the HEGMM algorithms as HE programs.
//
// A from-scratch implementation of the reference's algorithm layer
// (proj/src/algorithms.cpp, proj/src/lintrans.cpp, proj/src/matrix.cpp) that,
// instead of calling a Backend op by op, records the identical op stream once
// per product shape into an engine Program and then runs that program for any
// number of instances.  The op stream (order, rotation offsets, masks, counts
// per phase) is pinned against the reference by tests/test_op_stream.py.
#pragma once
#include <array>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.hpp"

namespace hgm {

enum class Order { Col = 0, Row = 1 };
enum class Algo { Basic = 0, Enhanced = 1, SquarePad = 2 };
// MultiplyOptions (algorithms.hpp:15-22) as flags
constexpr int kFlagEncryptedClientTransforms = 1;
enum class Dup { None, AVertical, BHorizontal };

// errors raised with the reference's exception classes (errors.hpp:17-27)
struct DimensionError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CapacityError : std::runtime_error { using std::runtime_error::runtime_error; };

struct Mat {
    size_t rows = 0, cols = 0;
    std::vector<i64> d;  // row-major
    Mat() = default;
    Mat(size_t r, size_t c) : rows(r), cols(c), d(r * c, 0) {}
    i64& at(size_t r, size_t c) { return d[r * cols + c]; }
    i64 at(size_t r, size_t c) const { return d[r * cols + c]; }
};

inline size_t flat_index(size_t r, size_t c, size_t rows, size_t cols, Order o) {
    return o == Order::Col ? r + c * rows : r * cols + c;
}

// Op counters per phase, OpStats field order (backend.hpp:50-57):
// add, mult_cc, mult_cp, rot, encrypt, decrypt; [k][0] client, [k][1] cloud.
struct Counts {
    std::array<std::array<u64, 2>, 6> c{};
    u64& at(int op, int phase) { return c[op][phase]; }
};
enum { kAdd = 0, kMultCC = 1, kMultCP = 2, kRot = 3, kEnc = 4, kDec = 5 };

// One diagonal of a plan: output slot i reads input slot i + offset where mask[i] = 1.
struct PlanEntry {
    i64 offset;
    MaskRef mask;  // 0/1 values, length = plan segment
};
struct Plan {
    std::vector<PlanEntry> entries;  // ascending offsets
    size_t in_len = 0, out_len = 0;
    size_t rotations() const;
};

struct Strategy {
    size_t p = 1, t = 1;
    Dup dup = Dup::None;
    Order order = Order::Col;
    size_t rows_w = 1, cols_w = 1, segment = 1;
    Counts predicted;
};
Strategy select_strategy(size_t m, size_t l, size_t n);

// A product shape compiled to a program.
struct MatmulProgram {
    Algo algo = Algo::Basic;
    size_t m = 0, l = 0, n = 0, segment = 0, slots = 0;  // dims the program runs on
    size_t m0 = 0, l0 = 0, n0 = 0;                        // caller's dims (square_pad pads)
    bool enc_transforms = false;
    Order order = Order::Col;
    Strategy strat;
    Schedule sched;        // client encrypt + cloud (encryptions are level 0)
    Schedule cloud_sched;  // cloud only: the encrypted inputs are Input slots
    int n_enc = 0;
    Counts counts;  // per instance, by phase
    // op stream in call order: (kind, arg) with kind 0 enc 1 dec 2 add 3 mult 4 cmult 5 rot
    std::vector<std::pair<int, i64>> stream;
    std::vector<MaskRef> stream_masks;  // one per cmult, in call order
    // client side
    std::vector<std::vector<i64>> pack(const i64* A, const i64* B) const;
    void unpack(const std::vector<i64>& slots_out, i64* C) const;
};

// Cached per (algo, order, flags, m, l, n, slots, N); order: -1 auto.
std::shared_ptr<const MatmulProgram> get_matmul_program(int algo, int order, size_t m, size_t l,
                                                        size_t n, size_t slots, u32 N, int flags = 0);
// Working flattened length of each algorithm (algorithms.cpp:172-196)
size_t enhanced_segment(size_t m, size_t l, size_t n);
bool fits(int algo, size_t m, size_t l, size_t n, size_t slots);

// Plans (exposed for tests)
std::shared_ptr<const Plan> eps_plan_embedded(size_t k, size_t m, size_t l, size_t n, Order o,
                                              size_t segment);
std::shared_ptr<const Plan> omega_plan_embedded(size_t k, size_t l, size_t m, size_t n, Order o,
                                                size_t segment);
std::shared_ptr<const Plan> shaped_eps_plan(size_t k, size_t rows, size_t out_cols, size_t period,
                                            Order o, size_t segment);
std::shared_ptr<const Plan> shaped_omega_plan(size_t k, size_t out_rows, size_t cols,
                                              size_t period, Order o, size_t segment);

}  // namespace hgm
