// engine.hpp -- HE programs and their batched execution on one GPU.
//
// A Program is the cloud-side op DAG of one HEGMM call (or of the pending
// ops of a lazy session), recorded through the reference's op vocabulary:
// encrypt / he_rot / he_cmult / he_add / he_mult (backend.hpp:113-119).
// The executor runs it for K independent instances in lockstep and applies
// only EXACT rewrites, so results stay bit-identical to op-by-op execution
// (oracle/bfv_oracle.cpp):
//   * he_rot by 0 (mod N/2) is the identity;
//   * identical rotations of one ciphertext are computed once (CSE);
//   * all rotations of one ciphertext share one ModUp (hoisting; exact because
//     the digit lift uses centred residues and commutes with X -> X^g);
//   * trees of he_add over he_cmult / he_add become one masked sum
//     (modular adds are associative and commutative);
//   * he_mult is a PENDING product and he_rot a PENDING key switch (oracle
//     XCt): add trees and masked sums work on the parts (tensors, Q ++ P
//     accumulators, plain ciphertexts), and scale-and-round + relinearisation
//     or ModDown run once when another op reads the value (a Mat node); a
//     product whose only reader is such a sum is accumulated straight into the
//     sum's tensor (fused: its own tensor is never stored);
//   * a masked sum of rotations sum_t m_t (.) Rot(x_t, g_t) whose masks belong to a
//     cached program is ONE key inner product over masked keys m_t (.) key_{g_t}
//     (mask multiplication distributes over the inner product mod q: the same
//     canonical residues as rotating, masking and adding);
//   * every op of one dependency level is one batched launch sequence over
//     all (node, instance) pairs; rotations are grouped by Galois key so that
//     one key read from HBM serves the whole group.
#pragma once
#include <functional>
#include <atomic>
#include <memory>
#include <vector>

#include "context.hpp"

namespace hgm {

struct MaskData {
    std::vector<i64> v;
    // masks of cached (never freed) HEGMM programs are `stable`: the device copy is
    // then found by id, without hashing the content (ids are never reused)
    bool stable = false;
    u64 id = next_id();
    static u64 next_id() {
        static std::atomic<u64> n{1};
        return n.fetch_add(1, std::memory_order_relaxed);
    }
};
using MaskRef = std::shared_ptr<const MaskData>;

struct PNode {
    enum Kind : unsigned char { Input, Enc, Rot, Comb, Mult, Mat };
    Kind kind = Input;
    std::vector<int> in;          // Rot / Mat: {src}; Mult: {a, b}; Comb: term inputs
    std::vector<MaskRef> masks;   // Comb: one per term, null = plain addend
    std::vector<char> fused;      // Comb (set by optimise): term is a Mult accumulated in place
    int pend = 0;                 // Input: kind of the supplied value (0: plain, ExecIO::input;
                                  // else parts, ExecIO::input_pending)
    u32 g = 1;                    // Rot: Galois element
    int slot = -1;                // Input / Enc: external index
    size_t S = 0;                 // logical segment length
};

struct Program {
    std::vector<PNode> nodes;
    std::vector<int> outputs;
    int n_inputs = 0;  // Input slots
    int n_enc = 0;     // Enc slots
    int add_input(size_t S, int kind = 0);
    int add_enc(size_t S);
    int add_rot(int src, u32 g);
    int add_comb(std::vector<int> in, std::vector<MaskRef> masks);
    int add_mult(int a, int b);
};

// A value's parts (oracle XCt): T a pending product (unscaled tensor over
// Q ++ B), A a pending key switch (accumulator over Q ++ P), X a plain
// ciphertext; plain nodes have kind kPartX.  A non-plain value is stored as
// [T][A][X] with only its parts present (part_layout).
enum : int { kPartT = 1, kPartA = 2, kPartX = 4 };
struct PartLayout {
    size_t t = 0, a = 0, x = 0, words = 0;
};
PartLayout part_layout(const Context& ctx, int kind);

// One rotation of a masked sum whose key-switch part is computed straight from
// the ModUp digits (k_ks_plan): the masks of every term reading that rotation.
struct KsTerm {
    int rot = -1, src = -1;  // the (never stored) Rot node and its source
    u32 g = 1;
    std::vector<MaskRef> masks;
};

// Optimised, levelised form of a Program (built once, reused for every batch).
struct Schedule {
    Program prog;                        // rewritten program
    std::vector<std::vector<int>> levels;
    std::vector<int> last_use_level;     // -1: never read
    std::vector<char> is_output;
    std::vector<int> kind;               // value parts per node (kPartT | kPartA | kPartX)
    std::vector<int> pending_out;        // per output: node whose parts are also returned, or -1
    std::vector<char> is_pending_output;
    size_t rot_count = 0, comb_count = 0, mult_count = 0, pending_count = 0, mat_count = 0;
    size_t moddown_count = 0, rescale_count = 0;  // Mat nodes reading a key-switch / product part
    // Masked sums of rotations (stable masks only): ks_terms[x] non-empty = Comb x's
    // key-switch part is one inner product over its rotations' masked keys; a Rot
    // read only by such sums is virtual (no level, no buffer).
    std::vector<std::vector<KsTerm>> ks_terms;
    std::vector<char> virt;
    // prescale[x]: masked sum x (ks_terms) is read only by its own ModDown, so its
    // masked keys may carry P^-1 over Q and that ModDown skips the product
    std::vector<char> prescale;
    size_t ks_comb_count = 0, masked_key_count = 0, acc_comb_count = 0;
    size_t stored_rot_count = 0;  // rot_count counts every rotation after CSE, stored or not
};
Schedule optimise(const Program& p);

struct ExecIO {
    int K = 1;
    // Input slot s of instance k -> device ciphertext
    std::function<const u64*(int s, int k)> input;
    // Enc slot s of instance k -> host values and encryption counter
    std::function<const i64*(int s, int k)> enc_values;
    std::function<u64(int s, int k)> enc_counter;
    // Input slot s of instance k -> its pending form (Input nodes with pend set)
    std::function<const u64*(int s, int k)> input_pending;
    // if set: receives, per output, a buffer of K non-plain values (or nullptr) and their kind
    std::vector<u64*>* pending_out = nullptr;
    std::vector<int>* pending_kind = nullptr;
};

// Executes `sch` for io.K instances; returns, for each output o, a device
// buffer of K consecutive ciphertexts (caller releases with ctx.release).
std::vector<u64*> execute(Context& ctx, const Schedule& sch, const ExecIO& io);

// Kernel-launch accounting of the last execute() on this thread.
struct ExecCounters {
    size_t levels = 0, launches = 0, rot_items = 0, modup_items = 0, comb_items = 0,
           mult_items = 0, enc_items = 0, mat_items = 0, plan_items = 0;
};
ExecCounters last_exec_counters();

}  // namespace hgm
