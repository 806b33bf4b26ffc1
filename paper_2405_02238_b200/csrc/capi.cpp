// capi.cpp -- the extern "C" boundary (include/hegmm_b200.h).
//
// A session (hgm_ctx) records every primitive call as a node of a lazy op
// graph and counts it immediately, exactly like the reference backend counts
// (backend.cpp:103-107, one counter bump per call, split by phase).  Work is
// executed when a result is needed (decrypt / export / flush): the pending
// sub-graph becomes a Program and runs through the batched executor, so the
// many independent rotations and masks of one HEGMM call share launches and
// ModUps.  Nodes still referenced by a pinned handle keep their ciphertext;
// every other intermediate is recomputed on demand (all ops are deterministic).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <functional>
#include <future>
#include <map>
#include <tuple>
#include <algorithm>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/hegmm_b200.h"
#include "capi_internal.hpp"
#include "context.hpp"
#include "engine.hpp"
#include "parallel.hpp"
#include "hegmm_algos.hpp"

using namespace hgm;

namespace {

thread_local std::string g_err;

struct DevBuf {
    Context* ctx;
    u64* p;
    DevBuf(Context* c, u64* q) : ctx(c), p(q) {}
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) ctx->release(p);
    }
};

struct SNode {
    PNode::Kind kind = PNode::Input;
    std::vector<std::shared_ptr<SNode>> in;
    std::vector<MaskRef> masks;
    u32 g = 1;
    size_t S = 0, depth = 0;
    int phase = 0;
    std::vector<i64> values;  // Enc
    u64 counter = 0;          // Enc
    std::shared_ptr<DevBuf> buf;
    std::shared_ptr<DevBuf> pbuf;  // the value's parts (engine.hpp), when it is not plain
    int pkind = 0;
    std::atomic<int> pins{0};
};

}  // namespace

// A session.  It is reference counted: the creator holds one reference and
// every live handle and batch holds one, so hgm_ctx_destroy with handles still
// alive only drops the creator's reference and the context (its device memory
// and keys) goes away with the last handle (no use-after-free from late
// releases, e.g. Python finalisers running after Context.close()).
struct hgm_ctx {
    std::unique_ptr<Context> ctx;
    int device = 0;
    bool os_seed = false;            // seed drawn from the OS CSPRNG: never exported
    std::mutex mu;                   // counters, encryption counter, pending registry
    std::recursive_mutex exec_mu;    // everything that touches the device (flush, batches, ring)
    std::atomic<int> phase{0};
    std::atomic<int> refs{1};
    Counts counts;
    u64 enc_counter = 0;
    std::atomic<size_t> live{0}, peak{0};
    // nodes handed out unmaterialised (hgm_flush materialises the pinned ones)
    std::vector<std::weak_ptr<SNode>> pending;
};

struct hgm_ct {
    hgm_ctx* owner;
    std::shared_ptr<SNode> node;
    std::atomic<int> refs{1};
    bool pinned = true;
};

namespace {

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

void ctx_retain(hgm_ctx* c) { c->refs.fetch_add(1, std::memory_order_relaxed); }
void ctx_release(hgm_ctx* c) {
    if (c->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) {
        c->pending.clear();
        c->ctx.reset();  // Context's destructor sets and restores its own device
        delete c;
    }
}

// Makes the context's device current for the duration of an entry point and
// restores the caller's current device afterwards (the library may be called
// from any thread, and a process may hold contexts on several GPUs).
struct DeviceScope {
    int prev = -1, want;
    explicit DeviceScope(const hgm_ctx* c) : want(c ? c->device : -1) {
        if (want < 0) return;
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != want) cudaSetDevice(want);
    }
    ~DeviceScope() {
        if (want >= 0 && prev >= 0 && prev != want) cudaSetDevice(prev);
    }
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return HGM_OK;
    } catch (const hgm::DimensionError& e) {
        return fail(HGM_EDIM, e.what());
    } catch (const hgm::CapacityError& e) {
        return fail(HGM_ECAP, e.what());
    } catch (const CudaError& e) {
        return fail(HGM_ECUDA, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(HGM_EARG, e.what());
    } catch (const std::exception& e) {
        return fail(HGM_EINTERNAL, e.what());
    }
}

// Reserves n consecutive encryption counters of the session (atomically, so
// concurrent and repeated calls never reuse (u, e0, e1)).
u64 reserve_counters(hgm_ctx* c, u64 n) {
    std::lock_guard<std::mutex> lk(c->mu);
    const u64 first = c->enc_counter;
    c->enc_counter += n;
    return first;
}

// counter0 == HGM_COUNTER_AUTO: the next count * E counters of the session
u64 resolve_counter0(hgm_ctx* c, uint64_t counter0, u64 n) {
    return counter0 == HGM_COUNTER_AUTO ? reserve_counters(c, n) : counter0;
}

u64 os_random_u64() {
    u64 v = 0;
    std::ifstream f("/dev/urandom", std::ios::binary);
    if (!f.read(reinterpret_cast<char*>(&v), sizeof(v))) throw std::runtime_error("cannot read /dev/urandom");
    return v;
}

void bump(hgm_ctx* c, int op) {
    std::lock_guard<std::mutex> lk(c->mu);
    c->counts.at(op, c->phase.load())++;
}

hgm_ct* make_handle(hgm_ctx* c, std::shared_ptr<SNode> n) {
    auto* h = new hgm_ct;
    h->owner = c;
    ctx_retain(c);
    if (!n->buf) {
        std::lock_guard<std::mutex> lk(c->mu);
        if (c->pending.size() >= 1024)  // prune released / materialised entries now and then
            c->pending.erase(std::remove_if(c->pending.begin(), c->pending.end(),
                                            [](const std::weak_ptr<SNode>& w) {
                                                auto p = w.lock();
                                                return !p || p->buf;
                                            }),
                             c->pending.end());
        c->pending.push_back(n);
    }
    h->node = std::move(n);
    h->node->pins++;
    const size_t now = ++c->live;
    size_t seen = c->peak.load();
    while (seen < now && !c->peak.compare_exchange_weak(seen, now)) {
    }
    return h;
}

std::shared_ptr<SNode> new_node(hgm_ctx* c, PNode::Kind k, size_t S, size_t depth) {
    auto n = std::make_shared<SNode>();
    n->kind = k;
    n->S = S;
    n->depth = depth;
    n->phase = c->phase.load();
    return n;
}

void check_values(hgm_ctx* c, size_t S) {
    if (S == 0) throw hgm::DimensionError("cannot encrypt an empty vector");
    if (S > c->ctx->slots())
        throw hgm::CapacityError("vector of length " + std::to_string(S) + " exceeds " +
                                 std::to_string(c->ctx->slots()) + " slots");
}

// Materialise `targets` (and every pinned node on their pending sub-graph).
void flush(hgm_ctx* c, const std::vector<std::shared_ptr<SNode>>& targets) {
    std::unordered_map<SNode*, int> index;
    std::vector<std::shared_ptr<SNode>> order;  // topological
    std::vector<std::shared_ptr<SNode>> inputs;
    Program prog;
    // iterative post-order DFS
    struct Frame {
        std::shared_ptr<SNode> n;
        size_t next;
    };
    for (const auto& t : targets) {
        if (t->buf || index.count(t.get())) continue;
        std::vector<Frame> st{{t, 0}};
        while (!st.empty()) {
            Frame& f = st.back();
            SNode* n = f.n.get();
            if (index.count(n)) {
                st.pop_back();
                continue;
            }
            if (!n->buf && f.next < n->in.size()) {
                auto child = n->in[f.next++];
                if (!index.count(child.get())) st.push_back({child, 0});
                continue;
            }
            int id;
            if (n->buf) {
                id = prog.add_input(n->S, n->pbuf ? n->pkind : 0);
                inputs.push_back(f.n);
            } else {
                std::vector<int> in;
                for (auto& x : n->in) in.push_back(index.at(x.get()));
                switch (n->kind) {
                    case PNode::Enc: id = prog.add_enc(n->S); break;
                    case PNode::Rot: id = prog.add_rot(in[0], n->g); break;
                    case PNode::Comb: id = prog.add_comb(in, n->masks); break;
                    case PNode::Mult: id = prog.add_mult(in[0], in[1]); break;
                    default: throw std::logic_error("unmaterialised input node");
                }
            }
            index.emplace(n, id);
            order.push_back(f.n);
            st.pop_back();
        }
    }
    // outputs: targets, plus pending nodes somebody still holds a pinned handle to
    std::vector<std::shared_ptr<SNode>> outs;
    for (const auto& t : targets)
        if (!t->buf) outs.push_back(t);
    for (const auto& n : order)
        if (!n->buf && n->pins.load() > 0) outs.push_back(n);
    if (outs.empty()) return;
    std::unordered_map<SNode*, size_t> out_pos;
    std::vector<std::shared_ptr<SNode>> uniq;
    for (auto& n : outs)
        if (!out_pos.count(n.get())) {
            out_pos.emplace(n.get(), uniq.size());
            uniq.push_back(n);
            prog.outputs.push_back(index.at(n.get()));
        }
    std::vector<SNode*> encs;
    for (const auto& n : order)
        if (!n->buf && n->kind == PNode::Enc) encs.push_back(n.get());
    const Schedule sch = optimise(prog);
    ExecIO io;
    io.K = 1;
    io.input = [&](int s, int) { return (const u64*)inputs[s]->buf->p; };
    io.enc_values = [&](int s, int) { return (const i64*)encs[s]->values.data(); };
    io.enc_counter = [&](int s, int) { return encs[s]->counter; };
    io.input_pending = [&](int s, int) { return (const u64*)inputs[s]->pbuf->p; };
    std::vector<u64*> pres;
    std::vector<int> pkinds;
    io.pending_out = &pres;
    io.pending_kind = &pkinds;
    std::vector<u64*> res = execute(*c->ctx, sch, io);
    for (size_t i = 0; i < uniq.size(); ++i) {
        uniq[i]->buf = std::make_shared<DevBuf>(c->ctx.get(), res[i]);
        // a non-plain value keeps its parts: later he_adds / he_cmults work on them
        if (pres[i]) {
            uniq[i]->pbuf = std::make_shared<DevBuf>(c->ctx.get(), pres[i]);
            uniq[i]->pkind = pkinds[i];
        }
        uniq[i]->in.clear();  // materialised: history no longer needed
    }
}

const SNode& node_of(const hgm_ct* h) { return *h->node; }

}  // namespace

extern "C" {

const char* hgm_last_error(void) { return g_err.c_str(); }

hgm_ctx* hgm_ctx_create_ex(int param_id, uint64_t seed, int device, int flags) {
    hgm_ctx* c = nullptr;
    const int rc = guarded([&] {
        if (flags & ~(HGM_CTX_KEYLESS | HGM_CTX_OS_SEED)) throw std::invalid_argument("unknown context flags");
        if (device < 0) throw std::invalid_argument("negative device ordinal");
        auto h = std::make_unique<hgm_ctx>();
        h->device = device;
        u32 key[8];
        if (flags & HGM_CTX_OS_SEED) {  // ChaCha12 keyed from the OS CSPRNG (never exported)
            h->os_seed = true;
            seed = os_random_u64();  // only the wire format's key-set fingerprint uses it
            for (int i = 0; i < 4; ++i) {
                const u64 v = os_random_u64();
                key[2 * i] = (u32)v;
                key[2 * i + 1] = (u32)(v >> 32);
            }
        }
        int prev = -1;
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        try {
            h->ctx = std::make_unique<Context>(param_id, seed, device, (flags & HGM_CTX_KEYLESS) != 0,
                                               h->os_seed ? key : nullptr);
        } catch (...) {
            if (prev >= 0) cudaSetDevice(prev);
            throw;
        }
        if (prev >= 0 && prev != device) cudaSetDevice(prev);  // the constructor made `device` current
        c = h.release();
    });
    return rc == HGM_OK ? c : nullptr;
}

hgm_ctx* hgm_ctx_create(int param_id, uint64_t seed, int device) {
    return hgm_ctx_create_ex(param_id, seed, device, 0);
}

void hgm_ctx_destroy(hgm_ctx* c) {
    if (c) ctx_release(c);
}

int hgm_ctx_info(const hgm_ctx* c, uint64_t* info, size_t cap) {
    const HostParams& h = c->ctx->host();
    if (cap < 8 + h.primes.size()) return fail(HGM_EARG, "info buffer too small");
    info[0] = h.N; info[1] = h.L; info[2] = h.K; info[3] = h.nB; info[4] = h.dnum;
    info[5] = kT; info[6] = h.alpha; info[7] = c->os_seed ? 0 : h.seed;
    for (size_t i = 0; i < h.primes.size(); ++i) info[8 + i] = h.primes[i];
    return HGM_OK;
}

size_t hgm_key_words(const hgm_ctx* c, int kind) {
    try {
        return c->ctx->key_words(kind);
    } catch (...) {
        return 0;
    }
}

int hgm_key_export(hgm_ctx* c, int kind, uint32_t elt, uint64_t* words, size_t n) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);
    DeviceScope dev(c);
    return guarded([&] {
        if (!words) throw std::invalid_argument("null output buffer");
        if (n < c->ctx->key_words(kind)) throw std::invalid_argument("key buffer too small");
        c->ctx->export_key(kind, elt, words);
    });
}

int hgm_key_upload(hgm_ctx* c, int kind, uint32_t elt, const uint64_t* words, size_t n) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);
    DeviceScope dev(c);
    return guarded([&] {
        if (!words) throw std::invalid_argument("null key buffer");
        c->ctx->upload_key(kind, elt, words, n);
    });
}

int hgm_key_drop_secret(hgm_ctx* c) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);
    DeviceScope dev(c);
    return guarded([&] { c->ctx->drop_secret(); });
}

int hgm_key_has(const hgm_ctx* c, int kind) {
    return kind == 0 ? c->ctx->has_secret() : kind == 1 ? c->ctx->has_public() : 0;
}

uint32_t hgm_galois_element(const hgm_ctx* c, int64_t offset) {
    return Context::galois_of(offset, (u32)c->ctx->host().N);
}
size_t hgm_slot_count(const hgm_ctx* c) { return c->ctx->slots(); }
size_t hgm_ct_words(const hgm_ctx* c) { return c->ctx->ct_words(); }

int hgm_encrypt_at(hgm_ctx* c, const int64_t* values, size_t S, uint64_t counter, hgm_ct** out) {
    return guarded([&] {
        check_values(c, S);
        if (!c->ctx->has_public()) throw std::invalid_argument("context holds no public key: upload it with hgm_key_upload");
        auto n = new_node(c, PNode::Enc, S, 0);
        n->values.assign(values, values + S);
        n->counter = counter;
        bump(c, kEnc);
        *out = make_handle(c, std::move(n));
    });
}
int hgm_encrypt(hgm_ctx* c, const int64_t* values, size_t S, hgm_ct** out) {
    // the counter is reserved atomically BEFORE encrypting: concurrent callers
    // never share (u, e0, e1); a failed call leaves a harmless gap
    return hgm_encrypt_at(c, values, S, reserve_counters(c, 1), out);
}

int hgm_encrypt_noise(hgm_ctx* c, const int64_t* values, size_t S, const int64_t* u, const int64_t* e0,
                      const int64_t* e1, hgm_ct** out) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);
    DeviceScope dev(c);
    return guarded([&] {
        check_values(c, S);
        if (!u || !e0 || !e1 || !out) throw std::invalid_argument("null noise or output buffer");
        const size_t N = c->ctx->host().N, W = c->ctx->ct_words();
        std::vector<i64> noise(3 * N);
        std::copy(u, u + N, noise.begin());
        std::copy(e0, e0 + N, noise.begin() + N);
        std::copy(e1, e1 + N, noise.begin() + 2 * N);
        const i64* vals = values;
        u64* p = c->ctx->alloc(W);
        try {
            c->ctx->encrypt_noise(1, &vals, &S, noise.data(), &p);
        } catch (...) {
            c->ctx->release(p);
            throw;
        }
        auto n = new_node(c, PNode::Input, S, 0);
        n->buf = std::make_shared<DevBuf>(c->ctx.get(), p);
        bump(c, kEnc);
        *out = make_handle(c, std::move(n));
    });
}

uint64_t hgm_reserve_counters(hgm_ctx* c, uint64_t n) { return reserve_counters(c, n); }

int hgm_decrypt(hgm_ctx* c, const hgm_ct* ct, int64_t* out, size_t cap) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        bump(c, kDec);
        const size_t S = node_of(ct).S;
        if (cap < S) throw std::invalid_argument("decrypt output buffer smaller than the segment");
        flush(c, {ct->node});
        const u64* p = ct->node->buf->p;
        c->ctx->decrypt(1, &p, &S, &out);
    });
}

int hgm_add(hgm_ctx* c, const hgm_ct* x, const hgm_ct* y, hgm_ct** out) {
    return guarded([&] {
        const SNode &a = node_of(x), &b = node_of(y);
        if (a.S != b.S)
            throw hgm::DimensionError("he_add segment mismatch: " + std::to_string(a.S) + " vs " + std::to_string(b.S));
        auto n = new_node(c, PNode::Comb, a.S, std::max(a.depth, b.depth));
        n->in = {x->node, y->node};
        n->masks = {nullptr, nullptr};
        bump(c, kAdd);
        *out = make_handle(c, std::move(n));
    });
}

int hgm_mul(hgm_ctx* c, const hgm_ct* x, const hgm_ct* y, hgm_ct** out) {
    return guarded([&] {
        const SNode &a = node_of(x), &b = node_of(y);
        if (a.S != b.S)
            throw hgm::DimensionError("he_mult segment mismatch: " + std::to_string(a.S) + " vs " + std::to_string(b.S));
        auto n = new_node(c, PNode::Mult, a.S, std::max(a.depth, b.depth) + 1);
        n->in = {x->node, y->node};
        bump(c, kMultCC);
        *out = make_handle(c, std::move(n));
    });
}

int hgm_cmul(hgm_ctx* c, const hgm_ct* x, const int64_t* mask, size_t S, hgm_ct** out) {
    return guarded([&] {
        const SNode& a = node_of(x);
        if (S != a.S)
            throw hgm::DimensionError("he_cmult mask length " + std::to_string(S) + " does not match segment " +
                                      std::to_string(a.S));
        auto md = std::make_shared<MaskData>();
        md->v.assign(mask, mask + S);
        auto n = new_node(c, PNode::Comb, a.S, a.depth);
        n->in = {x->node};
        n->masks = {md};
        bump(c, kMultCP);
        *out = make_handle(c, std::move(n));
    });
}

int hgm_rot(hgm_ctx* c, const hgm_ct* x, int64_t z, hgm_ct** out) {
    return guarded([&] {
        const SNode& a = node_of(x);
        auto n = new_node(c, PNode::Rot, a.S, a.depth);
        n->in = {x->node};
        n->g = Context::galois_of(z, (u32)c->ctx->host().N);
        bump(c, kRot);
        *out = make_handle(c, std::move(n));
    });
}

int hgm_apply_plan(hgm_ctx* c, const hgm_ct* x, size_t n_entries, const int64_t* offsets,
                   const int64_t* masks, size_t S, hgm_ct** out) {
    return guarded([&] {
        const SNode& a = node_of(x);
        if (S != a.S)
            throw hgm::DimensionError("ciphertext segment " + std::to_string(a.S) + " does not match plan length " +
                                      std::to_string(S));
        if (n_entries == 0) throw hgm::DimensionError("cannot apply an empty plan");
        std::shared_ptr<SNode> acc;
        for (size_t e = 0; e < n_entries; ++e) {
            std::shared_ptr<SNode> src = x->node;
            if (offsets[e] != 0) {
                auto r = new_node(c, PNode::Rot, S, a.depth);
                r->in = {x->node};
                r->g = Context::galois_of(offsets[e], (u32)c->ctx->host().N);
                bump(c, kRot);
                src = r;
            }
            auto md = std::make_shared<MaskData>();
            md->v.assign(masks + e * S, masks + (e + 1) * S);
            auto term = new_node(c, PNode::Comb, S, a.depth);
            term->in = {src};
            term->masks = {md};
            bump(c, kMultCP);
            if (!acc) {
                acc = term;
            } else {
                auto s = new_node(c, PNode::Comb, S, a.depth);
                s->in = {acc, term};
                s->masks = {nullptr, nullptr};
                bump(c, kAdd);
                acc = s;
            }
        }
        *out = make_handle(c, std::move(acc));
    });
}

int hgm_flush(hgm_ctx* c) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        // every node some caller still holds a pinned handle to, not yet computed
        std::vector<std::shared_ptr<SNode>> targets;
        {
            std::lock_guard<std::mutex> lk(c->mu);
            std::vector<std::weak_ptr<SNode>> keep;
            for (auto& w : c->pending) {
                auto p = w.lock();
                if (!p || p->buf) continue;
                if (p->pins.load() > 0) targets.push_back(p);
                else keep.push_back(w);  // unpinned: stays lazy (recomputed on demand)
            }
            c->pending.swap(keep);
        }
        if (targets.empty()) return;
        flush(c, targets);
        c->ctx->sync();
    });
}

int hgm_ct_export(hgm_ctx* c, const hgm_ct* ct, uint64_t* words) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        flush(c, {ct->node});
        c->ctx->sync();
        HGM_CUDA(cudaMemcpy(words, ct->node->buf->p, c->ctx->ct_words() * 8, cudaMemcpyDeviceToHost));
    });
}

int hgm_ct_import(hgm_ctx* c, const uint64_t* words, size_t S, size_t depth, hgm_ct** out) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        check_values(c, S);
        auto n = new_node(c, PNode::Input, S, depth);
        u64* p = c->ctx->alloc(c->ctx->ct_words());
        n->buf = std::make_shared<DevBuf>(c->ctx.get(), p);
        HGM_CUDA(cudaMemcpyAsync(p, words, c->ctx->ct_words() * 8, cudaMemcpyHostToDevice, c->ctx->stream()));
        c->ctx->sync();
        *out = make_handle(c, std::move(n));
    });
}

namespace {
struct WireHeader {
    char magic[4];
    uint32_t version;
    uint64_t keyset;
    uint32_t N, L, segment, depth, phase, reserved;
    uint64_t checksum;
};
static_assert(sizeof(WireHeader) == 48, "wire header layout");
uint64_t fnv1a(const void* p, size_t n, uint64_t h = 0xcbf29ce484222325ULL) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ULL;
    return h;
}
uint64_t keyset_fingerprint(const Context& ctx) {
    const auto& hp = ctx.host();
    uint64_t h = fnv1a(hp.primes.data(), hp.primes.size() * sizeof(u64));
    return fnv1a(&hp.seed, sizeof(hp.seed), h);
}
}  // namespace

size_t hgm_ct_wire_size(const hgm_ctx* c) { return sizeof(WireHeader) + c->ctx->ct_words() * 8; }

int hgm_ct_serialize(hgm_ctx* c, const hgm_ct* ct, void* buf, size_t cap) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        if (!ct || !buf) throw std::invalid_argument("null handle or buffer");
        const size_t W = c->ctx->ct_words();
        if (cap < sizeof(WireHeader) + W * 8) throw std::invalid_argument("buffer smaller than hgm_ct_wire_size()");
        uint64_t* words = reinterpret_cast<uint64_t*>(static_cast<char*>(buf) + sizeof(WireHeader));
        const int rc = hgm_ct_export(c, ct, words);
        if (rc != HGM_OK) throw std::runtime_error(g_err);
        WireHeader h{};
        std::memcpy(h.magic, "HGMC", 4);
        h.version = 1;
        h.keyset = keyset_fingerprint(*c->ctx);
        h.N = c->ctx->host().N;
        h.L = c->ctx->host().L;
        h.segment = (uint32_t)ct->node->S;
        h.depth = (uint32_t)ct->node->depth;
        h.phase = (uint32_t)ct->node->phase;
        h.checksum = fnv1a(words, W * 8);
        std::memcpy(buf, &h, sizeof(h));
    });
}

int hgm_ct_deserialize(hgm_ctx* c, const void* buf, size_t len, hgm_ct** out) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        if (!buf || !out) throw std::invalid_argument("null buffer or output");
        const size_t W = c->ctx->ct_words();
        if (len != sizeof(WireHeader) + W * 8) throw std::invalid_argument("wire size mismatch");
        WireHeader h;
        std::memcpy(&h, buf, sizeof(h));
        if (std::memcmp(h.magic, "HGMC", 4) != 0 || h.version != 1) throw std::invalid_argument("not a v1 HGMC ciphertext");
        if (h.keyset != keyset_fingerprint(*c->ctx) || h.N != c->ctx->host().N || h.L != c->ctx->host().L)
            throw std::invalid_argument("ciphertext from another parameter or key set");
        std::vector<uint64_t> words(W);
        std::memcpy(words.data(), static_cast<const char*>(buf) + sizeof(WireHeader), W * 8);
        if (fnv1a(words.data(), W * 8) != h.checksum) throw std::invalid_argument("ciphertext checksum mismatch");
        const auto& hp = c->ctx->host();
        for (size_t w = 0; w < W; ++w)
            if (words[w] >= hp.primes[(w / hp.N) % hp.L]) throw std::invalid_argument("non-canonical residue");
        if (h.segment == 0) throw hgm::DimensionError("empty ciphertext segment");
        check_values(c, h.segment);  // CapacityError beyond slot_count, as hgm_encrypt
        auto n = new_node(c, PNode::Input, h.segment, h.depth);
        n->phase = (int)h.phase;
        u64* p = c->ctx->alloc(W);
        n->buf = std::make_shared<DevBuf>(c->ctx.get(), p);
        HGM_CUDA(cudaMemcpyAsync(p, words.data(), W * 8, cudaMemcpyHostToDevice, c->ctx->stream()));
        c->ctx->sync();
        *out = make_handle(c, std::move(n));
    });
}

size_t hgm_ct_segment(const hgm_ct* ct) { return ct->node->S; }
size_t hgm_ct_depth(const hgm_ct* ct) { return ct->node->depth; }
int hgm_ct_phase(const hgm_ct* ct) { return ct->node->phase; }
hgm_ct* hgm_ct_retain(hgm_ct* ct) {
    ct->refs++;
    return ct;
}
int hgm_ct_set_pinned(hgm_ct* ct, int pinned) {
    if (!ct) return fail(HGM_EARG, "null handle");
    const bool p = pinned != 0;
    if (p != ct->pinned) {
        if (p)
            ct->node->pins++;
        else
            ct->node->pins--;
        ct->pinned = p;
    }
    return HGM_OK;
}

void hgm_ct_release(hgm_ct* ct) {
    if (!ct) return;
    if (--ct->refs == 0) {
        hgm_ctx* c = ct->owner;
        {
            DeviceScope dev(c);  // freeing the last reference to a node frees device memory
            if (ct->pinned) ct->node->pins--;
            c->live--;
            delete ct;
        }
        ctx_release(c);
    }
}

int hgm_stats(const hgm_ctx* c, uint64_t stats[12]) {
    auto* m = const_cast<hgm_ctx*>(c);
    std::lock_guard<std::mutex> lk(m->mu);
    for (int k = 0; k < 6; ++k) {
        stats[2 * k] = c->counts.c[k][0];
        stats[2 * k + 1] = c->counts.c[k][1];
    }
    return HGM_OK;
}
int hgm_reset_stats(hgm_ctx* c) {
    std::lock_guard<std::mutex> lk(c->mu);
    c->counts = Counts{};
    c->peak.store(c->live.load());
    return HGM_OK;
}
size_t hgm_peak_live(const hgm_ctx* c) { return c->peak.load(); }
int hgm_set_phase(hgm_ctx* c, int phase) {
    if (phase != 0 && phase != 1) return fail(HGM_EARG, "phase must be 0 (client) or 1 (cloud)");
    c->phase.store(phase);
    return HGM_OK;
}
int hgm_phase(const hgm_ctx* c) { return c->phase.load(); }

}  // extern "C"

namespace {

// share of free device memory a lockstep chunk may plan for (HGM_LOCKSTEP_FRAC)
double lockstep_fraction() {
    static const double f = [] {
        const char* e = std::getenv("HGM_LOCKSTEP_FRAC");
        const double v = e ? std::atof(e) : 0.45;
        return v > 0.05 && v < 0.95 ? v : 0.45;
    }();
    return f;
}

// Runs `count` instances of one compiled program in lockstep chunks: instance k
// reads A_k / B_k, encrypts with counters base(k) + s, and writes C_k (and its
// final ciphertext words when requested).
void run_instances(Context& ctx, const MatmulProgram& prog, size_t count,
                   const std::function<const i64*(size_t)>& a_of, const std::function<const i64*(size_t)>& b_of,
                   const std::function<u64(size_t)>& base_of, const std::function<i64*(size_t)>& c_of,
                   uint64_t* final_words) {
    const size_t W = ctx.ct_words();
    // instances per lockstep chunk: bounded by the rotated working set
    const size_t per_inst = (prog.sched.rot_count * ctx.ks_words() + (prog.sched.comb_count / 2 + 8) * W +
                             prog.sched.pending_count * ctx.pending_words()) * 8;
    size_t free_b = 0, total_b = 0;
    HGM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    size_t chunk = std::max<size_t>(1, (size_t)(lockstep_fraction() * (double)free_b) / per_inst);
    chunk = std::min<size_t>(chunk, 1024);
    // host packing of chunk i+1 and unpacking of chunk i-1 overlap chunk i's GPU work
    using Packed = std::vector<std::vector<std::vector<i64>>>;
    auto pack_chunk = [&](size_t c0) {
        const size_t K = std::min(chunk, count - c0);
        Packed p(K);
        parallel_for(K, [&](size_t k) { p[k] = prog.pack(a_of(c0 + k), b_of(c0 + k)); }, 4);
        return p;
    };
    std::future<Packed> next = std::async(std::launch::async, pack_chunk, (size_t)0);
    // Decrypted slots of chunk i land in pinned slot i % 2 asynchronously; the host
    // enqueues chunk i + 1 before waiting for them, so the GPU never idles at a
    // chunk boundary (the export path copies the final words synchronously).
    const size_t H = ctx.slots();
    struct Slot {
        u32* host = nullptr;
        cudaEvent_t ev = nullptr;
        std::future<void> unpacking;
    };
    Slot slot[2];
    for (int i = 0; i < 2; ++i) {
        slot[i].host = ctx.pinned_slot(i, std::max<size_t>(1, std::min(chunk, count) * H * sizeof(u32)));
        HGM_CUDA(cudaEventCreateWithFlags(&slot[i].ev, cudaEventDisableTiming));
    }
    auto finish = [&](Slot& sl, size_t c0, int K) {
        sl.unpacking = std::async(std::launch::async, [&prog, &c_of, &sl, c0, K, H, seg = prog.segment]() {
            HGM_CUDA(cudaEventSynchronize(sl.ev));
            parallel_for((size_t)K, [&](size_t k) {
                std::vector<i64> v(seg);
                const u32* src = sl.host + k * H;
                for (size_t j = 0; j < seg; ++j) v[j] = (i64)src[j];
                prog.unpack(v, c_of(c0 + k));
            }, 4);
        });
    };
    auto drain = [&]() {
        for (Slot& sl : slot)
            if (sl.unpacking.valid()) sl.unpacking.get();
    };
    // HGM_TRACE=1: per-chunk host timeline on stderr (where the end-to-end path waits)
    static const bool trace = [] {
        const char* e = std::getenv("HGM_TRACE");
        return e && e[0] == '1';
    }();
    const auto t_start = std::chrono::steady_clock::now();
    auto ms_since = [&]() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    };
    try {
        size_t i = 0;
        for (size_t c0 = 0; c0 < count; c0 += chunk, ++i) {
            const int K = (int)std::min(chunk, count - c0);
            const double tw0 = trace ? ms_since() : 0;
            Packed packed = next.get();
            if (trace) std::fprintf(stderr, "hgm_trace chunk %zu (K=%d): pack wait %.1f ms at %.1f\n", i, K,
                                    ms_since() - tw0, ms_since());
            if (c0 + chunk < count) next = std::async(std::launch::async, pack_chunk, c0 + chunk);
            ExecIO io;
            io.K = K;
            io.input = [](int, int) -> const u64* { return nullptr; };
            io.enc_values = [&](int s, int k) { return (const i64*)packed[k][s].data(); };
            io.enc_counter = [&](int s, int k) { return base_of(c0 + k) + (u64)s; };
            std::vector<u64*> res = execute(ctx, prog.sched, io);
            std::vector<const u64*> cts(K);
            std::vector<size_t> S(K, prog.segment);
            for (int k = 0; k < K; ++k) cts[k] = res[0] + (size_t)k * W;
            Slot& sl = slot[i % 2];
            if (sl.unpacking.valid()) sl.unpacking.get();  // chunk i - 2 is out of this slot
            ctx.decrypt_to(K, cts.data(), S.data(), sl.host);
            HGM_CUDA(cudaEventRecord(sl.ev, ctx.stream()));
            if (final_words) {  // stream-ordered (the library stream does not sync with the legacy one)
                HGM_CUDA(cudaMemcpyAsync(final_words + c0 * W, res[0], (size_t)K * W * 8, cudaMemcpyDeviceToHost,
                                         ctx.stream()));
                ctx.sync();
            }
            for (u64* r : res) ctx.release(r);
            finish(sl, c0, K);
            if (trace) std::fprintf(stderr, "hgm_trace chunk %zu enqueued at %.1f\n", i, ms_since());
        }
        drain();
        if (trace) std::fprintf(stderr, "hgm_trace drained at %.1f (chunk %zu instances)\n", ms_since(), chunk);
    } catch (...) {
        try { drain(); } catch (...) {}
        ctx.sync();
        for (Slot& sl : slot) cudaEventDestroy(sl.ev);
        throw;
    }
    ctx.sync();
    for (Slot& sl : slot) cudaEventDestroy(sl.ev);
}

void put_counts(const MatmulProgram& prog, uint64_t* stats) {
    if (!stats) return;
    for (int k = 0; k < 6; ++k) {
        stats[2 * k] = prog.counts.c[k][0];
        stats[2 * k + 1] = prog.counts.c[k][1];
    }
}

int matmul_batch_impl(hgm_ctx* c, int algo, int order, int flags, size_t m, size_t l, size_t n, size_t count,
                      const int64_t* A, const int64_t* B, int64_t* C, uint64_t counter0, uint64_t* stats,
                      uint64_t* final_words) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        if (order < -1 || order > 1) throw std::invalid_argument("order must be -1, 0 or 1");
        Context& ctx = *c->ctx;
        auto prog = get_matmul_program(algo, order, m, l, n, ctx.slots(), ctx.host().N, flags);
        put_counts(*prog, stats);
        if (count == 0) return;
        const u64 E = (u64)prog->n_enc;
        counter0 = resolve_counter0(c, counter0, count * E);
        run_instances(
            ctx, *prog, count, [&](size_t k) { return A + k * m * l; }, [&](size_t k) { return B + k * l * n; },
            [&](size_t k) { return counter0 + k * E; }, [&](size_t k) { return C + k * m * n; }, final_words);
    });
}

}  // namespace

extern "C" {

int hgm_blocked_mm(hgm_ctx* c, int algo, size_t m, size_t l, size_t n, const size_t* rows, size_t n_row,
                   const size_t* mids, size_t n_mid, const size_t* cols, size_t n_col, const int64_t* A,
                   const int64_t* B, int64_t* C, uint64_t counter0, int32_t* log) {
    return hgm_blocked_mm_ex(c, algo, m, l, n, rows, n_row, mids, n_mid, cols, n_col, A, B, C, counter0, 0, 0,
                             (size_t)-1, log, nullptr, nullptr, 0, nullptr, nullptr);
}

int hgm_blocked_mm_ex(hgm_ctx* c, int algo, size_t m, size_t l, size_t n, const size_t* rows, size_t n_row,
                      const size_t* mids, size_t n_mid, const size_t* cols, size_t n_col, const int64_t* A,
                      const int64_t* B, int64_t* C, uint64_t counter0, int flags, size_t out_first,
                      size_t out_count, int32_t* log, uint64_t* acc_words, int64_t* acc_meta, size_t acc_cap,
                      size_t* n_acc, size_t* n_decrypts) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        if (algo < 0 || algo > 2) throw hgm::DimensionError("unknown algorithm id");
        if (flags & ~(HGM_BLOCKED_ENCRYPTED_ACCUMULATION | HGM_BLOCKED_NO_DECRYPT))
            throw std::invalid_argument("unknown blocked_mm flag");
        const bool enc_acc = (flags & HGM_BLOCKED_ENCRYPTED_ACCUMULATION) != 0;
        const bool no_dec = (flags & HGM_BLOCKED_NO_DECRYPT) != 0;
        if (no_dec && !enc_acc) throw std::invalid_argument("HGM_BLOCKED_NO_DECRYPT needs encrypted accumulation");
        // BlockPlan::validate (algorithms.cpp:412-432)
        auto check = [](const size_t* p, size_t np, size_t total, const char* name) {
            if (np == 0) throw hgm::DimensionError(std::string("empty ") + name + " partition");
            size_t sum = 0;
            for (size_t i = 0; i < np; ++i) {
                if (p[i] == 0) throw hgm::DimensionError(std::string("zero-sized block in ") + name + " partition");
                sum += p[i];
            }
            if (sum != total)
                throw hgm::DimensionError(std::string(name) + " partition sums to " + std::to_string(sum) +
                                          ", expected " + std::to_string(total));
        };
        check(rows, n_row, m, "row");
        check(mids, n_mid, l, "mid");
        check(cols, n_col, n, "col");
        const size_t n_out = n_row * n_col;
        if (out_first > n_out) throw std::invalid_argument("output block range starts past the last block");
        out_count = std::min(out_count, n_out - out_first);
        if (!enc_acc && (out_first != 0 || out_count != n_out))
            throw std::invalid_argument("an output block range needs HGM_BLOCKED_ENCRYPTED_ACCUMULATION");
        Context& ctx = *c->ctx;
        const size_t slots = ctx.slots(), W = ctx.ct_words();
        auto offs = [](const size_t* p, size_t np) {
            std::vector<size_t> o(np + 1, 0);
            for (size_t i = 0; i < np; ++i) o[i + 1] = o[i] + p[i];
            return o;
        };
        const auto ro = offs(rows, n_row), mo = offs(mids, n_mid), co = offs(cols, n_col);
        struct Blk {
            size_t bi, bj, bk, mm, ll, nn;
            int used;
            bool fell;
            u64 base;
            std::vector<i64> a, b, cprod;
            std::shared_ptr<const MatmulProgram> prog;
            u64* ct = nullptr;  // encrypted accumulation: the product's ciphertext on the device
        };
        std::vector<Blk> blocks;
        u64 ctr = 0;  // relative counters over ALL blocks (a shard encrypts exactly as a full run)
        for (size_t bi = 0; bi < n_row; ++bi)
            for (size_t bj = 0; bj < n_col; ++bj)
                for (size_t bk = 0; bk < n_mid; ++bk) {  // the reference loop order (algorithms.cpp:472-492)
                    Blk k{bi, bj, bk, rows[bi], mids[bk], cols[bj], algo, false, 0, {}, {}, {}, nullptr, nullptr};
                    if (algo == 1 && !hgm::fits(1, k.mm, k.ll, k.nn, slots)) {
                        k.used = 0;  // duplicated working set outgrows the slots (algorithms.cpp:456-466)
                        k.fell = true;
                    }
                    k.prog = get_matmul_program(k.used, -1, k.mm, k.ll, k.nn, slots, ctx.host().N);
                    k.base = ctr;
                    ctr += (u64)k.prog->n_enc;
                    const size_t ob = bi * n_col + bj;
                    if (ob < out_first || ob >= out_first + out_count) {
                        blocks.push_back(std::move(k));  // kept for the log and the counters only
                        continue;
                    }
                    k.a.resize(k.mm * k.ll);
                    k.b.resize(k.ll * k.nn);
                    k.cprod.resize(k.mm * k.nn);
                    for (size_t r = 0; r < k.mm; ++r)
                        for (size_t q = 0; q < k.ll; ++q) k.a[r * k.ll + q] = A[(ro[bi] + r) * l + mo[bk] + q];
                    for (size_t r = 0; r < k.ll; ++r)
                        for (size_t q = 0; q < k.nn; ++q) k.b[r * k.nn + q] = B[(mo[bk] + r) * n + co[bj] + q];
                    blocks.push_back(std::move(k));
                }
        const u64 base = resolve_counter0(c, counter0, ctr);
        for (Blk& k : blocks) k.base += base;
        auto mine = [&](const Blk& k) {
            const size_t ob = k.bi * n_col + k.bj;
            return ob >= out_first && ob < out_first + out_count;
        };
        // one lockstep batch per distinct (algorithm, shape)
        std::map<std::tuple<int, size_t, size_t, size_t>, std::vector<size_t>> groups;
        for (size_t i = 0; i < blocks.size(); ++i)
            if (mine(blocks[i]))
                groups[std::make_tuple(blocks[i].used, blocks[i].mm, blocks[i].ll, blocks[i].nn)].push_back(i);
        std::vector<u64*> owned;  // device ciphertexts of the encrypted path
        size_t decrypts = 0;
        try {
            for (auto& kv : groups) {
                const auto& ids = kv.second;
                const Blk& f = blocks[ids[0]];
                const MatmulProgram& prog = *f.prog;
                if (!enc_acc) {
                    run_instances(
                        ctx, prog, ids.size(), [&](size_t k) { return (const i64*)blocks[ids[k]].a.data(); },
                        [&](size_t k) { return (const i64*)blocks[ids[k]].b.data(); },
                        [&](size_t k) { return blocks[ids[k]].base; },
                        [&](size_t k) { return blocks[ids[k]].cprod.data(); }, nullptr);
                    decrypts += ids.size();
                    continue;
                }
                // client encrypt + cloud program; the products stay on the device
                u64* out = ctx.alloc(ids.size() * W);
                owned.push_back(out);
                for (size_t c0 = 0; c0 < ids.size(); c0 += 256) {
                    const int K = (int)std::min<size_t>(256, ids.size() - c0);
                    std::vector<std::vector<std::vector<i64>>> packed(K);
                    parallel_for((size_t)K, [&](size_t k) {
                        const Blk& b = blocks[ids[c0 + k]];
                        packed[k] = prog.pack(b.a.data(), b.b.data());
                    }, 4);
                    ExecIO io;
                    io.K = K;
                    io.input = [](int, int) -> const u64* { return nullptr; };
                    io.enc_values = [&](int s, int k) { return (const i64*)packed[k][s].data(); };
                    io.enc_counter = [&](int s, int k) { return blocks[ids[c0 + k]].base + (u64)s; };
                    std::vector<u64*> res = execute(ctx, prog.sched, io);
                    HGM_CUDA(cudaMemcpyAsync(out + c0 * W, res[0], (size_t)K * W * 8, cudaMemcpyDeviceToDevice,
                                             ctx.stream()));
                    for (u64* r : res) ctx.release(r);
                    ctx.sync();  // `packed` is host staging
                }
                for (size_t k = 0; k < ids.size(); ++k) blocks[ids[k]].ct = out + k * W;
            }
            if (n_acc) *n_acc = 0;
            if (enc_acc) {
                // per output block and slot layout (working rows, cols, flatten order): sum the
                // block products' ciphertexts over the mid dimension on the GPU
                struct Cls {
                    size_t ob;
                    size_t rep;                 // index of the class's first block product
                    std::vector<size_t> terms;  // its block products, mid-dimension order
                };
                std::vector<Cls> classes;
                std::map<std::tuple<size_t, size_t, size_t, int>, size_t> cidx;
                for (size_t bidx = 0; bidx < blocks.size(); ++bidx) {
                    const Blk& k = blocks[bidx];
                    if (!mine(k)) continue;
                    const MatmulProgram& p = *k.prog;
                    const size_t rw = p.algo == Algo::Enhanced ? p.strat.rows_w : p.m;
                    const size_t cw = p.algo == Algo::Enhanced ? p.strat.cols_w : p.n;
                    const auto key = std::make_tuple(k.bi * n_col + k.bj, rw, cw, (int)p.order);
                    auto it = cidx.find(key);
                    if (it == cidx.end()) {
                        it = cidx.emplace(key, classes.size()).first;
                        classes.push_back(Cls{k.bi * n_col + k.bj, bidx, {}});
                    }
                    classes[it->second].terms.push_back(bidx);
                }
                u64* acc = ctx.alloc(std::max<size_t>(1, classes.size()) * W);
                owned.push_back(acc);
                size_t depth = 0;
                for (const Cls& cl : classes) depth = std::max(depth, cl.terms.size());
                std::vector<const u64*> sa, sb;
                std::vector<u64*> so;
                for (size_t i = 0; i < classes.size(); ++i) {  // acc = term 0 + term 1
                    const auto& t = classes[i].terms;
                    if (t.size() == 1) {
                        HGM_CUDA(cudaMemcpyAsync(acc + i * W, blocks[t[0]].ct, W * 8, cudaMemcpyDeviceToDevice,
                                                 ctx.stream()));
                    } else {
                        sa.push_back(blocks[t[0]].ct);
                        sb.push_back(blocks[t[1]].ct);
                        so.push_back(acc + i * W);
                    }
                }
                ctx.add((int)so.size(), sa.data(), sb.data(), so.data());
                for (size_t d = 2; d < depth; ++d) {  // acc += term d, one launch per depth level
                    sa.clear();
                    sb.clear();
                    so.clear();
                    for (size_t i = 0; i < classes.size(); ++i)
                        if (classes[i].terms.size() > d) {
                            sa.push_back(acc + i * W);
                            sb.push_back(blocks[classes[i].terms[d]].ct);
                            so.push_back(acc + i * W);
                        }
                    ctx.add((int)so.size(), sa.data(), sb.data(), so.data());
                }
                // one decrypt per accumulated class (the reference: one per block product)
                std::vector<const u64*> cts(classes.size());
                std::vector<size_t> S(classes.size());
                std::vector<std::vector<i64>> slotv(classes.size());
                std::vector<i64*> outp(classes.size());
                for (size_t i = 0; i < classes.size(); ++i) {
                    cts[i] = acc + i * W;
                    S[i] = blocks[classes[i].rep].prog->segment;
                    slotv[i].resize(S[i]);
                    outp[i] = slotv[i].data();
                }
                if (!classes.empty() && !no_dec) ctx.decrypt((int)classes.size(), cts.data(), S.data(), outp.data());
                decrypts = no_dec ? 0 : classes.size();
                // the class's decrypted sum lands in its first product's slot of C; the
                // other products of the class contribute nothing more
                for (const Cls& cl : classes) {
                    if (no_dec) {
                        for (size_t t : cl.terms) std::fill(blocks[t].cprod.begin(), blocks[t].cprod.end(), 0);
                        continue;
                    }
                    Blk& r = blocks[cl.rep];
                    r.prog->unpack(slotv[&cl - classes.data()], r.cprod.data());
                    for (size_t t : cl.terms)
                        if (t != cl.rep) std::fill(blocks[t].cprod.begin(), blocks[t].cprod.end(), 0);
                }
                if (acc_words || acc_meta || n_acc) {
                    if (classes.size() > acc_cap && (acc_words || acc_meta))
                        throw std::invalid_argument("accumulated ciphertexts (" + std::to_string(classes.size()) +
                                                    ") exceed acc_cap");
                    for (size_t i = 0; i < classes.size() && (acc_words || acc_meta); ++i) {
                        const Blk& r = blocks[classes[i].rep];
                        if (acc_words)
                            HGM_CUDA(cudaMemcpyAsync(acc_words + i * W, acc + i * W, W * 8, cudaMemcpyDeviceToHost,
                                                     ctx.stream()));
                        if (acc_meta) {
                            int64_t* mt = acc_meta + 8 * i;
                            mt[0] = (int64_t)classes[i].ob;
                            mt[1] = r.used;
                            mt[2] = (int64_t)r.mm;
                            mt[3] = (int64_t)r.ll;
                            mt[4] = (int64_t)r.nn;
                            mt[5] = (int64_t)r.prog->order;
                            mt[6] = (int64_t)classes[i].terms.size();
                            mt[7] = (int64_t)r.prog->segment;
                        }
                    }
                    if (n_acc) *n_acc = classes.size();
                    ctx.sync();
                }
            }
        } catch (...) {
            ctx.sync();
            for (u64* p : owned) ctx.release(p);
            throw;
        }
        for (u64* p : owned) ctx.release(p);
        ctx.sync();
        if (n_decrypts) *n_decrypts = decrypts;
        for (size_t ob = out_first; ob < out_first + out_count; ++ob) {  // the blocks this call computes
            const size_t bi = ob / n_col, bj = ob % n_col;
            for (size_t r = 0; r < rows[bi]; ++r)
                std::fill(C + (ro[bi] + r) * n + co[bj], C + (ro[bi] + r) * n + co[bj] + cols[bj], 0);
        }
        for (size_t i = 0; i < blocks.size(); ++i) {
            const Blk& k = blocks[i];
            if (log) {
                log[4 * i] = k.used;
                log[4 * i + 1] = k.fell ? 1 : 0;
                log[4 * i + 2] = (int32_t)k.mm;
                log[4 * i + 3] = (int32_t)k.ll;
            }
            if (!mine(k)) continue;
            for (size_t r = 0; r < k.mm; ++r)
                for (size_t q = 0; q < k.nn; ++q) {
                    i64& dst = C[(ro[k.bi] + r) * n + co[k.bj] + q];
                    dst = (dst + k.cprod[r * k.nn + q]) % (i64)kT;
                }
        }
    });
}

}  // extern "C"

struct hgm_batch {
    hgm_ctx* owner = nullptr;  // holds a context reference once fully built
    std::shared_ptr<const MatmulProgram> prog;
    size_t count = 0;
    u64* in = nullptr;   // [count][n_enc][W]
    u64* out = nullptr;  // [count][W]
    Context* dctx = nullptr;
    ~hgm_batch() {
        if (dctx) {
            dctx->release(in);
            dctx->release(out);
        }
    }
};

namespace hgm {

Context& session_context(hgm_ctx* c) { return *c->ctx; }
int session_device(const hgm_ctx* c) { return c->device; }
std::recursive_mutex& session_exec_mutex(hgm_ctx* c) { return c->exec_mu; }
void session_retain(hgm_ctx* c) { ctx_retain(c); }
void session_release(hgm_ctx* c) { ctx_release(c); }
hgm_ctx* batch_session(hgm_batch* b) { return b ? b->owner : nullptr; }
const u64* batch_results(const hgm_batch* b, size_t* count) {
    if (count) *count = b ? b->count : 0;
    return b ? b->out : nullptr;
}
int set_error(int code, const std::string& msg) { return fail(code, msg); }
bool is_device_pointer(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // unregistered host memory on older runtimes
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace hgm

namespace {

size_t lockstep_chunk(Context& ctx, const MatmulProgram& prog) {
    const size_t W = ctx.ct_words();
    // stored rotation accumulators; sums computed straight from the ModUp digits
    // (Schedule::ks_terms) store their own accumulator instead
    const size_t accs = prog.cloud_sched.stored_rot_count + prog.cloud_sched.ks_comb_count;
    const size_t per_inst = (accs * ctx.ks_words() + (prog.cloud_sched.comb_count / 2 + 8) * W +
                             prog.cloud_sched.pending_count * ctx.pending_words()) * 8;
    size_t free_b = 0, total_b = 0;
    HGM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    size_t chunk = std::max<size_t>(1, (size_t)(lockstep_fraction() * (double)free_b) / per_inst);
    return std::min<size_t>(chunk, 1024);
}

}  // namespace

extern "C" {

int hgm_batch_encrypt(hgm_ctx* c, int algo, int order, int flags, size_t m, size_t l, size_t n, size_t count,
                      const int64_t* A, const int64_t* B, uint64_t counter0, hgm_batch** out) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        if (order < -1 || order > 1) throw std::invalid_argument("order must be -1, 0 or 1");
        Context& ctx = *c->ctx;
        auto b = std::make_unique<hgm_batch>();
        b->prog = get_matmul_program(algo, order, m, l, n, ctx.slots(), ctx.host().N, flags);
        b->count = count;
        const size_t W = ctx.ct_words(), E = b->prog->n_enc;
        counter0 = resolve_counter0(c, counter0, count * E);
        b->dctx = &ctx;
        b->in = ctx.alloc(std::max<size_t>(1, count * E) * W);
        b->out = ctx.alloc(std::max<size_t>(1, count) * W);
        const size_t chunk = 1024;
        for (size_t c0 = 0; c0 < count; c0 += chunk) {
            const size_t K = std::min(chunk, count - c0);
            std::vector<std::vector<std::vector<i64>>> packed(K);
            std::vector<const i64*> vals;
            std::vector<size_t> S;
            std::vector<u64> ctr;
            std::vector<u64*> dst;
            parallel_for(K, [&](size_t k) { packed[k] = b->prog->pack(A + (c0 + k) * m * l, B + (c0 + k) * l * n); }, 4);
            for (size_t k = 0; k < K; ++k) {
                for (size_t s = 0; s < E; ++s) {
                    vals.push_back(packed[k][s].data());
                    S.push_back(b->prog->segment);
                    ctr.push_back(counter0 + (c0 + k) * E + s);
                    dst.push_back(b->in + ((c0 + k) * E + s) * W);
                }
            }
            ctx.encrypt((int)vals.size(), vals.data(), S.data(), ctr.data(), dst.data());
            ctx.sync();  // `packed` is host staging for this chunk
        }
        b->owner = c;
        ctx_retain(c);
        *out = b.release();
    });
}

int hgm_batch_cloud(hgm_ctx* c, hgm_batch* b, float* device_ms) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        Context& ctx = *c->ctx;
        const MatmulProgram& prog = *b->prog;
        const size_t W = ctx.ct_words(), E = prog.n_enc;
        const size_t chunk = lockstep_chunk(ctx, prog);
        cudaEvent_t e0, e1;
        HGM_CUDA(cudaEventCreate(&e0));
        HGM_CUDA(cudaEventCreate(&e1));
        HGM_CUDA(cudaEventRecord(e0, ctx.stream()));
        for (size_t c0 = 0; c0 < b->count; c0 += chunk) {
            const int K = (int)std::min(chunk, b->count - c0);
            ExecIO io;
            io.K = K;
            io.input = [&](int s, int k) -> const u64* { return b->in + ((c0 + k) * E + s) * W; };
            io.enc_values = [](int, int) -> const i64* { throw std::logic_error("cloud program encrypts"); };
            io.enc_counter = [](int, int) -> u64 { return 0; };
            std::vector<u64*> res = execute(ctx, prog.cloud_sched, io);
            HGM_CUDA(cudaMemcpyAsync(b->out + c0 * W, res[0], (size_t)K * W * 8, cudaMemcpyDeviceToDevice,
                                     ctx.stream()));
            for (u64* r : res) ctx.release(r);
        }
        HGM_CUDA(cudaEventRecord(e1, ctx.stream()));
        HGM_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        HGM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (device_ms) *device_ms = ms;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

uint64_t* hgm_batch_output(hgm_batch* b, size_t i) {
    if (!b || i >= b->count) return nullptr;
    return b->out + i * b->owner->ctx->ct_words();
}

int hgm_batch_decrypt_words(hgm_ctx* c, const uint64_t* dev_words, size_t count, size_t S, int64_t* out) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        Context& ctx = *c->ctx;
        if (S == 0 || S > ctx.slots()) throw hgm::DimensionError("bad segment");
        const size_t W = ctx.ct_words();
        const size_t chunk = 1024;
        for (size_t c0 = 0; c0 < count; c0 += chunk) {
            const size_t K = std::min(chunk, count - c0);
            std::vector<const u64*> cts(K);
            std::vector<size_t> Sv(K, S);
            std::vector<i64*> outp(K);
            for (size_t k = 0; k < K; ++k) {
                cts[k] = dev_words + (c0 + k) * W;
                outp[k] = out + (c0 + k) * S;
            }
            ctx.decrypt((int)K, cts.data(), Sv.data(), outp.data());
        }
    });
}

int hgm_decrypt_products(hgm_ctx* c, int algo, int order, int flags, size_t m, size_t l, size_t n,
                         const uint64_t* dev_words, size_t count, int64_t* C) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        if (order < -1 || order > 1) throw std::invalid_argument("order must be -1, 0 or 1");
        auto prog = get_matmul_program(algo, order, m, l, n, c->ctx->slots(), c->ctx->host().N, flags);
        std::vector<i64> slots(count * prog->segment);
        // host words (e.g. a host gather) are staged through the device
        const u64* words = dev_words;
        u64* staged = nullptr;
        if (count && !is_device_pointer(dev_words)) {
            staged = c->ctx->alloc(count * c->ctx->ct_words());
            HGM_CUDA(cudaMemcpyAsync(staged, dev_words, count * c->ctx->ct_words() * 8, cudaMemcpyHostToDevice,
                                     c->ctx->stream()));
            words = staged;
        }
        const int rc = hgm_batch_decrypt_words(c, words, count, prog->segment, slots.data());
        if (staged) {
            c->ctx->release(staged);
            c->ctx->sync();
        }
        if (rc != HGM_OK) throw std::runtime_error(g_err);
        parallel_for(count, [&](size_t k) {
            std::vector<i64> v(slots.begin() + k * prog->segment, slots.begin() + (k + 1) * prog->segment);
            prog->unpack(v, C + k * m * n);
        });
    });
}

int hgm_batch_decrypt(hgm_ctx* c, hgm_batch* b, int64_t* C) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        const MatmulProgram& prog = *b->prog;
        std::vector<i64> slots(b->count * prog.segment);
        const int rc = hgm_batch_decrypt_words(c, b->out, b->count, prog.segment, slots.data());
        if (rc != HGM_OK) throw std::runtime_error(g_err);
        parallel_for(b->count, [&](size_t k) {
            std::vector<i64> v(slots.begin() + k * prog.segment, slots.begin() + (k + 1) * prog.segment);
            prog.unpack(v, C + k * prog.m * prog.n);
        });
    });
}

void hgm_batch_free(hgm_batch* b) {
    if (!b) return;
    hgm_ctx* c = b->owner;
    {
        std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);
        DeviceScope dev(c);
        try {
            delete b;  // stream-ordered frees
            c->ctx->sync();
        } catch (const std::exception& e) {
            g_err = e.what();
        }
    }
    ctx_release(c);
}

int hgm_program_info(int algo, int order, int flags, size_t m, size_t l, size_t n, size_t slots, uint32_t N,
                     uint64_t* stats, uint64_t* facts) {
    return guarded([&] {
        auto p = get_matmul_program(algo, order, m, l, n, slots, N, flags);
        if (stats)
            for (int k = 0; k < 6; ++k) {
                stats[2 * k] = p->counts.c[k][0];
                stats[2 * k + 1] = p->counts.c[k][1];
            }
        if (facts) {
            facts[0] = p->segment;
            facts[1] = p->n_enc;
            facts[2] = p->cloud_sched.rot_count;
            facts[3] = p->cloud_sched.comb_count;
            facts[4] = p->cloud_sched.mult_count;
            facts[5] = p->cloud_sched.levels.size();
            facts[6] = (u64)p->order;
            facts[7] = p->cloud_sched.moddown_count;
            facts[8] = p->cloud_sched.rescale_count;
            // slot layout of the decrypted product: working rows, cols (flat_index with facts[6])
            facts[9] = p->algo == Algo::Enhanced ? p->strat.rows_w : p->m;
            facts[10] = p->algo == Algo::Enhanced ? p->strat.cols_w : p->n;
        }
    });
}

long hgm_program_keys(int algo, int order, int flags, size_t m, size_t l, size_t n, size_t slots, uint32_t N,
                      uint32_t* elements, size_t cap) {
    long result = 0;
    const int rc = guarded([&] {
        auto p = get_matmul_program(algo, order, m, l, n, slots, N, flags);
        std::vector<u32> els;
        bool relin = false;
        for (const auto& nd : p->sched.prog.nodes) {
            if (nd.kind == PNode::Rot && nd.g != 1) els.push_back(nd.g);
            if (nd.kind == PNode::Mult) relin = true;
        }
        std::sort(els.begin(), els.end());
        els.erase(std::unique(els.begin(), els.end()), els.end());
        if (relin) els.insert(els.begin(), 0u);
        result = (long)els.size();
        if (elements) std::copy(els.begin(), els.begin() + std::min(cap, els.size()), elements);
    });
    return rc == HGM_OK ? result : -rc;
}

long hgm_program_stream(int algo, int order, int flags, size_t m, size_t l, size_t n, size_t slots, uint32_t N,
                        int64_t* hdr, size_t hdr_cap, int64_t* data, size_t data_cap, size_t* data_len) {
    long result = 0;
    const int rc = guarded([&] {
        auto p = get_matmul_program(algo, order, m, l, n, slots, N, flags);
        size_t dl = 0;
        for (const auto& mk : p->stream_masks) dl += mk->v.size();
        if (data_len) *data_len = dl;
        result = (long)p->stream.size();
        if (!hdr) return;
        if (hdr_cap < p->stream.size() * 3 || data_cap < dl) throw std::invalid_argument("buffers too small");
        size_t off = 0, mi = 0;
        for (size_t i = 0; i < p->stream.size(); ++i) {
            hdr[3 * i] = p->stream[i].first;
            hdr[3 * i + 1] = p->stream[i].second;
            hdr[3 * i + 2] = 0;
            if (p->stream[i].first == 4) {
                const auto& v = p->stream_masks[mi++]->v;
                hdr[3 * i + 2] = (int64_t)v.size();
                std::copy(v.begin(), v.end(), data + off);
                off += v.size();
            }
        }
    });
    return rc == HGM_OK ? result : -rc;
}

long hgm_plan_info(int kind, size_t k, size_t a, size_t b, size_t c, int order, size_t segment,
                   int64_t* offsets, uint64_t* weights, size_t cap) {
    long result = 0;
    const int rc = guarded([&] {
        if (order != 0 && order != 1) throw std::invalid_argument("order must be 0 or 1");
        const Order o = (Order)order;
        std::shared_ptr<const Plan> p;
        switch (kind) {
            case 0: p = eps_plan_embedded(k, a, b, c, o, segment); break;
            case 1: p = omega_plan_embedded(k, a, b, c, o, segment); break;
            case 4: p = shaped_eps_plan(k, a, b, c, o, segment); break;
            case 5: p = shaped_omega_plan(k, a, b, c, o, segment); break;
            default: throw std::invalid_argument("unknown plan kind");
        }
        result = (long)p->entries.size();
        for (size_t i = 0; i < p->entries.size() && i < cap; ++i) {
            offsets[i] = p->entries[i].offset;
            u64 w = 0;
            for (i64 v : p->entries[i].mask->v) w += v != 0;
            weights[i] = w;
        }
    });
    return rc == HGM_OK ? result : -rc;
}

int hgm_matmul_batch(hgm_ctx* c, int algo, int order, int flags, size_t m, size_t l, size_t n, size_t count,
                     const int64_t* A, const int64_t* B, int64_t* C, uint64_t counter0, uint64_t* stats) {
    return matmul_batch_impl(c, algo, order, flags, m, l, n, count, A, B, C, counter0, stats, nullptr);
}
int hgm_matmul_batch_export(hgm_ctx* c, int algo, int order, int flags, size_t m, size_t l, size_t n,
                            size_t count, const int64_t* A, const int64_t* B, int64_t* C, uint64_t counter0,
                            uint64_t* final_words) {
    return matmul_batch_impl(c, algo, order, flags, m, l, n, count, A, B, C, counter0, nullptr, final_words);
}

int hgm_bench_ntt(hgm_ctx* c, int forward, size_t limbs, int iters, float* ms) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        Context& ctx = *c->ctx;
        const u32 N = ctx.host().N, L = ctx.host().L;
        u64* buf = ctx.alloc(limbs * N);
        ctx.fill_residues(buf, (u32)limbs, 0, L, 0x6e7474);  // canonical operands, not zeros
        NttJobs j = jobs_contig(buf, (u32)limbs, 0, L);
        ctx.ntt(forward != 0, j);  // warm-up
        cudaEvent_t e0, e1;
        HGM_CUDA(cudaEventCreate(&e0));
        HGM_CUDA(cudaEventCreate(&e1));
        HGM_CUDA(cudaEventRecord(e0, ctx.stream()));
        for (int i = 0; i < iters; ++i) ctx.ntt(forward != 0, j);
        HGM_CUDA(cudaEventRecord(e1, ctx.stream()));
        HGM_CUDA(cudaEventSynchronize(e1));
        float t = 0;
        HGM_CUDA(cudaEventElapsedTime(&t, e0, e1));
        *ms = t / iters;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        ctx.release(buf);
        ctx.sync();
    });
}

int hgm_test_chacha(const uint32_t* key, uint64_t nonce, uint64_t counter, int rounds, uint32_t* out) {
    return guarded([&] {
        if (!key || !out || rounds <= 0 || rounds % 2) throw std::invalid_argument("bad ChaCha test arguments");
        chacha_block(key, nonce, counter, rounds, out);
    });
}

int hgm_bench_keyswitch(hgm_ctx* c, size_t items, int iters, float* ms) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        if (items == 0 || iters <= 0 || !ms) throw std::invalid_argument("bad benchmark arguments");
        *ms = c->ctx->bench_inner_product((int)items, iters);
    });
}

int hgm_bench_keyswitch_plan(hgm_ctx* c, size_t instances, size_t sums, size_t terms, size_t tile, int iters,
                             float* ms) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        if (instances == 0 || sums == 0 || terms == 0 || tile == 0 || iters <= 0 || !ms)
            throw std::invalid_argument("bad benchmark arguments");
        *ms = c->ctx->bench_plan((int)instances, (int)sums, (int)terms, (int)tile, iters);
    });
}

int hgm_device_sync(hgm_ctx* c) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] { c->ctx->sync(); });
}

int hgm_test_ntt(hgm_ctx* c, int forward, int prime, uint64_t* data, size_t count) {
    std::lock_guard<std::recursive_mutex> exec_lk(c->exec_mu);  // one device user at a time
    DeviceScope dev(c);
    return guarded([&] {
        Context& ctx = *c->ctx;
        const u32 N = ctx.host().N;
        const int p = prime < 0 ? kTIndex : prime;
        if (prime >= (int)ctx.host().primes.size()) throw std::invalid_argument("prime index out of range");
        u64* buf = ctx.alloc(count * N);
        HGM_CUDA(cudaMemcpyAsync(buf, data, count * N * 8, cudaMemcpyHostToDevice, ctx.stream()));
        ctx.ntt(forward != 0, jobs_contig(buf, (u32)count, (u32)p, 1));
        HGM_CUDA(cudaMemcpyAsync(data, buf, count * N * 8, cudaMemcpyDeviceToHost, ctx.stream()));
        ctx.release(buf);
        ctx.sync();
    });
}

uint64_t hgm_launch_count(const hgm_ctx* c) { return c->ctx->launches(); }

}  // extern "C"
