// engine.cpp -- program optimisation and level-batched execution.
#include "engine.hpp"

#include <algorithm>
#include <map>
#include <stdexcept>
#include <unordered_map>

namespace hgm {

int Program::add_input(size_t S) {
    PNode n;
    n.kind = PNode::Input;
    n.slot = n_inputs++;
    n.S = S;
    nodes.push_back(std::move(n));
    return (int)nodes.size() - 1;
}
int Program::add_enc(size_t S) {
    PNode n;
    n.kind = PNode::Enc;
    n.slot = n_enc++;
    n.S = S;
    nodes.push_back(std::move(n));
    return (int)nodes.size() - 1;
}
int Program::add_rot(int src, u32 g) {
    PNode n;
    n.kind = PNode::Rot;
    n.in = {src};
    n.g = g;
    n.S = nodes.at(src).S;
    nodes.push_back(std::move(n));
    return (int)nodes.size() - 1;
}
int Program::add_comb(std::vector<int> in, std::vector<MaskRef> masks) {
    if (in.empty() || in.size() != masks.size()) throw std::logic_error("bad masked sum");
    PNode n;
    n.kind = PNode::Comb;
    n.S = nodes.at(in[0]).S;
    n.in = std::move(in);
    n.masks = std::move(masks);
    nodes.push_back(std::move(n));
    return (int)nodes.size() - 1;
}
int Program::add_mult(int a, int b) {
    PNode n;
    n.kind = PNode::Mult;
    n.in = {a, b};
    n.S = nodes.at(a).S;
    nodes.push_back(std::move(n));
    return (int)nodes.size() - 1;
}

namespace {

std::vector<char> liveness(const Program& q) {
    std::vector<char> live(q.nodes.size(), 0);
    std::vector<int> stack(q.outputs.begin(), q.outputs.end());
    while (!stack.empty()) {
        const int x = stack.back();
        stack.pop_back();
        if (live[x]) continue;
        live[x] = 1;
        for (int y : q.nodes[x].in) stack.push_back(y);
    }
    return live;
}

thread_local ExecCounters g_counters;

}  // namespace

ExecCounters last_exec_counters() { return g_counters; }

Schedule optimise(const Program& p) {
    Schedule s;
    Program& q = s.prog;
    q = p;
    const size_t n = q.nodes.size();
    // 1. rotation aliases: identity rotations and duplicate (src, g) pairs
    std::vector<int> alias(n);
    for (size_t i = 0; i < n; ++i) alias[i] = (int)i;
    auto root = [&](int x) {
        while (alias[x] != x) x = alias[x];
        return x;
    };
    std::map<std::pair<int, u32>, int> rots;
    for (size_t i = 0; i < n; ++i) {
        PNode& nd = q.nodes[i];
        for (int& x : nd.in) x = root(x);
        if (nd.kind == PNode::Rot) {
            if (nd.g == 1) {
                alias[i] = nd.in[0];
            } else {
                auto key = std::make_pair(nd.in[0], nd.g);
                auto it = rots.find(key);
                if (it != rots.end())
                    alias[i] = it->second;
                else
                    rots.emplace(key, (int)i);
            }
        }
    }
    for (int& o : q.outputs) o = root(o);
    // 2. uses among live nodes
    std::vector<char> live = liveness(q);
    s.is_output.assign(n, 0);
    for (int o : q.outputs) s.is_output[o] = 1;
    std::vector<int> uses(n, 0);
    for (size_t i = 0; i < n; ++i)
        if (live[i])
            for (int x : q.nodes[i].in) ++uses[x];
    // 3. fold single-use plain addends that are masked sums into their consumer
    for (size_t i = 0; i < n; ++i) {
        PNode& nd = q.nodes[i];
        if (!live[i] || nd.kind != PNode::Comb) continue;
        std::vector<int> in;
        std::vector<MaskRef> masks;
        for (size_t t = 0; t < nd.in.size(); ++t) {
            const int x = nd.in[t];
            const PNode& child = q.nodes[x];
            if (!nd.masks[t] && child.kind == PNode::Comb && uses[x] == 1 && !s.is_output[x]) {
                in.insert(in.end(), child.in.begin(), child.in.end());
                masks.insert(masks.end(), child.masks.begin(), child.masks.end());
            } else {
                in.push_back(x);
                masks.push_back(nd.masks[t]);
            }
        }
        nd.in = std::move(in);
        nd.masks = std::move(masks);
    }
    live = liveness(q);
    // 4. levels
    std::vector<int> level(n, -1);
    int max_level = -1;
    for (size_t i = 0; i < n; ++i) {
        if (!live[i]) continue;
        const PNode& nd = q.nodes[i];
        if (nd.kind == PNode::Input) continue;
        int lv = 0;
        if (nd.kind != PNode::Enc)
            for (int x : nd.in) lv = std::max(lv, level[x] + 1);
        level[i] = lv;
        max_level = std::max(max_level, lv);
    }
    s.levels.assign(max_level + 1, {});
    s.last_use_level.assign(n, -1);
    for (size_t i = 0; i < n; ++i) {
        if (level[i] < 0) continue;
        s.levels[level[i]].push_back((int)i);
        const PNode& nd = q.nodes[i];
        if (nd.kind == PNode::Rot) ++s.rot_count;
        if (nd.kind == PNode::Comb) ++s.comb_count;
        if (nd.kind == PNode::Mult) ++s.mult_count;
        for (int x : nd.in) s.last_use_level[x] = std::max(s.last_use_level[x], level[i]);
    }
    return s;
}

std::vector<u64*> execute(Context& ctx, const Schedule& sch, const ExecIO& io) {
    const Program& P = sch.prog;
    const int K = io.K;
    const size_t W = ctx.ct_words(), MW = ctx.modup_words();
    g_counters = ExecCounters{};
    g_counters.levels = sch.levels.size();
    std::vector<u64*> base(P.nodes.size(), nullptr);
    auto ptr = [&](int node, int k) -> const u64* {
        const PNode& nd = P.nodes[node];
        if (nd.kind == PNode::Input) return io.input(nd.slot, k);
        return base[node] + (size_t)k * W;
    };
    std::unordered_map<const MaskData*, const u64*> mask_dev;
    auto resolve = [&](const MaskRef& m) -> const u64* {
        if (!m) return nullptr;
        auto it = mask_dev.find(m.get());
        if (it != mask_dev.end()) return it->second;
        const u64* d = ctx.mask_plain(m->v.data(), m->v.size(), m->stable ? m->id : 0);
        mask_dev.emplace(m.get(), d);
        return d;
    };
    for (size_t lv = 0; lv < sch.levels.size(); ++lv) {
        const std::vector<int>& nodes = sch.levels[lv];
        std::vector<int> enc, rot, comb, mult;
        for (int x : nodes) {
            base[x] = ctx.alloc((size_t)K * W);
            switch (P.nodes[x].kind) {
                case PNode::Enc: enc.push_back(x); break;
                case PNode::Rot: rot.push_back(x); break;
                case PNode::Comb: comb.push_back(x); break;
                case PNode::Mult: mult.push_back(x); break;
                default: throw std::logic_error("input node scheduled");
            }
        }
        if (!enc.empty()) {
            std::vector<const i64*> vals;
            std::vector<size_t> S;
            std::vector<u64> ctr;
            std::vector<u64*> out;
            for (int x : enc)
                for (int k = 0; k < K; ++k) {
                    vals.push_back(io.enc_values(P.nodes[x].slot, k));
                    S.push_back(P.nodes[x].S);
                    ctr.push_back(io.enc_counter(P.nodes[x].slot, k));
                    out.push_back(base[x] + (size_t)k * W);
                }
            ctx.encrypt((int)vals.size(), vals.data(), S.data(), ctr.data(), out.data());
            g_counters.enc_items += vals.size();
        }
        if (!rot.empty()) {
            // hoisting: one ModUp per distinct source (and instance)
            std::vector<int> srcs;
            for (int x : rot) srcs.push_back(P.nodes[x].in[0]);
            std::sort(srcs.begin(), srcs.end());
            srcs.erase(std::unique(srcs.begin(), srcs.end()), srcs.end());
            u64* mbuf = ctx.alloc(srcs.size() * (size_t)K * MW);
            std::vector<const u64*> mct;
            std::vector<u64*> mout;
            for (size_t si = 0; si < srcs.size(); ++si)
                for (int k = 0; k < K; ++k) {
                    mct.push_back(ptr(srcs[si], k));
                    mout.push_back(mbuf + (si * K + k) * MW);
                }
            ctx.modup((int)mct.size(), mct.data(), mout.data());
            g_counters.modup_items += mct.size();
            // rotations grouped by Galois element: one key serves the group
            std::vector<int> order(rot);
            std::stable_sort(order.begin(), order.end(),
                             [&](int a, int b) { return P.nodes[a].g < P.nodes[b].g; });
            // items tiled over instances: within a tile of kRotTile instances the
            // rotations run key by key, so the tile's ModUp digits stay in L2 while
            // every Galois key streams past them once (instead of re-reading each
            // instance's digits from HBM for every one of its rotations)
            constexpr int kRotTile = 8;
            std::vector<const u64*> mu, cts;
            std::vector<u32> gs;
            std::vector<u64*> out;
            for (int k0 = 0; k0 < K; k0 += kRotTile)
                for (int x : order) {
                    const int src = P.nodes[x].in[0];
                    const size_t si = std::lower_bound(srcs.begin(), srcs.end(), src) - srcs.begin();
                    for (int k = k0; k < std::min(K, k0 + kRotTile); ++k) {
                        mu.push_back(mbuf + (si * K + k) * MW);
                        cts.push_back(ptr(src, k));
                        gs.push_back(P.nodes[x].g);
                        out.push_back(base[x] + (size_t)k * W);
                    }
                }
            ctx.rotate((int)mu.size(), mu.data(), cts.data(), gs.data(), out.data());
            g_counters.rot_items += mu.size();
            ctx.release(mbuf);
        }
        if (!comb.empty()) {
            std::vector<u32> off{0};
            std::vector<const u64*> in, masks;
            std::vector<u64*> out;
            for (int x : comb) {
                const PNode& nd = P.nodes[x];
                std::vector<const u64*> md(nd.in.size());
                for (size_t t = 0; t < nd.in.size(); ++t) md[t] = resolve(nd.masks[t]);
                for (int k = 0; k < K; ++k) {
                    for (size_t t = 0; t < nd.in.size(); ++t) {
                        in.push_back(ptr(nd.in[t], k));
                        masks.push_back(md[t]);
                    }
                    off.push_back((u32)in.size());
                    out.push_back(base[x] + (size_t)k * W);
                }
            }
            ctx.lincomb((int)out.size(), off.data(), in.data(), masks.data(), out.data());
            g_counters.comb_items += out.size();
        }
        if (!mult.empty()) {
            std::vector<const u64*> a, b;
            std::vector<u64*> out;
            for (int x : mult)
                for (int k = 0; k < K; ++k) {
                    a.push_back(ptr(P.nodes[x].in[0], k));
                    b.push_back(ptr(P.nodes[x].in[1], k));
                    out.push_back(base[x] + (size_t)k * W);
                }
            ctx.mult((int)a.size(), a.data(), b.data(), out.data());
            g_counters.mult_items += a.size();
        }
        // release buffers whose last reader ran at this level
        for (size_t x = 0; x < P.nodes.size(); ++x)
            if (base[x] && sch.last_use_level[x] == (int)lv && !sch.is_output[x]) {
                ctx.release(base[x]);
                base[x] = nullptr;
            }
    }
    std::vector<u64*> outs;
    std::vector<char> handed(P.nodes.size(), 0);
    for (int o : P.outputs) {
        if (P.nodes[o].kind == PNode::Input || handed[o] || !base[o]) {
            u64* c = ctx.alloc((size_t)K * W);
            std::vector<const u64*> src;
            std::vector<u64*> dst;
            for (int k = 0; k < K; ++k) {
                src.push_back(ptr(o, k));
                dst.push_back(c + (size_t)k * W);
            }
            ctx.copy(K, src.data(), dst.data());
            outs.push_back(c);
        } else {
            outs.push_back(base[o]);
            handed[o] = 1;
        }
    }
    // outputs that were never handed over (e.g. duplicates) are released
    for (size_t x = 0; x < P.nodes.size(); ++x)
        if (base[x] && sch.is_output[x] && !handed[x]) ctx.release(base[x]);
    return outs;
}

}  // namespace hgm
