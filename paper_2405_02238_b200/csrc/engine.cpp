// engine.cpp -- program optimisation and level-batched execution.
#include "engine.hpp"

#include <algorithm>
#include <functional>
#include <map>
#include <stdexcept>
#include <unordered_map>

namespace hgm {

int Program::add_input(size_t S, bool pending) {
    PNode n;
    n.kind = PNode::Input;
    n.pend = pending;
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
    const size_t n0 = q.nodes.size();
    // 1. rotation aliases: identity rotations and duplicate (src, g) pairs.  An
    //    identity rotation of a pending product still reads its materialised
    //    value (oracle rot() of a pending operand), so it becomes a Mat node.
    std::vector<int> alias(n0);
    for (size_t i = 0; i < n0; ++i) alias[i] = (int)i;
    auto root = [&](int x) {
        while (alias[x] != x) x = alias[x];
        return x;
    };
    std::vector<char> pk(n0, 0);
    std::map<std::pair<int, u32>, int> rots;
    std::map<int, int> mats;
    for (size_t i = 0; i < n0; ++i) {
        PNode& nd = q.nodes[i];
        for (int& x : nd.in) x = root(x);
        switch (nd.kind) {
            case PNode::Input: pk[i] = nd.pend; break;
            case PNode::Mult: pk[i] = 1; break;
            case PNode::Comb:
                for (size_t t = 0; t < nd.in.size(); ++t)
                    if (!nd.masks[t] && pk[nd.in[t]]) pk[i] = 1;
                break;
            default: break;
        }
        if (nd.kind == PNode::Rot) {
            const int src = nd.in[0];
            if (nd.g == 1 && !pk[src]) {
                alias[i] = src;
            } else if (nd.g == 1) {
                auto it = mats.find(src);
                if (it != mats.end()) {
                    alias[i] = it->second;
                } else {
                    nd.kind = PNode::Mat;
                    mats.emplace(src, (int)i);
                }
            } else {
                auto key = std::make_pair(src, nd.g);
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
    s.is_output.assign(n0, 0);
    for (int o : q.outputs) s.is_output[o] = 1;
    std::vector<int> uses(n0, 0);
    for (size_t i = 0; i < n0; ++i)
        if (live[i])
            for (int x : q.nodes[i].in) ++uses[x];
    // 3. fold single-use plain addends that are masked sums into their consumer
    //    (a pending child's tensor and addend join the parent's: he_add is
    //    associative on pending values too)
    for (size_t i = 0; i < n0; ++i) {
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
    // 4. every read of a pending value other than a plain sum term reads its
    //    materialised form (one Mat node per value); pending outputs return both
    auto mat_of = [&](int x) {
        auto it = mats.find(x);
        if (it != mats.end()) return it->second;
        PNode m;
        m.kind = PNode::Mat;
        m.in = {x};
        m.S = q.nodes[x].S;
        q.nodes.push_back(std::move(m));
        pk.push_back(0);
        const int id = (int)q.nodes.size() - 1;
        mats.emplace(x, id);
        return id;
    };
    live = liveness(q);
    for (size_t i = 0; i < n0; ++i) {
        if (!live[i] || q.nodes[i].kind == PNode::Mat) continue;
        for (size_t t = 0; t < q.nodes[i].in.size(); ++t) {  // (mat_of appends: no references held)
            const int x = q.nodes[i].in[t];
            const bool sum_term = q.nodes[i].kind == PNode::Comb && !q.nodes[i].masks[t];
            if (pk[x] && !sum_term) {
                const int m = mat_of(x);
                q.nodes[i].in[t] = m;
            }
        }
    }
    s.pending_out.assign(q.outputs.size(), -1);
    for (size_t o = 0; o < q.outputs.size(); ++o) {
        const int x = q.outputs[o];
        if (pk[x]) {
            s.pending_out[o] = x;
            q.outputs[o] = mat_of(x);
        }
    }
    const size_t n = q.nodes.size();
    // liveness from the outputs and the pending outputs
    {
        std::vector<int> stack(q.outputs.begin(), q.outputs.end());
        for (int x : s.pending_out)
            if (x >= 0) stack.push_back(x);
        live.assign(n, 0);
        while (!stack.empty()) {
            const int x = stack.back();
            stack.pop_back();
            if (live[x]) continue;
            live[x] = 1;
            for (int y : q.nodes[x].in) stack.push_back(y);
        }
    }
    s.is_output.assign(n, 0);
    for (int o : q.outputs) s.is_output[o] = 1;
    s.is_pending_output.assign(n, 0);
    for (int x : s.pending_out)
        if (x >= 0) s.is_pending_output[x] = 1;
    // 5. fusion: a product read only by one plain term of a pending sum is
    //    accumulated straight into that sum's tensor
    uses.assign(n, 0);
    for (size_t i = 0; i < n; ++i)
        if (live[i])
            for (int x : q.nodes[i].in) ++uses[x];
    std::vector<char> fused_node(n, 0);
    for (size_t i = 0; i < n; ++i) {
        PNode& nd = q.nodes[i];
        if (!live[i] || nd.kind != PNode::Comb) continue;
        nd.fused.assign(nd.in.size(), 0);
        for (size_t t = 0; t < nd.in.size(); ++t) {
            const int x = nd.in[t];
            if (!nd.masks[t] && q.nodes[x].kind == PNode::Mult && uses[x] == 1 && !s.is_pending_output[x] &&
                !s.is_output[x]) {
                nd.fused[t] = 1;
                fused_node[x] = 1;
            }
        }
    }
    // 6. levels.  Inputs precede their readers, except Mat nodes appended in
    //    step 4, whose source does precede the reader: computed on first use.
    std::vector<int> level(n, -1);
    std::vector<char> done(n, 0);
    int max_level = -1;
    auto get = [&](int x) -> int {
        if (!done[x]) {  // an appended Mat: its source is done
            level[x] = level[q.nodes[x].in[0]] + 1;
            done[x] = 1;
        }
        return level[x];
    };
    auto level_of = [&](int i) -> int {
        if (done[i]) return level[i];
        const PNode& nd = q.nodes[i];
        int lv = -1;
        if (nd.kind == PNode::Enc) {
            lv = 0;
        } else if (nd.kind != PNode::Input) {
            lv = 0;
            for (size_t t = 0; t < nd.in.size(); ++t) {
                const int x = nd.in[t];
                if (nd.kind == PNode::Comb && nd.fused[t]) {
                    for (int y : q.nodes[x].in) lv = std::max(lv, get(y) + 1);
                } else {
                    lv = std::max(lv, get(x) + 1);
                }
            }
        }
        done[i] = 1;
        level[i] = lv;
        return lv;
    };
    for (size_t i = 0; i < n; ++i)
        if (live[i] && !fused_node[i]) max_level = std::max(max_level, level_of((int)i));
    s.levels.assign(max_level + 1, {});
    s.last_use_level.assign(n, -1);
    for (size_t i = 0; i < n; ++i) {
        if (!live[i] || fused_node[i] || level[i] < 0) continue;
        s.levels[level[i]].push_back((int)i);
        const PNode& nd = q.nodes[i];
        if (nd.kind == PNode::Rot) ++s.rot_count;
        if (nd.kind == PNode::Comb) ++s.comb_count;
        if (nd.kind == PNode::Mat) ++s.mat_count;
        if (pk[i]) ++s.pending_count;
        for (size_t t = 0; t < nd.in.size(); ++t) {
            const int x = nd.in[t];
            if (nd.kind == PNode::Comb && nd.fused[t]) {
                ++s.mult_count;
                for (int y : q.nodes[x].in) s.last_use_level[y] = std::max(s.last_use_level[y], level[i]);
            } else {
                s.last_use_level[x] = std::max(s.last_use_level[x], level[i]);
            }
        }
        if (nd.kind == PNode::Mult) ++s.mult_count;
    }
    s.pk = pk;
    return s;
}

std::vector<u64*> execute(Context& ctx, const Schedule& sch, const ExecIO& io) {
    const Program& P = sch.prog;
    const int K = io.K;
    const size_t W = ctx.ct_words(), MW = ctx.modup_words(), PW = ctx.pending_words(), TW = ctx.tensor_words();
    g_counters = ExecCounters{};
    g_counters.levels = sch.levels.size();
    ctx.trim_mask_cache();  // between programs: no mask pointer is held here yet
    std::vector<u64*> base(P.nodes.size(), nullptr);   // plain values
    std::vector<u64*> pbase(P.nodes.size(), nullptr);  // pending values [T][addend]
    auto ptr = [&](int node, int k) -> const u64* {
        const PNode& nd = P.nodes[node];
        if (nd.kind == PNode::Input) return io.input(nd.slot, k);
        return base[node] + (size_t)k * W;
    };
    auto pptr = [&](int node, int k) -> const u64* {
        const PNode& nd = P.nodes[node];
        if (nd.kind == PNode::Input) return io.input_pending(nd.slot, k);
        return pbase[node] + (size_t)k * PW;
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
        std::vector<int> enc, rot, comb, pcomb, mult, mat;
        for (int x : nodes) {
            if (sch.pk[x])
                pbase[x] = ctx.alloc((size_t)K * PW);
            else
                base[x] = ctx.alloc((size_t)K * W);
            switch (P.nodes[x].kind) {
                case PNode::Enc: enc.push_back(x); break;
                case PNode::Rot: rot.push_back(x); break;
                case PNode::Comb: (sch.pk[x] ? pcomb : comb).push_back(x); break;
                case PNode::Mult: mult.push_back(x); break;
                case PNode::Mat: mat.push_back(x); break;
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
        // plain masked sums, and the addends of pending sums (plain terms, masked
        // terms, and the addends of pending non-fused terms)
        if (!comb.empty() || !pcomb.empty()) {
            std::vector<u32> off{0};
            std::vector<const u64*> in, masks;
            std::vector<u64*> out;
            for (int pass = 0; pass < 2; ++pass)
                for (int x : pass == 0 ? comb : pcomb) {
                    const PNode& nd = P.nodes[x];
                    std::vector<const u64*> md(nd.in.size());
                    for (size_t t = 0; t < nd.in.size(); ++t) md[t] = resolve(nd.masks[t]);
                    for (int k = 0; k < K; ++k) {
                        for (size_t t = 0; t < nd.in.size(); ++t) {
                            const int y = nd.in[t];
                            if (pass == 1 && !nd.masks[t] && sch.pk[y]) {
                                if (nd.fused[t]) continue;
                                in.push_back(pptr(y, k) + TW);  // its addend
                            } else {
                                in.push_back(ptr(y, k));
                            }
                            masks.push_back(md[t]);
                        }
                        off.push_back((u32)in.size());
                        out.push_back(pass == 0 ? base[x] + (size_t)k * W : pbase[x] + (size_t)k * PW + TW);
                    }
                }
            ctx.lincomb((int)out.size(), off.data(), in.data(), masks.data(), out.data());
            g_counters.comb_items += out.size();
        }
        // tensors of pending sums: stored pending terms summed, fused products
        // accumulated; non-fused products get their own tensor (addend zero)
        if (!pcomb.empty() || !mult.empty()) {
            std::vector<u32> toff{0}, moff{0};
            std::vector<const u64*> tin, ma, mb;
            std::vector<u64*> tout, mout;
            std::vector<unsigned char> tinit, minit;
            for (int x : pcomb) {
                const PNode& nd = P.nodes[x];
                bool has_t = false;
                for (size_t t = 0; t < nd.in.size(); ++t)
                    if (!nd.masks[t] && sch.pk[nd.in[t]] && !nd.fused[t]) has_t = true;
                for (int k = 0; k < K; ++k) {
                    u64* T = pbase[x] + (size_t)k * PW;
                    if (has_t) {
                        for (size_t t = 0; t < nd.in.size(); ++t)
                            if (!nd.masks[t] && sch.pk[nd.in[t]] && !nd.fused[t]) tin.push_back(pptr(nd.in[t], k));
                        toff.push_back((u32)tin.size());
                        tout.push_back(T);
                        tinit.push_back(0);
                    }
                    bool any = false;
                    for (size_t t = 0; t < nd.in.size(); ++t)
                        if (!nd.masks[t] && nd.fused[t]) {
                            const PNode& m = P.nodes[nd.in[t]];
                            ma.push_back(ptr(m.in[0], k));
                            mb.push_back(ptr(m.in[1], k));
                            any = true;
                        }
                    if (any) {
                        moff.push_back((u32)ma.size());
                        mout.push_back(T);
                        minit.push_back(has_t ? 1 : 0);
                    }
                }
            }
            for (int x : mult) {
                const PNode& nd = P.nodes[x];
                std::vector<u64*> addends;
                for (int k = 0; k < K; ++k) {
                    ma.push_back(ptr(nd.in[0], k));
                    mb.push_back(ptr(nd.in[1], k));
                    moff.push_back((u32)ma.size());
                    mout.push_back(pbase[x] + (size_t)k * PW);
                    minit.push_back(0);
                    HGM_CUDA(cudaMemsetAsync(pbase[x] + (size_t)k * PW + TW, 0, W * 8, ctx.stream()));
                }
            }
            if (!tout.empty()) ctx.tsum((int)tout.size(), toff.data(), tin.data(), tout.data(), tinit.data());
            if (!mout.empty())
                ctx.tensor_acc((int)mout.size(), moff.data(), ma.data(), mb.data(), mout.data(), minit.data());
            g_counters.mult_items += ma.size();
        }
        if (!mat.empty()) {
            std::vector<const u64*> T, A;
            std::vector<u64*> out;
            for (int x : mat)
                for (int k = 0; k < K; ++k) {
                    const u64* p = pptr(P.nodes[x].in[0], k);
                    T.push_back(p);
                    A.push_back(p + TW);
                    out.push_back(base[x] + (size_t)k * W);
                }
            ctx.materialize((int)out.size(), T.data(), A.data(), out.data());
            g_counters.mat_items += out.size();
        }
        // release buffers whose last reader ran at this level
        for (size_t x = 0; x < P.nodes.size(); ++x)
            if (sch.last_use_level[x] == (int)lv) {
                if (base[x] && !sch.is_output[x]) {
                    ctx.release(base[x]);
                    base[x] = nullptr;
                }
                if (pbase[x] && !sch.is_pending_output[x]) {
                    ctx.release(pbase[x]);
                    pbase[x] = nullptr;
                }
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
    // pending forms of pending outputs
    std::vector<char> phanded(P.nodes.size(), 0);
    if (io.pending_out) io.pending_out->assign(P.outputs.size(), nullptr);
    for (size_t o = 0; o < sch.pending_out.size() && io.pending_out; ++o) {
        const int x = sch.pending_out[o];
        if (x < 0) continue;
        if (P.nodes[x].kind == PNode::Input || phanded[x] || !pbase[x]) {
            u64* c = ctx.alloc((size_t)K * PW);
            for (int k = 0; k < K; ++k)
                HGM_CUDA(cudaMemcpyAsync(c + (size_t)k * PW, pptr(x, k), PW * 8, cudaMemcpyDeviceToDevice,
                                         ctx.stream()));
            (*io.pending_out)[o] = c;
        } else {
            (*io.pending_out)[o] = pbase[x];
            phanded[x] = 1;
        }
    }
    for (size_t x = 0; x < P.nodes.size(); ++x)
        if (pbase[x] && sch.is_pending_output[x] && !phanded[x]) ctx.release(pbase[x]);
    return outs;
}

}  // namespace hgm
