// engine.cpp -- program optimisation and level-batched execution.
#include "engine.hpp"

#include <algorithm>
#include <functional>
#include <map>
#include <stdexcept>
#include <unordered_map>

namespace hgm {

int Program::add_input(size_t S, int kind) {
    PNode n;
    n.kind = PNode::Input;
    n.pend = kind;
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

PartLayout part_layout(const Context& ctx, int kind) {
    PartLayout l;
    size_t o = 0;
    if (kind & kPartT) { l.t = o; o += ctx.tensor_words(); }
    if (kind & kPartA) { l.a = o; o += ctx.ks_words(); }
    if (kind & kPartX) { l.x = o; o += ctx.ct_words(); }
    l.words = o;
    return l;
}

namespace {
// the parts a Comb term contributes (oracle cmult_x / add_any): a masked value
// with a pending product is read materialised
int term_kind(int in_kind, bool masked) {
    if (masked && (in_kind & kPartT)) return kPartX;
    return in_kind;
}
}  // namespace

Schedule optimise(const Program& p) {
    Schedule s;
    Program& q = s.prog;
    q = p;
    const size_t n0 = q.nodes.size();
    // 1. value kinds, rotation aliases (identity rotations and duplicate (src, g)
    //    pairs).  An identity rotation of a non-plain value reads its materialised
    //    value (oracle rot_x), so it becomes a Mat node.
    std::vector<int> alias(n0);
    for (size_t i = 0; i < n0; ++i) alias[i] = (int)i;
    auto root = [&](int x) {
        while (alias[x] != x) x = alias[x];
        return x;
    };
    std::vector<int> kind(n0, kPartX);
    std::map<std::pair<int, u32>, int> rots;
    std::map<int, int> mats;
    for (size_t i = 0; i < n0; ++i) {
        PNode& nd = q.nodes[i];
        for (int& x : nd.in) x = root(x);
        switch (nd.kind) {
            case PNode::Input: kind[i] = nd.pend ? nd.pend : kPartX; break;
            case PNode::Mult: kind[i] = kPartT; break;
            case PNode::Comb: {
                int k = 0;
                for (size_t t = 0; t < nd.in.size(); ++t) k |= term_kind(kind[nd.in[t]], nd.masks[t] != nullptr);
                kind[i] = k;
                break;
            }
            case PNode::Rot: {
                const int src = nd.in[0];
                if (nd.g == 1 && kind[src] == kPartX) {
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
                    kind[i] = kPartA;
                    auto key = std::make_pair(src, nd.g);
                    auto it = rots.find(key);
                    if (it != rots.end())
                        alias[i] = it->second;
                    else
                        rots.emplace(key, (int)i);
                }
                break;
            }
            default: break;
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
    //    (he_add is partwise, so a non-plain child's parts join the parent's)
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
    // 4. every read of a non-plain value that is not a Comb term taking its parts
    //    reads its materialised form (one Mat node per value); non-plain outputs
    //    return both
    auto mat_of = [&](int x) {
        auto it = mats.find(x);
        if (it != mats.end()) return it->second;
        PNode m;
        m.kind = PNode::Mat;
        m.in = {x};
        m.S = q.nodes[x].S;
        q.nodes.push_back(std::move(m));
        kind.push_back(kPartX);
        const int id = (int)q.nodes.size() - 1;
        mats.emplace(x, id);
        return id;
    };
    live = liveness(q);
    for (size_t i = 0; i < n0; ++i) {
        if (!live[i] || q.nodes[i].kind == PNode::Mat) continue;
        for (size_t t = 0; t < q.nodes[i].in.size(); ++t) {  // (mat_of appends: no references held)
            const int x = q.nodes[i].in[t];
            if (kind[x] == kPartX) continue;
            const bool comb = q.nodes[i].kind == PNode::Comb, masked = comb && q.nodes[i].masks[t];
            if (comb && (!masked || !(kind[x] & kPartT))) continue;  // the term takes x's parts
            // a non-plain Input's materialised form is supplied (ExecIO::input), except
            // where a Comb term would read it: there it needs a plain node
            if (q.nodes[x].kind == PNode::Input && !comb) continue;
            const int m = mat_of(x);
            q.nodes[i].in[t] = m;
        }
    }
    s.pending_out.assign(q.outputs.size(), -1);
    for (size_t o = 0; o < q.outputs.size(); ++o) {
        const int x = q.outputs[o];
        if (kind[x] != kPartX) {
            s.pending_out[o] = x;
            if (q.nodes[x].kind != PNode::Input) q.outputs[o] = mat_of(x);
        }
    }
    const size_t n = q.nodes.size();
    // liveness from the outputs and the non-plain outputs
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
    // 5. fusion: a product read only by one plain term of a sum is accumulated
    //    straight into that sum's tensor
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
    // 5b. masked sums of rotations: a sum whose key-switch terms are all masked
    //     (stable masks) Rot nodes takes them as one inner product over masked
    //     keys; Rot nodes read only by such sums are never stored.
    s.ks_terms.assign(n, {});
    s.virt.assign(n, 0);
    {
        static const bool on = [] {
            const char* e = std::getenv("HGM_KS_PLAN");
            return !(e && e[0] == '0');
        }();
        std::vector<char> fus(n, 0);
        for (size_t i = 0; i < n && on; ++i) {
            const PNode& nd = q.nodes[i];
            if (!live[i] || nd.kind != PNode::Comb || !(kind[i] & kPartA)) continue;
            bool ok = true;
            for (size_t t = 0; t < nd.in.size() && ok; ++t) {
                const int x = nd.in[t];
                if (!(term_kind(kind[x], nd.masks[t] != nullptr) & kPartA)) continue;
                ok = nd.masks[t] && nd.masks[t]->stable && q.nodes[x].kind == PNode::Rot && kind[x] == kPartA &&
                     !s.is_output[x] && !s.is_pending_output[x];
            }
            fus[i] = ok;
        }
        for (bool changed = on; changed;) {
            changed = false;
            std::vector<char> v(n, 0);
            for (size_t x = 0; x < n; ++x)
                v[x] = live[x] && q.nodes[x].kind == PNode::Rot && kind[x] == kPartA && !s.is_output[x] &&
                       !s.is_pending_output[x];
            for (size_t i = 0; i < n; ++i) {
                if (!live[i]) continue;
                const PNode& nd = q.nodes[i];
                for (size_t t = 0; t < nd.in.size(); ++t)
                    if (!(nd.kind == PNode::Comb && fus[i] && nd.masks[t])) v[nd.in[t]] = 0;
            }
            for (size_t i = 0; i < n; ++i) {
                if (!fus[i]) continue;
                const PNode& nd = q.nodes[i];
                for (size_t t = 0; t < nd.in.size(); ++t)
                    if ((kind[nd.in[t]] & kPartA) && !v[nd.in[t]]) {
                        fus[i] = 0;
                        changed = true;
                        break;
                    }
            }
            if (!changed) s.virt = v;
        }
        // a sum with only a key-switch part whose every reader is a ModDown (Mat) and
        // that is no output itself: its accumulator may be kept as P^-1 acc over Q
        s.prescale.assign(n, 0);
        for (size_t i = 0; i < n; ++i)
            s.prescale[i] = fus[i] && kind[i] == kPartA && !s.is_output[i] && !s.is_pending_output[i];
        for (size_t j = 0; j < n; ++j) {
            if (!live[j]) continue;
            const PNode& rd = q.nodes[j];
            for (int x : rd.in)
                if (rd.kind != PNode::Mat) s.prescale[x] = 0;
        }
        std::map<std::pair<u64, std::vector<u64>>, int> distinct;
        for (size_t i = 0; i < n; ++i) {
            if (!fus[i]) continue;
            const PNode& nd = q.nodes[i];
            std::vector<KsTerm>& kt = s.ks_terms[i];
            for (size_t t = 0; t < nd.in.size(); ++t) {
                const int x = nd.in[t];
                if (!s.virt[x]) continue;
                auto it = std::find_if(kt.begin(), kt.end(), [&](const KsTerm& k) { return k.rot == x; });
                if (it == kt.end()) {
                    KsTerm k;
                    k.rot = x;
                    k.src = q.nodes[x].in[0];
                    k.g = q.nodes[x].g;
                    kt.push_back(std::move(k));
                    it = kt.end() - 1;
                }
                it->masks.push_back(nd.masks[t]);
            }
            for (const KsTerm& k : kt) {
                std::vector<u64> ids;
                for (const MaskRef& m : k.masks) ids.push_back(m->id);
                std::sort(ids.begin(), ids.end());
                distinct.emplace(std::make_pair((u64)k.g | ((u64)s.prescale[i] << 32), std::move(ids)), 0);
            }
            ++s.ks_comb_count;
        }
        s.masked_key_count = distinct.size();
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
                if (nd.kind == PNode::Comb && (nd.fused[t] || s.virt[x])) {
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
        if (live[i] && !fused_node[i] && !s.virt[i]) max_level = std::max(max_level, level_of((int)i));
    s.levels.assign(max_level + 1, {});
    s.last_use_level.assign(n, -1);
    for (size_t i = 0; i < n; ++i) {
        if (live[i] && s.virt[i]) ++s.rot_count;  // executed inside the sums that read it
        if (!live[i] || fused_node[i] || s.virt[i] || level[i] < 0) continue;
        s.levels[level[i]].push_back((int)i);
        const PNode& nd = q.nodes[i];
        if (nd.kind == PNode::Rot) { ++s.rot_count; ++s.stored_rot_count; }
        if (nd.kind == PNode::Comb) ++s.comb_count;
        if (nd.kind == PNode::Comb && (kind[i] & kPartA)) ++s.acc_comb_count;
        if (nd.kind == PNode::Mat) {
            ++s.mat_count;
            if (kind[nd.in[0]] & kPartA) ++s.moddown_count;
            if (kind[nd.in[0]] & kPartT) ++s.rescale_count;
        }
        if (kind[i] & kPartT) ++s.pending_count;
        for (size_t t = 0; t < nd.in.size(); ++t) {
            const int x = nd.in[t];
            if (nd.kind == PNode::Comb && nd.fused[t]) {
                ++s.mult_count;
                for (int y : q.nodes[x].in) s.last_use_level[y] = std::max(s.last_use_level[y], level[i]);
            } else if (s.virt[x]) {
                for (int y : q.nodes[x].in) s.last_use_level[y] = std::max(s.last_use_level[y], level[i]);
            } else {
                s.last_use_level[x] = std::max(s.last_use_level[x], level[i]);
            }
        }
        if (nd.kind == PNode::Mult) ++s.mult_count;
    }
    s.kind = kind;
    return s;
}

std::vector<u64*> execute(Context& ctx, const Schedule& sch, const ExecIO& io) {
    const Program& P = sch.prog;
    const int K = io.K;
    const size_t MW = ctx.modup_words();
    g_counters = ExecCounters{};
    g_counters.levels = sch.levels.size();
    ctx.trim_mask_cache();  // between programs: no mask pointer is held here yet
    const bool masked_keys_ok = sch.masked_key_count > 0 && ctx.masked_keys_fit(sch.masked_key_count);
    const bool prescale_ok = ctx.can_prescale();
    std::vector<char> prescaled_now(P.nodes.size(), 0);  // set when a sum ran over P^-1-scaled masked keys
    if (masked_keys_ok) ctx.trim_masked_keys(sch.masked_key_count);
    std::vector<u64*> buf(P.nodes.size(), nullptr);
    std::vector<PartLayout> lay(P.nodes.size());
    for (size_t x = 0; x < P.nodes.size(); ++x) lay[x] = part_layout(ctx, sch.kind[x]);
    // pointer to a part of node `node`'s value for instance k
    auto part = [&](int node, int k, int which) -> const u64* {
        const PNode& nd = P.nodes[node];
        const PartLayout& l = lay[node];
        const size_t off = which == kPartT ? l.t : which == kPartA ? l.a : l.x;
        if (nd.kind == PNode::Input)
            return (nd.pend ? io.input_pending(nd.slot, k) : io.input(nd.slot, k)) + off;
        return buf[node] + (size_t)k * l.words + off;
    };
    auto wpart = [&](int node, int k, int which) { return const_cast<u64*>(part(node, k, which)); };
    // the value's start (all parts), and its plain (materialised) form: plain nodes,
    // or an Input's supplied materialised form
    auto whole = [&](int node, int k) -> const u64* {
        const PNode& nd = P.nodes[node];
        if (nd.kind == PNode::Input) return nd.pend ? io.input_pending(nd.slot, k) : io.input(nd.slot, k);
        return buf[node] + (size_t)k * lay[node].words;
    };
    auto plain = [&](int node, int k) -> const u64* {
        const PNode& nd = P.nodes[node];
        if (nd.kind == PNode::Input) return io.input(nd.slot, k);
        return part(node, k, kPartX);
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
        std::vector<int> enc, rot, comb, mult, mat;
        for (int x : nodes) {
            buf[x] = ctx.alloc((size_t)K * lay[x].words);
            switch (P.nodes[x].kind) {
                case PNode::Enc: enc.push_back(x); break;
                case PNode::Rot: rot.push_back(x); break;
                case PNode::Comb: comb.push_back(x); break;
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
                    out.push_back(wpart(x, k, kPartX));
                }
            ctx.encrypt((int)vals.size(), vals.data(), S.data(), ctr.data(), out.data());
            g_counters.enc_items += vals.size();
        }
        // masked sums of rotations taken straight from the ModUp digits (Schedule::ks_terms)
        std::vector<int> kcomb;
        for (int x : comb)
            if (!sch.ks_terms[x].empty()) kcomb.push_back(x);
        if (!rot.empty() || !kcomb.empty()) {
            // hoisting: one ModUp per distinct source (and instance)
            std::vector<int> srcs;
            for (int x : rot) srcs.push_back(P.nodes[x].in[0]);
            for (int x : kcomb)
                for (const KsTerm& kt : sch.ks_terms[x]) srcs.push_back(kt.src);
            std::sort(srcs.begin(), srcs.end());
            srcs.erase(std::unique(srcs.begin(), srcs.end()), srcs.end());
            u64* mbuf = ctx.alloc(srcs.size() * (size_t)K * MW);
            std::vector<const u64*> mct;
            std::vector<u64*> mout;
            for (size_t si = 0; si < srcs.size(); ++si)
                for (int k = 0; k < K; ++k) {
                    mct.push_back(plain(srcs[si], k));
                    mout.push_back(mbuf + (si * K + k) * MW);
                }
            ctx.modup((int)mct.size(), mct.data(), mout.data());
            g_counters.modup_items += mct.size();
            auto digits_of = [&](int src, int k) -> const u64* {
                const size_t si = std::lower_bound(srcs.begin(), srcs.end(), src) - srcs.begin();
                return mbuf + (si * K + k) * MW;
            };
            if (!rot.empty()) {
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
                        for (int k = k0; k < std::min(K, k0 + kRotTile); ++k) {
                            mu.push_back(digits_of(src, k));
                            cts.push_back(plain(src, k));
                            gs.push_back(P.nodes[x].g);
                            out.push_back(wpart(x, k, kPartA));
                        }
                    }
                // a pending key switch: the accumulator, P phi(c0) folded in (no ModDown)
                ctx.rotate_acc((int)mu.size(), mu.data(), cts.data(), gs.data(), out.data());
                g_counters.rot_items += mu.size();
            }
            if (!kcomb.empty()) {
                // masked keys of every sum (cached per context); a sum whose keys the
                // cache cannot hold runs rotation by rotation (same value)
                std::vector<std::vector<const u64*>> mk(kcomb.size());
                std::vector<int> slow;
                for (size_t ci = 0; ci < kcomb.size(); ++ci) {
                    const std::vector<KsTerm>& kts = sch.ks_terms[kcomb[ci]];
                    bool ok = masked_keys_ok;
                    const bool pre = prescale_ok && sch.prescale[kcomb[ci]];
                    for (size_t t = 0; t < kts.size() && ok; ++t) {
                        std::vector<u64> ids;
                        std::vector<const u64*> devs;
                        for (const MaskRef& m : kts[t].masks) ids.push_back(m->id);
                        const u64* d = ctx.masked_key(kts[t].g, ids, nullptr, pre);  // cached?
                        if (!d) {
                            for (const MaskRef& m : kts[t].masks) devs.push_back(resolve(m));
                            d = ctx.masked_key(kts[t].g, ids, &devs, pre);
                        }
                        if (!d) ok = false;
                        mk[ci].push_back(d);
                    }
                    if (!ok) {
                        mk[ci].clear();
                        slow.push_back(kcomb[ci]);
                    } else if (pre) {
                        prescaled_now[kcomb[ci]] = 1;  // its accumulators hold P^-1 acc over Q
                    }
                }
                // one group per (tile of instances, sum); tiles in order, sum by sum inside a
                // tile, so the tile's ModUp digits stay in L2 while the masked keys stream
                // past them, each read once per tile
                static const int tile = [] {
                    const char* e = std::getenv("HGM_PLAN_TILE");
                    const int v = e ? std::atoi(e) : 16;
                    return v < 1 ? 1 : v;
                }();
                std::vector<PlanGroup> groups;
                std::vector<const u64*> mkey, dig, c0;
                std::vector<u32> gs;
                std::vector<u64*> out;
                auto flush = [&]() {
                    ctx.rotate_plan(groups, mkey, gs, dig, c0, out);
                    g_counters.plan_items += out.size();
                    groups.clear(); mkey.clear(); dig.clear(); c0.clear(); gs.clear(); out.clear();
                };
                for (int k0 = 0; k0 < K; k0 += tile) {
                    for (size_t ci = 0; ci < kcomb.size(); ++ci) {
                        if (mk[ci].empty()) continue;
                        const int x = kcomb[ci];
                        const std::vector<KsTerm>& kts = sch.ks_terms[x];
                        {
                            const int k1 = k0;
                            PlanGroup G{};
                            G.item0 = (u32)out.size();
                            G.cnt = (u32)(std::min(K, k0 + tile) - k0);
                            G.term0 = (u32)mkey.size();
                            G.nterms = (u32)kts.size();
                            G.dbase = (u32)dig.size();
                            for (size_t t = 0; t < kts.size(); ++t) {
                                mkey.push_back(mk[ci][t]);
                                gs.push_back(kts[t].g);
                            }
                            for (u32 u = 0; u < G.cnt; ++u) {
                                for (size_t t = 0; t < kts.size(); ++t) {
                                    dig.push_back(digits_of(kts[t].src, k1 + (int)u));
                                    c0.push_back(plain(kts[t].src, k1 + (int)u));
                                }
                                out.push_back(wpart(x, k1 + (int)u, kPartA));
                            }
                            groups.push_back(G);
                        }
                    }
                    if (out.size() >= 8192) flush();
                }
                flush();
                // the same sums rotation by rotation: accumulators in temporaries, then the masked sum
                const size_t AW = ctx.ks_words();
                for (size_t s0 = 0; s0 < slow.size();) {
                    size_t s1 = s0, terms = 0;
                    while (s1 < slow.size() && (s1 == s0 || (terms + P.nodes[slow[s1]].in.size()) * K * AW * 8 <= ((size_t)8 << 30))) {
                        terms += P.nodes[slow[s1]].in.size();
                        ++s1;
                    }
                    u64* tmp = ctx.alloc(terms * (size_t)K * AW);
                    std::vector<const u64*> mu, cts, ain, amask;
                    std::vector<u32> rg, aoff{0};
                    std::vector<u64*> racc, aout;
                    size_t slot = 0;
                    for (size_t si = s0; si < s1; ++si) {
                        const int x = slow[si];
                        const PNode& nd = P.nodes[x];
                        std::map<int, size_t> rot_slot;  // each distinct rotation once
                        for (size_t t = 0; t < nd.in.size(); ++t)
                            if (sch.virt[nd.in[t]] && !rot_slot.count(nd.in[t])) {
                                const int y = nd.in[t];
                                rot_slot.emplace(y, slot);
                                for (int k = 0; k < K; ++k) {
                                    mu.push_back(digits_of(P.nodes[y].in[0], k));
                                    cts.push_back(plain(P.nodes[y].in[0], k));
                                    rg.push_back(P.nodes[y].g);
                                    racc.push_back(tmp + (slot * K + k) * AW);
                                }
                                ++slot;
                            }
                        for (int k = 0; k < K; ++k) {
                            for (size_t t = 0; t < nd.in.size(); ++t)
                                if (sch.virt[nd.in[t]]) {
                                    ain.push_back(tmp + (rot_slot[nd.in[t]] * K + k) * AW);
                                    amask.push_back(resolve(nd.masks[t]));
                                }
                            aoff.push_back((u32)ain.size());
                            aout.push_back(wpart(x, k, kPartA));
                        }
                    }
                    ctx.rotate_acc((int)mu.size(), mu.data(), cts.data(), rg.data(), racc.data());
                    ctx.lincomb_qp((int)aout.size(), aoff.data(), ain.data(), amask.data(), aout.data());
                    g_counters.rot_items += mu.size();
                    g_counters.comb_items += aout.size();
                    ctx.release(tmp);
                    s0 = s1;
                }
            }
            ctx.release(mbuf);
        }
        // sums: plain parts (masked or not), key-switch parts over Q ++ P, tensors
        if (!comb.empty()) {
            std::vector<u32> xoff{0}, aoff{0};
            std::vector<const u64*> xin, xmask, ain, amask;
            std::vector<u64*> xout, aout;
            for (int x : comb) {
                const PNode& nd = P.nodes[x];
                const int kx = sch.kind[x];
                std::vector<const u64*> md(nd.in.size());
                for (size_t t = 0; t < nd.in.size(); ++t)
                    md[t] = sch.virt[nd.in[t]] ? nullptr : resolve(nd.masks[t]);  // virtual: masked keys
                for (int k = 0; k < K; ++k) {
                    for (size_t t = 0; t < nd.in.size(); ++t) {
                        const int y = nd.in[t];
                        const int ky = sch.kind[y];
                        if (!nd.fused.empty() && nd.fused[t]) continue;
                        if (ky & kPartX) {
                            xin.push_back(part(y, k, kPartX));
                            xmask.push_back(md[t]);
                        }
                        if ((ky & kPartA) && !sch.virt[y]) {
                            ain.push_back(part(y, k, kPartA));
                            amask.push_back(md[t]);
                        }
                    }
                    if (kx & kPartX) {
                        xoff.push_back((u32)xin.size());
                        xout.push_back(wpart(x, k, kPartX));
                    }
                    if ((kx & kPartA) && sch.ks_terms[x].empty()) {
                        aoff.push_back((u32)ain.size());
                        aout.push_back(wpart(x, k, kPartA));
                    }
                }
            }
            if (!xout.empty()) ctx.lincomb((int)xout.size(), xoff.data(), xin.data(), xmask.data(), xout.data());
            if (!aout.empty()) ctx.lincomb_qp((int)aout.size(), aoff.data(), ain.data(), amask.data(), aout.data());
            g_counters.comb_items += xout.size() + aout.size();
        }
        // tensors: stored tensor terms summed, fused products accumulated;
        // non-fused products get their own tensor
        {
            std::vector<u32> toff{0}, moff{0};
            std::vector<const u64*> tin, ma, mb;
            std::vector<u64*> tout, mout;
            std::vector<unsigned char> tinit, minit;
            for (int x : comb) {
                if (!(sch.kind[x] & kPartT)) continue;
                const PNode& nd = P.nodes[x];
                bool has_t = false;
                for (size_t t = 0; t < nd.in.size(); ++t)
                    if (!nd.masks[t] && (sch.kind[nd.in[t]] & kPartT) && !nd.fused[t]) has_t = true;
                for (int k = 0; k < K; ++k) {
                    u64* T = wpart(x, k, kPartT);
                    if (has_t) {
                        for (size_t t = 0; t < nd.in.size(); ++t)
                            if (!nd.masks[t] && (sch.kind[nd.in[t]] & kPartT) && !nd.fused[t])
                                tin.push_back(part(nd.in[t], k, kPartT));
                        toff.push_back((u32)tin.size());
                        tout.push_back(T);
                        tinit.push_back(0);
                    }
                    bool any = false;
                    for (size_t t = 0; t < nd.in.size(); ++t)
                        if (!nd.masks[t] && nd.fused[t]) {
                            const PNode& m = P.nodes[nd.in[t]];
                            ma.push_back(plain(m.in[0], k));
                            mb.push_back(plain(m.in[1], k));
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
                for (int k = 0; k < K; ++k) {
                    ma.push_back(plain(nd.in[0], k));
                    mb.push_back(plain(nd.in[1], k));
                    moff.push_back((u32)ma.size());
                    mout.push_back(wpart(x, k, kPartT));
                    minit.push_back(0);
                }
            }
            if (!tout.empty()) ctx.tsum((int)tout.size(), toff.data(), tin.data(), tout.data(), tinit.data());
            if (!mout.empty())
                ctx.tensor_acc((int)mout.size(), moff.data(), ma.data(), mb.data(), mout.data(), minit.data());
            g_counters.mult_items += ma.size();
        }
        if (!mat.empty()) {
            // products (+ plain part), then ModDown of key-switch parts, added
            std::vector<const u64*> T, Xp, A1, A1p, A2;
            std::vector<u64*> outT, outA1, outA1p, outA2;
            std::vector<const u64*> addx_a, addx_b;
            std::vector<u64*> addx_o;
            for (int x : mat) {
                const int src = P.nodes[x].in[0];
                const int ks = sch.kind[src];
                for (int k = 0; k < K; ++k) {
                    u64* o = wpart(x, k, kPartX);
                    if (ks & kPartT) {
                        T.push_back(part(src, k, kPartT));
                        Xp.push_back((ks & kPartX) ? part(src, k, kPartX) : nullptr);
                        outT.push_back(o);
                        if (ks & kPartA) {
                            A2.push_back(part(src, k, kPartA));
                            outA2.push_back(o);
                        }
                    } else {  // key switch part (+ plain part)
                        (prescaled_now[src] ? A1p : A1).push_back(part(src, k, kPartA));
                        (prescaled_now[src] ? outA1p : outA1).push_back(o);
                        if (ks & kPartX) {
                            addx_a.push_back(o);
                            addx_b.push_back(part(src, k, kPartX));
                            addx_o.push_back(o);
                        }
                    }
                }
            }
            if (!T.empty()) {
                bool any_x = false;
                for (auto* p : Xp) any_x |= p != nullptr;
                if (any_x) {
                    // materialize() adds one addend per item: split the items by presence
                    std::vector<const u64*> T1, X1, T0;
                    std::vector<u64*> O1, O0;
                    for (size_t i = 0; i < T.size(); ++i) {
                        if (Xp[i]) { T1.push_back(T[i]); X1.push_back(Xp[i]); O1.push_back(outT[i]); }
                        else { T0.push_back(T[i]); O0.push_back(outT[i]); }
                    }
                    ctx.materialize((int)O1.size(), T1.data(), X1.data(), O1.data());
                    ctx.materialize((int)O0.size(), T0.data(), nullptr, O0.data());
                } else {
                    ctx.materialize((int)outT.size(), T.data(), nullptr, outT.data());
                }
            }
            if (!A1.empty()) ctx.moddown((int)A1.size(), A1.data(), outA1.data());
            if (!A1p.empty()) ctx.moddown((int)A1p.size(), A1p.data(), outA1p.data(), true);
            if (!addx_o.empty()) ctx.add((int)addx_o.size(), addx_a.data(), addx_b.data(), addx_o.data());
            if (!A2.empty()) {  // T and A together: ModDown into a temporary, added
                u64* tmp = ctx.alloc(A2.size() * ctx.ct_words());
                std::vector<u64*> to(A2.size());
                std::vector<const u64*> tc(A2.size());
                for (size_t i = 0; i < A2.size(); ++i) tc[i] = to[i] = tmp + i * ctx.ct_words();
                ctx.moddown((int)A2.size(), A2.data(), to.data());
                std::vector<const u64*> oa(outA2.begin(), outA2.end());
                ctx.add((int)A2.size(), oa.data(), tc.data(), outA2.data());
                ctx.release(tmp);
            }
            g_counters.mat_items += mat.size() * (size_t)K;
        }
        // release buffers whose last reader ran at this level
        for (size_t x = 0; x < P.nodes.size(); ++x)
            if (buf[x] && sch.last_use_level[x] == (int)lv && !sch.is_output[x] && !sch.is_pending_output[x]) {
                ctx.release(buf[x]);
                buf[x] = nullptr;
            }
    }
    const size_t W = ctx.ct_words();
    std::vector<u64*> outs;
    std::vector<char> handed(P.nodes.size(), 0);
    for (int o : P.outputs) {  // outputs are plain (Mat nodes for non-plain values)
        if (P.nodes[o].kind == PNode::Input || handed[o] || !buf[o]) {
            u64* c = ctx.alloc((size_t)K * W);
            std::vector<const u64*> src;
            std::vector<u64*> dst;
            for (int k = 0; k < K; ++k) {
                src.push_back(plain(o, k));
                dst.push_back(c + (size_t)k * W);
            }
            ctx.copy(K, src.data(), dst.data());
            outs.push_back(c);
        } else {
            outs.push_back(buf[o]);
            handed[o] = 1;
        }
    }
    // parts of non-plain outputs
    std::vector<char> phanded(P.nodes.size(), 0);
    if (io.pending_out) io.pending_out->assign(P.outputs.size(), nullptr);
    if (io.pending_kind) io.pending_kind->assign(P.outputs.size(), 0);
    for (size_t o = 0; o < sch.pending_out.size() && io.pending_out; ++o) {
        const int x = sch.pending_out[o];
        if (x < 0) continue;
        const size_t PW = lay[x].words;
        if (io.pending_kind) (*io.pending_kind)[o] = sch.kind[x];
        if (P.nodes[x].kind == PNode::Input || phanded[x] || !buf[x]) {
            u64* c = ctx.alloc((size_t)K * PW);
            for (int k = 0; k < K; ++k)
                HGM_CUDA(cudaMemcpyAsync(c + (size_t)k * PW, whole(x, k), PW * 8, cudaMemcpyDeviceToDevice,
                                         ctx.stream()));
            (*io.pending_out)[o] = c;
        } else {
            (*io.pending_out)[o] = buf[x];
            phanded[x] = 1;
        }
    }
    for (size_t x = 0; x < P.nodes.size(); ++x) {
        if (!buf[x]) continue;
        const bool keep_plain = sch.is_output[x] && handed[x];
        const bool keep_parts = sch.is_pending_output[x] && phanded[x];
        if (!keep_plain && !keep_parts) ctx.release(buf[x]);
    }
    return outs;
}

}  // namespace hgm
