// parallel.hpp -- host-side parallel loop for the client work around the GPU
// path (packing slot vectors, residue conversion into pinned staging, unpacking).
#pragma once
#include <algorithm>
#include <cstddef>
#include <thread>
#include <vector>

namespace hgm {

inline unsigned host_threads() {
    static const unsigned t = [] {
        const unsigned h = std::thread::hardware_concurrency();
        return std::max(1u, std::min(h ? h : 1u, 32u));
    }();
    return t;
}

// f(i) for i in [0, n), split into contiguous ranges over host_threads();
// serial below `grain` items.
template <typename F>
void parallel_for(size_t n, F&& f, size_t grain = 16) {
    const size_t T = std::min<size_t>(host_threads(), (n + grain - 1) / std::max<size_t>(grain, 1));
    if (T <= 1) {
        for (size_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(T - 1);
    const size_t per = (n + T - 1) / T;
    for (size_t t = 1; t < T; ++t) {
        const size_t b = t * per, e = std::min(n, b + per);
        if (b >= e) break;
        th.emplace_back([&f, b, e] {
            for (size_t i = b; i < e; ++i) f(i);
        });
    }
    for (size_t i = 0; i < std::min(n, per); ++i) f(i);
    for (auto& x : th) x.join();
}

}  // namespace hgm
