// Host check of the device arithmetic helpers in csrc/common.cuh (their non-CUDA
// branches compute the same values as the PTX forms): Shoup and Barrett products,
// the column accumulator and both 128-bit reductions against unsigned __int128,
// for every prime of every parameter set, on random and extreme operands.
// Build: g++ -O2 -std=c++17 -I ../../paper_2405_02238_b200/csrc arith_check.cpp ../../paper_2405_02238_b200/csrc/params.cpp
#include <cstdio>
#include <cstdlib>

#include "params.hpp"

using namespace hgm;
using u128 = unsigned __int128;

static u64 rng_state = 0x9e3779b97f4a7c15ULL;
static u64 rnd() {
    rng_state += 0x9e3779b97f4a7c15ULL;
    return mix64(rng_state);
}

#define CHECK(cond, ...)                         \
    do {                                         \
        if (!(cond)) {                           \
            std::printf("FAIL: " __VA_ARGS__);   \
            std::printf("\n");                   \
            return 1;                            \
        }                                        \
    } while (0)

template <int S>
static int check_prime(const Prime& P, int products_wide) {
    const u64 q = P.q;
    const u64 edge[] = {0, 1, 2, q - 1, q - 2, q / 2, (q - 1) / 2 + 1};
    auto pick = [&](int i) { return i < 7 ? edge[i] : rnd() % q; };
    for (int it = 0; it < 20000; ++it) {
        const u64 a = pick(it % 11), b = pick((it / 11) % 11);
        // shifted Barrett product of two residues
        CHECK(mul_mod(a, b, P) == (u64)((u128)a * b % q), "mul_mod q=%llu", (unsigned long long)q);
        // Shoup product of any 64-bit a by a residue w
        const u64 w = b, ws = (u64)(((u128)w << 64) / q), any = it % 3 ? rnd() : ~0ULL - (u64)it;
        CHECK(shoup_mul(any, w, ws, q) == (u64)((u128)any * w % q), "shoup_mul");
        CHECK(shoup_lazy3(any, w, ws, q) < 3 * q && shoup_lazy3(any, w, ws, q) % q == (u64)((u128)any * w % q),
              "shoup_lazy3 range");
        CHECK(shoup_lazy(any, w, ws, q) < 2 * q, "shoup_lazy range");
        // column accumulator: 4 products and a residue, one reduce_acc
        u64 xs[8], ys[8];
        for (int k = 0; k < 8; ++k) {
            xs[k] = it < 64 ? q - 1 : pick((it + k) % 13);
            ys[k] = it < 64 ? q - 1 : pick((it + 3 * k) % 13);
        }
        const u64 r0 = it < 64 ? q - 1 : rnd() % q;
        {
            Cols c;
            c.x = r0;
            u128 want = r0;
            for (int k = 0; k < 4; ++k) {
                c.mac(split<S>(xs[k]), split<S>(ys[k]));
                want += (u128)xs[k] * ys[k];
            }
            CHECK(reduce_acc(c.fold<S>(), P) == (u64)(want % q), "reduce_acc (4 products + residue)");
        }
        // two folds of 4 products and a residue, one reduce_acc_wide (k_ks_plan)
        {
            Acc s{r0, 0};
            u128 want = r0;
            for (int t = 0; t < products_wide / 4; ++t) {
                Cols c;
                for (int k = 0; k < 4; ++k) {
                    c.mac(split<S>(xs[4 * t + k]), split<S>(ys[4 * t + k]));
                    want += (u128)xs[4 * t + k] * ys[4 * t + k];
                }
                const Acc f = c.fold<S>();
                add128(s.lo, s.hi, f.lo, f.hi);
            }
            CHECK(reduce_acc_wide(s, P) == (u64)(want % q), "reduce_acc_wide (8 products + residue) q=%llu it=%d",
                  (unsigned long long)q, it);
        }
        // sums and differences
        CHECK(add_mod(a, b, q) == (a + b) % q, "add_mod");
        CHECK(sub_mod(a, b, q) == (a + q - b) % q, "sub_mod");
    }
    return 0;
}

int main() {
    for (int id = 0; id < 3; ++id) {
        const HostParams hp = make_params(id, 1);
        for (size_t i = 0; i < hp.primes.size(); ++i) {
            const Prime& P = hp.dev.pr[i];
            CHECK(P.q == hp.primes[i] && (P.q & 0xffffffffULL) == 1, "prime table");
            const int rc = hp.spec.qbits == 60 ? check_prime<30>(P, 8) : check_prime<28>(P, 8);
            if (rc) return rc;
        }
    }
    std::printf("arith ok\n");
    return 0;
}
