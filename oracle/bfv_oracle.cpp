// bfv_oracle.cpp -- TEST INFRASTRUCTURE ONLY.  See bfv_oracle.h.
//
// Definitional, op-by-op RNS-BFV.  Every primitive follows the op semantics
// of the reference backend contract:
//   encrypt  : proj/src/backend.cpp:118-134 (empty -> DimensionError,
//              S > slot_count -> CapacityError, values reduced mod t)
//   decrypt  : proj/src/backend.cpp:136-139 (returns the S logical slots,
//              canonical in [0, t) as SlotBackend{N/2, 65537} does)
//   he_add   : proj/src/backend.cpp:141-153
//   he_mult  : proj/src/backend.cpp:155-167 (a PENDING product: the tensor is
//              scaled, rounded and relinearised when a non-add op reads it,
//              so he_add chains of products round once -- see XCt below)
//   he_cmult : proj/src/backend.cpp:169-183 (mask length == segment; masks a
//              value's plain and key-switch parts, see XCt below)
//   he_rot   : proj/src/backend.cpp:185-197 (left rotation; BFV rotates the
//              whole N/2-slot row, see backend.hpp:129-131 and SURVEY.md §8
//              "Row semantics verified"; a PENDING key switch: ModDown runs
//              when a non-add, non-mask op reads it, once per masked sum)
// The arithmetic below is the spec the GPU library reproduces bit-exactly:
// integer-only scale-and-round, centred (symmetric) digit lifting in ModUp,
// Galois element g = 3^z mod 2N, and a counter-based sampler.  The oracle's
// rotation applies the automorphism in the COEFFICIENT domain and key-switches
// the permuted polynomial (no hoisting); the GPU hoists ModUp and permutes in
// the NTT domain.  Equality of the two is what proves hoisting exact.
#include "bfv_oracle.h"

#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

using u64 = uint64_t;
using i64 = int64_t;
using u128 = unsigned __int128;
using Poly = std::vector<u64>;

thread_local std::string g_err;

// ---------------------------------------------------------------- arithmetic
inline u64 mulmod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
inline u64 addmod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
inline u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
u64 powmod(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    while (e) { if (e & 1) r = mulmod(r, a, q); a = mulmod(a, a, q); e >>= 1; }
    return r;
}
u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }  // q prime
inline u64 from_signed(i64 v, u64 q) {
    if (v >= 0) return (u64)v % q;
    u64 m = (u64)(-(v + 1)) % q;  // -(v) - 1, avoids INT64_MIN overflow
    return q - 1 - m;
}
// centred representative of y in [0,q): y > (q-1)/2 maps to y - q
inline i64 centred(u64 y, u64 q) { return y > (q - 1) / 2 ? -(i64)(q - y) : (i64)y; }

bool is_prime(u64 n) {
    if (n < 2) return false;
    for (u64 p : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull})
        if (n % p == 0) return n == p;
    u64 d = n - 1; int s = 0;
    while (!(d & 1)) { d >>= 1; ++s; }
    for (u64 a : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
        u64 x = powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; ++r) { x = mulmod(x, x, n); if (x == n - 1) { comp = false; break; } }
        if (comp) return false;
    }
    return true;
}

unsigned brv(unsigned x, unsigned bits) {
    unsigned r = 0;
    for (unsigned i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

// 128-bit fixed-point fraction: floor(a * 2^128 / q) for a < q, as (hi, lo).
struct Frac { u64 hi, lo; };
Frac frac128(u64 a, u64 q) {
    u128 num = (u128)a << 64;
    u64 hi = (u64)(num / q);
    u64 rem = (u64)(num % q);
    u64 lo = (u64)(((u128)rem << 64) / q);
    return {hi, lo};
}
// y * F in units of 2^-64 (the low product of y*F.lo is dropped)
inline u128 fx_term(u64 y, Frac f) { return (u128)y * f.hi + (u64)(((u128)y * f.lo) >> 64); }
inline u64 fx_round(u128 s) { return (u64)((s + ((u128)1 << 63)) >> 64); }

// ---------------------------------------------------------------- sampler
inline u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
u64 prng(u64 seed, u64 stream, u64 idx) {
    u64 h = mix64(seed ^ 0x5851f42d4c957f2dULL);
    h = mix64(h ^ stream);
    return mix64(h + (idx + 1) * 0x9e3779b97f4a7c15ULL);
}
// |x| CDT for the discrete Gaussian sigma = 3.2, tail cut 19 (SEAL's 6 sigma):
// T[k] = floor(2^63 * P(|X| <= k)); committed from a double-precision derivation; oracle/gen_cdt.py recomputes it
// exactly (60-digit decimal) and checks every entry to within 2^-50 (tests/test_oracle.py).
const u64 kCdt[20] = {
    0x0ff52b40a5917e80ULL, 0x2e5a25d4bf0e3e00ULL, 0x489ae26955b04800ULL, 0x5d2bc20f621bf000ULL,
    0x6bc8694c3cc81000ULL, 0x7532d89ac6ba8000ULL, 0x7ab396cb74436c00ULL, 0x7d9e4e916643f000ULL,
    0x7f05495819eb2400ULL, 0x7fa1ce9c0039ac00ULL, 0x7fdfb3f212e8c800ULL, 0x7ff5e6f9d2315400ULL,
    0x7ffd1f97bc440c00ULL, 0x7fff40fa0088d800ULL, 0x7fffd2e835e1cc00ULL, 0x7ffff65243870400ULL,
    0x7ffffe1db476a400ULL, 0x7fffffac0a1dd000ULL, 0x7ffffff428673c00ULL, 0x8000000000000000ULL};
i64 gauss(u64 seed, u64 stream, u64 idx) {
    u64 r = prng(seed, stream, idx);
    u64 mag = r & 0x7fffffffffffffffULL;
    i64 k = 0;
    while (mag >= kCdt[k]) ++k;
    return (r >> 63) ? -k : k;
}
inline i64 ternary(u64 seed, u64 stream, u64 idx) {
    return (i64)(((u128)prng(seed, stream, idx) * 3) >> 64) - 1;
}
inline u64 uniform(u64 seed, u64 stream, u64 idx, u64 q) {
    return (u64)(((u128)prng(seed, stream, idx) * q) >> 64);
}
// stream tags (the GPU library uses the same constants)
constexpr u64 kStreamSk = 1ULL << 56, kStreamPkA = 2ULL << 56, kStreamPkE = 3ULL << 56,
              kStreamKsA = 4ULL << 56, kStreamKsE = 5ULL << 56, kStreamEncU = 6ULL << 56,
              kStreamEncE0 = 7ULL << 56, kStreamEncE1 = 8ULL << 56;

// ---------------------------------------------------------------- params
struct Spec { unsigned logN, qbits, L, K, dnum, nB; };
const Spec kSpecs[] = {{13, 60, 3, 1, 3, 4}, {15, 55, 8, 4, 2, 9}, {12, 60, 3, 1, 3, 4}};
constexpr u64 kT = 65537;

struct Prime {
    u64 q = 0, psi = 0, ninv = 0;
    Poly psi_rev, psi_rev_shoup, ipsi_rev, ipsi_rev_shoup;
};

// Smallest x >= 2 whose (q-1)/2N power is a primitive 2N-th root (psi^N = -1).
u64 find_psi(u64 q, unsigned N) {
    for (u64 x = 2;; ++x) {
        u64 psi = powmod(x, (q - 1) / (2 * N), q);
        if (powmod(psi, N, q) == q - 1) return psi;
    }
}

void make_tables(Prime& p, unsigned logN) {
    const unsigned N = 1u << logN;
    p.psi = find_psi(p.q, N);
    const u64 ipsi = invmod(p.psi, p.q);
    p.ninv = invmod(N, p.q);
    p.psi_rev.resize(N); p.ipsi_rev.resize(N);
    p.psi_rev_shoup.resize(N); p.ipsi_rev_shoup.resize(N);
    for (unsigned i = 0; i < N; ++i) {
        unsigned e = brv(i, logN);
        p.psi_rev[i] = powmod(p.psi, e, p.q);
        p.ipsi_rev[i] = powmod(ipsi, e, p.q);
        p.psi_rev_shoup[i] = (u64)(((u128)p.psi_rev[i] << 64) / p.q);
        p.ipsi_rev_shoup[i] = (u64)(((u128)p.ipsi_rev[i] << 64) / p.q);
    }
}

inline u64 shoup(u64 a, u64 w, u64 ws, u64 q) {
    u64 hi = (u64)(((u128)a * ws) >> 64);
    u64 r = a * w - hi * q;
    return r >= q ? r - q : r;
}

// Forward negacyclic NTT, Cooley-Tukey, natural in / bit-reversed out:
// out[k] = sum_j a[j] psi^{j (2 brv(k) + 1)}.
void ntt_fwd(Poly& a, const Prime& p) {
    const size_t N = a.size();
    const u64 q = p.q;
    for (size_t m = 1, t = N / 2; m < N; m <<= 1, t >>= 1)
        for (size_t i = 0; i < m; ++i) {
            const u64 w = p.psi_rev[m + i], ws = p.psi_rev_shoup[m + i];
            for (size_t j = 2 * i * t; j < 2 * i * t + t; ++j) {
                u64 U = a[j], V = shoup(a[j + t], w, ws, q);
                a[j] = addmod(U, V, q);
                a[j + t] = submod(U, V, q);
            }
        }
}
// Inverse, Gentleman-Sande, bit-reversed in / natural out, scaled by N^-1.
void ntt_inv(Poly& a, const Prime& p) {
    const size_t N = a.size();
    const u64 q = p.q;
    for (size_t m = N / 2, t = 1; m >= 1; m >>= 1, t <<= 1)
        for (size_t i = 0; i < m; ++i) {
            const u64 w = p.ipsi_rev[m + i], ws = p.ipsi_rev_shoup[m + i];
            for (size_t j = 2 * i * t; j < 2 * i * t + t; ++j) {
                u64 U = a[j], V = a[j + t];
                a[j] = addmod(U, V, q);
                a[j + t] = shoup(submod(U, V, q), w, ws, q);
            }
        }
    for (auto& v : a) v = mulmod(v, p.ninv, q);
}

struct KsKey { std::vector<std::vector<Poly>> k0, k1; };  // [digit][limb in Q++P]

}  // namespace

struct orc_ctx {
    Spec spec{};
    unsigned N = 0, logN = 0, L = 0, K = 0, nB = 0, dnum = 0, alpha = 0;
    u64 seed = 0;
    std::vector<Prime> pr;  // Q ++ P ++ B
    Prime tp;               // plaintext modulus t
    std::vector<unsigned> slot_ntt;  // slot index (row*N/2 + col) -> NTT index
    std::vector<i64> s_coeff;
    std::vector<Poly> s_ntt;  // over Q ++ P
    std::vector<Poly> pk0, pk1;  // over Q
    std::map<u64, std::unique_ptr<KsKey>> keys;
    // NTT-domain lifts of masks over Q ++ P, by content (a cache: the values are
    // exactly what cmult / mask_qp would compute again)
    mutable std::mutex mask_mu;
    mutable std::map<std::vector<int64_t>, std::shared_ptr<const std::vector<Poly>>> masks;

    // constants
    std::vector<u64> delta;            // floor(Q/t) mod q_i
    std::vector<u64> qhat_inv;         // (Q/q_i)^-1 mod q_i
    std::vector<Frac> t_over_q;        // t / q_i (decrypt)
    std::vector<Frac> one_over_q;      // 1 / q_i   (Q -> B exact)
    std::vector<std::vector<u64>> qhat_mod_b;  // [i][j] (Q/q_i) mod b_j
    std::vector<u64> Q_mod_b;
    std::vector<u64> dhat_inv;         // (Q B / q_i)^-1 mod q_i
    std::vector<std::vector<u64>> W;   // floor(tB/q_i) mod b_j
    std::vector<Frac> F;               // frac(tB/q_i)
    std::vector<u64> T;                // t Q^-1 mod b_j
    std::vector<u64> bhat_inv;         // (B/b_j)^-1 mod b_j
    std::vector<Frac> one_over_b;
    std::vector<std::vector<u64>> bhat_mod_q;  // [j][i] (B/b_j) mod q_i
    std::vector<u64> B_mod_q;
    // key switching
    std::vector<std::vector<u64>> dg_hat_inv;            // [d][local] (Q_d/q_i)^-1 mod q_i
    std::vector<std::vector<std::vector<u64>>> dg_hat;   // [d][local][r] (Q_d/q_i) mod r
    std::vector<u64> P_mod_r;                            // P mod r (r in Q)
    std::vector<u64> phat_inv;                           // (P/p_k)^-1 mod p_k
    std::vector<std::vector<u64>> phat_mod_q;            // [k][i] (P/p_k) mod q_i
    std::vector<u64> P_inv_q;                            // P^-1 mod q_i

    const Prime& P(unsigned r) const { return pr[r]; }
    unsigned R() const { return L + K; }
    unsigned bidx(unsigned j) const { return L + K + j; }
};

namespace {

Poly lift_signed(const std::vector<i64>& v, u64 q) {
    Poly out(v.size());
    for (size_t j = 0; j < v.size(); ++j) out[j] = from_signed(v[j], q);
    return out;
}

void build(orc_ctx& c, int id) {
    if (id < 0 || id > 2) throw std::invalid_argument("unknown param id");
    c.spec = kSpecs[id];
    c.logN = c.spec.logN; c.N = 1u << c.logN;
    c.L = c.spec.L; c.K = c.spec.K; c.nB = c.spec.nB; c.dnum = c.spec.dnum;
    c.alpha = c.L / c.dnum;
    const unsigned N = c.N, L = c.L, K = c.K, nB = c.nB;
    // primes: descending q = 2^bits - k*2^32 + 1 (= 1 mod 2^32, hence mod 2N)
    const unsigned need = L + K + nB;
    for (u64 k = 1; c.pr.size() < need; ++k) {
        u64 cand = (1ULL << c.spec.qbits) - (k << 32) + 1;
        if (is_prime(cand)) { Prime p; p.q = cand; c.pr.push_back(p); }
    }
    for (auto& p : c.pr) make_tables(p, c.logN);
    c.tp.q = kT;
    make_tables(c.tp, c.logN);
    // slot map
    c.slot_ntt.resize(N);
    const unsigned H = N / 2;
    u64 ex = 1;
    for (unsigned i = 0; i < H; ++i) {
        c.slot_ntt[i] = brv((unsigned)((ex - 1) / 2), c.logN);
        u64 ex2 = 2 * N - ex;
        c.slot_ntt[H + i] = brv((unsigned)((ex2 - 1) / 2), c.logN);
        ex = ex * 3 % (2 * N);
    }
    auto qv = [&](unsigned i) { return c.pr[i].q; };
    auto bv = [&](unsigned j) { return c.pr[c.bidx(j)].q; };
    // decrypt / encrypt constants
    u64 Q_mod_t = 1;
    for (unsigned i = 0; i < L; ++i) Q_mod_t = mulmod(Q_mod_t, qv(i) % kT, kT);
    c.delta.resize(L); c.qhat_inv.resize(L); c.t_over_q.resize(L); c.one_over_q.resize(L);
    for (unsigned i = 0; i < L; ++i) {
        u64 q = qv(i), qhat = 1;
        for (unsigned k = 0; k < L; ++k) if (k != i) qhat = mulmod(qhat, qv(k) % q, q);
        c.qhat_inv[i] = invmod(qhat, q);
        // floor(Q/t) = (Q - (Q mod t)) / t  ==  -(Q mod t) * t^-1  (mod q_i)
        c.delta[i] = mulmod(q - (Q_mod_t % q), invmod(kT % q, q), q) % q;
        c.t_over_q[i] = frac128(kT, q);
        c.one_over_q[i] = frac128(1, q);
    }
    // mult constants
    c.qhat_mod_b.assign(L, std::vector<u64>(nB));
    c.Q_mod_b.resize(nB);
    for (unsigned j = 0; j < nB; ++j) {
        u64 b = bv(j), Qb = 1;
        for (unsigned i = 0; i < L; ++i) Qb = mulmod(Qb, qv(i) % b, b);
        c.Q_mod_b[j] = Qb;
        for (unsigned i = 0; i < L; ++i) {
            u64 h = 1;
            for (unsigned k = 0; k < L; ++k) if (k != i) h = mulmod(h, qv(k) % b, b);
            c.qhat_mod_b[i][j] = h;
        }
    }
    c.dhat_inv.resize(L); c.W.assign(L, std::vector<u64>(nB)); c.F.resize(L);
    for (unsigned i = 0; i < L; ++i) {
        u64 q = qv(i), Bq = 1;
        for (unsigned j = 0; j < nB; ++j) Bq = mulmod(Bq, bv(j) % q, q);
        u64 qhat = 1;
        for (unsigned k = 0; k < L; ++k) if (k != i) qhat = mulmod(qhat, qv(k) % q, q);
        c.dhat_inv[i] = invmod(mulmod(qhat, Bq, q), q);
        u64 tB_mod_q = mulmod(kT % q, Bq, q);  // (tB) mod q_i
        c.F[i] = frac128(tB_mod_q, q);
        for (unsigned j = 0; j < nB; ++j) {
            u64 b = bv(j);
            // floor(tB/q_i) = (tB - (tB mod q_i)) / q_i == -(tB mod q_i) q_i^-1 (mod b_j)
            c.W[i][j] = mulmod((b - tB_mod_q % b) % b, invmod(q % b, b), b);
        }
    }
    c.T.resize(nB); c.bhat_inv.resize(nB); c.one_over_b.resize(nB);
    c.bhat_mod_q.assign(nB, std::vector<u64>(L)); c.B_mod_q.resize(L);
    for (unsigned j = 0; j < nB; ++j) {
        u64 b = bv(j);
        c.T[j] = mulmod(kT % b, invmod(c.Q_mod_b[j], b), b);
        u64 bh = 1;
        for (unsigned k = 0; k < nB; ++k) if (k != j) bh = mulmod(bh, bv(k) % b, b);
        c.bhat_inv[j] = invmod(bh, b);
        c.one_over_b[j] = frac128(1, b);
        for (unsigned i = 0; i < L; ++i) {
            u64 q = qv(i), h = 1;
            for (unsigned k = 0; k < nB; ++k) if (k != j) h = mulmod(h, bv(k) % q, q);
            c.bhat_mod_q[j][i] = h;
        }
    }
    for (unsigned i = 0; i < L; ++i) {
        u64 q = qv(i), Bq = 1;
        for (unsigned j = 0; j < nB; ++j) Bq = mulmod(Bq, bv(j) % q, q);
        c.B_mod_q[i] = Bq;
    }
    // key switching constants
    const unsigned R = c.R(), A = c.alpha;
    c.dg_hat_inv.assign(c.dnum, std::vector<u64>(A));
    c.dg_hat.assign(c.dnum, std::vector<std::vector<u64>>(A, std::vector<u64>(R)));
    for (unsigned d = 0; d < c.dnum; ++d)
        for (unsigned a = 0; a < A; ++a) {
            unsigned i = d * A + a;
            u64 q = qv(i), h = 1;
            for (unsigned a2 = 0; a2 < A; ++a2) if (a2 != a) h = mulmod(h, qv(d * A + a2) % q, q);
            c.dg_hat_inv[d][a] = invmod(h, q);
            for (unsigned r = 0; r < R; ++r) {
                u64 m = c.pr[r].q, hr = 1;
                for (unsigned a2 = 0; a2 < A; ++a2) if (a2 != a) hr = mulmod(hr, qv(d * A + a2) % m, m);
                c.dg_hat[d][a][r] = hr;
            }
        }
    c.P_mod_r.resize(L);
    c.P_inv_q.resize(L);
    for (unsigned i = 0; i < L; ++i) {
        u64 q = qv(i), Pm = 1;
        for (unsigned k = 0; k < K; ++k) Pm = mulmod(Pm, c.pr[L + k].q % q, q);
        c.P_mod_r[i] = Pm;
        c.P_inv_q[i] = invmod(Pm, q);
    }
    c.phat_inv.resize(K);
    c.phat_mod_q.assign(K, std::vector<u64>(L));
    for (unsigned k = 0; k < K; ++k) {
        u64 p = c.pr[L + k].q, h = 1;
        for (unsigned k2 = 0; k2 < K; ++k2) if (k2 != k) h = mulmod(h, c.pr[L + k2].q % p, p);
        c.phat_inv[k] = invmod(h, p);
        for (unsigned i = 0; i < L; ++i) {
            u64 q = qv(i), hq = 1;
            for (unsigned k2 = 0; k2 < K; ++k2) if (k2 != k) hq = mulmod(hq, c.pr[L + k2].q % q, q);
            c.phat_mod_q[k][i] = hq;
        }
    }
    // secret key
    c.s_coeff.resize(N);
    for (unsigned j = 0; j < N; ++j) c.s_coeff[j] = ternary(c.seed, kStreamSk, j);
    c.s_ntt.resize(R);
    for (unsigned r = 0; r < R; ++r) {
        c.s_ntt[r] = lift_signed(c.s_coeff, c.pr[r].q);
        ntt_fwd(c.s_ntt[r], c.pr[r]);
    }
    // public key: pk1 = a (sampled directly in the NTT domain), pk0 = -a s + e
    std::vector<i64> e(N);
    for (unsigned j = 0; j < N; ++j) e[j] = gauss(c.seed, kStreamPkE, j);
    c.pk0.resize(L); c.pk1.resize(L);
    for (unsigned i = 0; i < L; ++i) {
        const u64 q = qv(i);
        Poly a(N), ee = lift_signed(e, q);
        for (unsigned j = 0; j < N; ++j) a[j] = uniform(c.seed, kStreamPkA, (u64)i * N + j, q);
        ntt_fwd(ee, c.pr[i]);
        Poly p0(N);
        for (unsigned j = 0; j < N; ++j) p0[j] = submod(ee[j], mulmod(a[j], c.s_ntt[i][j], q), q);
        c.pk0[i] = std::move(p0);
        c.pk1[i] = std::move(a);
    }
}

// automorphism X -> X^g on a coefficient-domain polynomial
Poly automorph_coeff(const Poly& a, u64 g, u64 q) {
    const size_t N = a.size();
    Poly out(N);
    for (size_t j = 0; j < N; ++j) {
        u64 idx = (u64)j * g % (2 * N);
        if (idx < N) out[idx] = a[j];
        else out[idx - N] = a[j] ? q - a[j] : 0;
    }
    return out;
}

// Switching key for the target secret s' (given over Q ++ P, NTT domain).
KsKey make_key(const orc_ctx& c, u64 kid, const std::vector<Poly>& sp) {
    const unsigned N = c.N, R = c.R();
    KsKey k;
    k.k0.assign(c.dnum, std::vector<Poly>(R, Poly(N)));
    k.k1.assign(c.dnum, std::vector<Poly>(R, Poly(N)));
    for (unsigned d = 0; d < c.dnum; ++d) {
        const u64 sa = kStreamKsA | (kid << 8) | d, se = kStreamKsE | (kid << 8) | d;
        std::vector<i64> e(N);
        for (unsigned j = 0; j < N; ++j) e[j] = gauss(c.seed, se, j);
        for (unsigned r = 0; r < R; ++r) {
            const u64 q = c.pr[r].q;
            Poly ee = lift_signed(e, q);
            ntt_fwd(ee, c.pr[r]);
            const bool in_digit = r < c.L && r / c.alpha == d;
            for (unsigned j = 0; j < N; ++j) {
                u64 a = uniform(c.seed, sa, (u64)r * N + j, q);
                u64 v = submod(ee[j], mulmod(a, c.s_ntt[r][j], q), q);
                if (in_digit) v = addmod(v, mulmod(c.P_mod_r[r], sp[r][j], q), q);
                k.k0[d][r][j] = v;
                k.k1[d][r][j] = a;
            }
        }
    }
    return k;
}

const KsKey& get_key(orc_ctx& c, u64 kid) {
    auto it = c.keys.find(kid);
    if (it != c.keys.end()) return *it->second;
    std::vector<Poly> sp(c.R());
    for (unsigned r = 0; r < c.R(); ++r) {
        const u64 q = c.pr[r].q;
        if (kid == 0) {  // relinearisation key: s^2
            sp[r].resize(c.N);
            for (unsigned j = 0; j < c.N; ++j) sp[r][j] = mulmod(c.s_ntt[r][j], c.s_ntt[r][j], q);
        } else {  // Galois key: phi_g(s)
            sp[r] = automorph_coeff(lift_signed(c.s_coeff, q), kid, q);
            ntt_fwd(sp[r], c.pr[r]);
        }
    }
    auto k = std::make_unique<KsKey>(make_key(c, kid, sp));
    return *c.keys.emplace(kid, std::move(k)).first->second;
}

// Hybrid key switching of a coefficient-domain polynomial d (L limbs, mod Q).
// Returns (u0, u1) over Q in the NTT domain.
// The key-switch accumulator before ModDown: (acc0, acc1) over Q ++ P, NTT domain.
void ks_acc(orc_ctx& c, const std::vector<Poly>& d, u64 kid, std::vector<Poly>& acc0, std::vector<Poly>& acc1) {
    const KsKey& key = get_key(c, kid);
    const unsigned N = c.N, L = c.L, R = c.R(), A = c.alpha;
    acc0.assign(R, Poly(N, 0));
    acc1.assign(R, Poly(N, 0));
    for (unsigned dg = 0; dg < c.dnum; ++dg) {
        // centred digit residues y_i = [d_i (Q_d/q_i)^-1]_{q_i}
        std::vector<std::vector<i64>> y(A, std::vector<i64>(N));
        for (unsigned a = 0; a < A; ++a) {
            const unsigned i = dg * A + a;
            for (unsigned j = 0; j < N; ++j)
                y[a][j] = centred(mulmod(d[i][j], c.dg_hat_inv[dg][a], c.pr[i].q), c.pr[i].q);
        }
        for (unsigned r = 0; r < R; ++r) {
            const u64 q = c.pr[r].q;
            Poly x(N);
            if (r < L && r / A == dg) {
                x = d[r];
            } else {
                for (unsigned j = 0; j < N; ++j) {
                    u64 s = 0;
                    for (unsigned a = 0; a < A; ++a)
                        s = addmod(s, mulmod(from_signed(y[a][j], q), c.dg_hat[dg][a][r], q), q);
                    x[j] = s;
                }
            }
            ntt_fwd(x, c.pr[r]);
            for (unsigned j = 0; j < N; ++j) {
                acc0[r][j] = addmod(acc0[r][j], mulmod(x[j], key.k0[dg][r][j], q), q);
                acc1[r][j] = addmod(acc1[r][j], mulmod(x[j], key.k1[dg][r][j], q), q);
            }
        }
    }
}

// ModDown: round(acc / P) over Q, NTT domain in and out.
void moddown(const orc_ctx& c, const std::vector<Poly>& acc, std::vector<Poly>& out) {
    const unsigned N = c.N, L = c.L, K = c.K;
    {
        std::vector<Poly> w(K);
        for (unsigned k = 0; k < K; ++k) { w[k] = acc[L + k]; ntt_inv(w[k], c.pr[L + k]); }
        out.assign(L, Poly(N));
        for (unsigned i = 0; i < L; ++i) {
            const u64 q = c.pr[i].q;
            Poly conv(N);
            for (unsigned j = 0; j < N; ++j) {
                u64 s = 0;
                for (unsigned k = 0; k < K; ++k) {
                    const u64 p = c.pr[L + k].q;
                    i64 z = centred(mulmod(w[k][j], c.phat_inv[k], p), p);
                    s = addmod(s, mulmod(from_signed(z, q), c.phat_mod_q[k][i], q), q);
                }
                conv[j] = s;
            }
            ntt_fwd(conv, c.pr[i]);
            for (unsigned j = 0; j < N; ++j)
                out[i][j] = mulmod(submod(acc[i][j], conv[j], q), c.P_inv_q[i], q);
        }
    }
}

// Hybrid key switching of a coefficient-domain polynomial d (L limbs, mod Q).
// Returns (u0, u1) over Q in the NTT domain.
void key_switch(orc_ctx& c, const std::vector<Poly>& d, u64 kid, std::vector<Poly>& u0,
                std::vector<Poly>& u1) {
    std::vector<Poly> acc0, acc1;
    ks_acc(c, d, kid, acc0, acc1);
    moddown(c, acc0, u0);
    moddown(c, acc1, u1);
}

struct Ct {
    std::vector<Poly> c0, c1;
};

Ct load(const orc_ctx& c, const uint64_t* buf) {
    Ct ct;
    ct.c0.resize(c.L); ct.c1.resize(c.L);
    for (unsigned i = 0; i < c.L; ++i) {
        ct.c0[i].assign(buf + (size_t)i * c.N, buf + (size_t)(i + 1) * c.N);
        ct.c1[i].assign(buf + (size_t)(c.L + i) * c.N, buf + (size_t)(c.L + i + 1) * c.N);
    }
    return ct;
}
void store(const orc_ctx& c, const Ct& ct, uint64_t* buf) {
    for (unsigned i = 0; i < c.L; ++i) {
        std::memcpy(buf + (size_t)i * c.N, ct.c0[i].data(), c.N * 8);
        std::memcpy(buf + (size_t)(c.L + i) * c.N, ct.c1[i].data(), c.N * 8);
    }
}

void check_segment(const orc_ctx& c, size_t S) {
    if (S == 0) throw std::invalid_argument("DimensionError: cannot encrypt an empty vector");
    if (S > c.N / 2)
        throw std::length_error("CapacityError: vector of length " + std::to_string(S) +
                                " exceeds " + std::to_string(c.N / 2) + " slots");
}

// batch encoding: row 0 <- values mod t (zero tail), row 1 <- 0, INTT mod t
Poly encode(const orc_ctx& c, const int64_t* v, size_t S) {
    Poly slots(c.N, 0);
    for (size_t i = 0; i < S; ++i) slots[c.slot_ntt[i]] = from_signed(v[i], kT);
    ntt_inv(slots, c.tp);
    return slots;
}

// encryption with given randomness: c0 = pk0 u + e0 + Delta m, c1 = pk1 u + e1
Ct encrypt_with(orc_ctx& c, const int64_t* v, size_t S, const std::vector<i64>& u, const std::vector<i64>& e0,
                const std::vector<i64>& e1);

Ct encrypt(orc_ctx& c, const int64_t* v, size_t S, u64 ctr) {
    const unsigned N = c.N;
    std::vector<i64> u(N), e0(N), e1(N);
    for (unsigned j = 0; j < N; ++j) {
        u[j] = ternary(c.seed, kStreamEncU | ctr, j);
        e0[j] = gauss(c.seed, kStreamEncE0 | ctr, j);
        e1[j] = gauss(c.seed, kStreamEncE1 | ctr, j);
    }
    return encrypt_with(c, v, S, u, e0, e1);
}

Ct encrypt_with(orc_ctx& c, const int64_t* v, size_t S, const std::vector<i64>& u, const std::vector<i64>& e0,
                const std::vector<i64>& e1) {
    const unsigned N = c.N;
    Poly m = encode(c, v, S);
    Ct ct;
    ct.c0.resize(c.L); ct.c1.resize(c.L);
    for (unsigned i = 0; i < c.L; ++i) {
        const u64 q = c.pr[i].q;
        Poly U = lift_signed(u, q), E0 = lift_signed(e0, q), E1 = lift_signed(e1, q);
        for (unsigned j = 0; j < N; ++j) E0[j] = addmod(E0[j], mulmod(c.delta[i], m[j], q), q);
        ntt_fwd(U, c.pr[i]); ntt_fwd(E0, c.pr[i]); ntt_fwd(E1, c.pr[i]);
        Poly a(N), b(N);
        for (unsigned j = 0; j < N; ++j) {
            a[j] = addmod(mulmod(c.pk0[i][j], U[j], q), E0[j], q);
            b[j] = addmod(mulmod(c.pk1[i][j], U[j], q), E1[j], q);
        }
        ct.c0[i] = std::move(a);
        ct.c1[i] = std::move(b);
    }
    return ct;
}

// phase x = c0 + c1 s in coefficient form; returns per-coefficient fixed-point
// t*x/Q (units 2^-64, taken mod 2^128)
std::vector<u128> scaled_phase(orc_ctx& c, const Ct& ct) {
    const unsigned N = c.N, L = c.L;
    std::vector<Poly> x(L);
    for (unsigned i = 0; i < L; ++i) {
        const u64 q = c.pr[i].q;
        x[i].resize(N);
        for (unsigned j = 0; j < N; ++j)
            x[i][j] = addmod(ct.c0[i][j], mulmod(ct.c1[i][j], c.s_ntt[i][j], q), q);
        ntt_inv(x[i], c.pr[i]);
    }
    std::vector<u128> S(N, 0);
    for (unsigned j = 0; j < N; ++j)
        for (unsigned i = 0; i < L; ++i)
            S[j] += fx_term(mulmod(x[i][j], c.qhat_inv[i], c.pr[i].q), c.t_over_q[i]);
    return S;
}

std::vector<i64> decrypt(orc_ctx& c, const Ct& ct, size_t S) {
    std::vector<u128> ph = scaled_phase(c, ct);
    Poly m(c.N);
    for (unsigned j = 0; j < c.N; ++j) m[j] = fx_round(ph[j]) % kT;
    ntt_fwd(m, c.tp);
    std::vector<i64> out(S);
    for (size_t i = 0; i < S; ++i) out[i] = (i64)m[c.slot_ntt[i]];
    return out;
}

Ct add(const orc_ctx& c, const Ct& a, const Ct& b) {
    Ct o = a;
    for (unsigned i = 0; i < c.L; ++i) {
        const u64 q = c.pr[i].q;
        for (unsigned j = 0; j < c.N; ++j) {
            o.c0[i][j] = addmod(a.c0[i][j], b.c0[i][j], q);
            o.c1[i][j] = addmod(a.c1[i][j], b.c1[i][j], q);
        }
    }
    return o;
}

// The batch-encoded mask, centred mod t, lifted to every prime of Q ++ P and
// NTT'd (cached by content).
std::shared_ptr<const std::vector<Poly>> mask_ntt(const orc_ctx& c, const int64_t* mask, size_t S) {
    std::vector<int64_t> key(mask, mask + S);
    {
        std::lock_guard<std::mutex> lk(c.mask_mu);
        auto it = c.masks.find(key);
        if (it != c.masks.end()) return it->second;
    }
    Poly m = encode(c, mask, S);
    auto out = std::make_shared<std::vector<Poly>>(c.R());
    for (unsigned r = 0; r < c.R(); ++r) {
        const u64 q = c.pr[r].q;
        Poly& mm = (*out)[r];
        mm.resize(c.N);
        for (unsigned j = 0; j < c.N; ++j) mm[j] = from_signed(centred(m[j], kT), q);
        ntt_fwd(mm, c.pr[r]);
    }
    std::lock_guard<std::mutex> lk(c.mask_mu);
    return c.masks.emplace(std::move(key), std::move(out)).first->second;
}

Ct cmult(const orc_ctx& c, const Ct& a, const int64_t* mask, size_t S) {
    const auto mp = mask_ntt(c, mask, S);
    Ct o = a;
    for (unsigned i = 0; i < c.L; ++i) {
        const u64 q = c.pr[i].q;
        const Poly& mm = (*mp)[i];
        for (unsigned j = 0; j < c.N; ++j) {
            o.c0[i][j] = mulmod(a.c0[i][j], mm[j], q);
            o.c1[i][j] = mulmod(a.c1[i][j], mm[j], q);
        }
    }
    return o;
}

// exact Q -> B conversion of a coefficient-domain polynomial (centred lift)
std::vector<Poly> q_to_b(const orc_ctx& c, const std::vector<Poly>& x) {
    const unsigned N = c.N, L = c.L, nB = c.nB;
    std::vector<Poly> out(nB, Poly(N));
    std::vector<u64> y(L);
    for (unsigned j = 0; j < N; ++j) {
        u128 S = 0;
        for (unsigned i = 0; i < L; ++i) {
            y[i] = mulmod(x[i][j], c.qhat_inv[i], c.pr[i].q);
            S += fx_term(y[i], c.one_over_q[i]);
        }
        const u64 v = fx_round(S);
        for (unsigned k = 0; k < nB; ++k) {
            const u64 b = c.pr[c.bidx(k)].q;
            u64 s = 0;
            for (unsigned i = 0; i < L; ++i) s = addmod(s, mulmod(y[i] % b, c.qhat_mod_b[i][k], b), b);
            out[k][j] = submod(s, mulmod(v % b, c.Q_mod_b[k], b), b);
        }
    }
    return out;
}

// round(t x / Q) for x given over Q ++ B (coefficient domain), result over Q
std::vector<Poly> scale_round(const orc_ctx& c, const std::vector<Poly>& xq,
                              const std::vector<Poly>& xb) {
    const unsigned N = c.N, L = c.L, nB = c.nB;
    std::vector<Poly> out(L, Poly(N));
    std::vector<u64> a(L), yb(nB), cb(nB);
    for (unsigned j = 0; j < N; ++j) {
        u128 S = 0;
        for (unsigned i = 0; i < L; ++i) {
            a[i] = mulmod(xq[i][j], c.dhat_inv[i], c.pr[i].q);
            S += fx_term(a[i], c.F[i]);
        }
        const u64 Rr = fx_round(S);
        for (unsigned k = 0; k < nB; ++k) {
            const u64 b = c.pr[c.bidx(k)].q;
            u64 s = Rr % b;
            for (unsigned i = 0; i < L; ++i) s = addmod(s, mulmod(a[i] % b, c.W[i][k], b), b);
            s = addmod(s, mulmod(xb[k][j], c.T[k], b), b);
            yb[k] = s;
        }
        // exact B -> Q
        u128 S2 = 0;
        for (unsigned k = 0; k < nB; ++k) {
            const u64 b = c.pr[c.bidx(k)].q;
            cb[k] = mulmod(yb[k], c.bhat_inv[k], b);
            S2 += fx_term(cb[k], c.one_over_b[k]);
        }
        const u64 v = fx_round(S2);
        for (unsigned i = 0; i < L; ++i) {
            const u64 q = c.pr[i].q;
            u64 s = 0;
            for (unsigned k = 0; k < nB; ++k) s = addmod(s, mulmod(cb[k] % q, c.bhat_mod_q[k][i], q), q);
            out[i][j] = submod(s, mulmod(v % q, c.B_mod_q[i], q), q);
        }
    }
    return out;
}

// Product of two ciphertexts BEFORE scale-and-round: the tensor
// (x0 y0, x0 y1 + x1 y0, x1 y1) of the exact centred lifts over Q ++ B, NTT
// domain (limbs: Q primes, then B primes).
struct Tensor {
    std::vector<Poly> t[3];  // each L + nB limbs
};
Tensor tensor_of(const orc_ctx& c, const Ct& x, const Ct& y) {
    const unsigned N = c.N, L = c.L, nB = c.nB;
    const std::vector<Poly>* in[4] = {&x.c0, &x.c1, &y.c0, &y.c1};
    std::vector<Poly> bext[4];
    for (int p = 0; p < 4; ++p) {
        std::vector<Poly> coeff = *in[p];
        for (unsigned i = 0; i < L; ++i) ntt_inv(coeff[i], c.pr[i]);
        bext[p] = q_to_b(c, coeff);
        for (unsigned k = 0; k < nB; ++k) ntt_fwd(bext[p][k], c.pr[c.bidx(k)]);
    }
    Tensor T;
    for (int t = 0; t < 3; ++t) T.t[t].assign(L + nB, Poly(N));
    auto tensor = [&](const Poly& a0, const Poly& a1, const Poly& b0, const Poly& b1, u64 q, unsigned r) {
        for (unsigned j = 0; j < N; ++j) {
            T.t[0][r][j] = mulmod(a0[j], b0[j], q);
            T.t[1][r][j] = addmod(mulmod(a0[j], b1[j], q), mulmod(a1[j], b0[j], q), q);
            T.t[2][r][j] = mulmod(a1[j], b1[j], q);
        }
    };
    for (unsigned i = 0; i < L; ++i) tensor(x.c0[i], x.c1[i], y.c0[i], y.c1[i], c.pr[i].q, i);
    for (unsigned k = 0; k < nB; ++k)
        tensor(bext[0][k], bext[1][k], bext[2][k], bext[3][k], c.pr[c.bidx(k)].q, L + k);
    return T;
}

// A ciphertext value has up to three parts, and its plain value is their sum:
//   X  a plain (c0, c1) over Q                         (always present, may be 0)
//   T  a PENDING PRODUCT: a sum of unscaled tensors over Q ++ B; its plain value
//      is round(t/Q * T) relinearised
//   A  a PENDING KEY SWITCH: a sum of key-switch accumulators over Q ++ P (NTT
//      domain) of rotations, P phi(c0) folded in; its plain value is ModDown(A)
// Semantics (the GPU library follows them exactly):
//   he_mult(x, y)  -> {T = tensor(plain(x), plain(y))}
//   he_rot(x, z)   -> {A = KS_g(phi(plain(x).c1)) + P phi(plain(x).c0)}  (z = 0: {X = plain(x)})
//   he_cmult(x, m) -> {X = m X, A = m A}; if x has T: {X = m plain(x)}
//   he_add(x, y)   -> partwise sum
//   decrypt, export, and every other reader use plain(x).
// A lone rotation or product materialises to exactly the eager result (ModDown
// of A + P y is ModDown(A) + y), while sums of products and masked sums of
// rotations are scaled, relinearised or moded down once instead of per term.
enum : int { kPartT = 1, kPartA = 2 };
struct XCt {
    Ct add;                  // X
    bool pending = false;    // T present
    Tensor T;
    bool ks = false;         // A present
    std::vector<Poly> A0, A1;  // R limbs each
    int kind() const { return (pending ? kPartT : 0) | (ks ? kPartA : 0); }
};

Ct zero_ct(const orc_ctx& c) {
    Ct z;
    z.c0.assign(c.L, Poly(c.N, 0));
    z.c1.assign(c.L, Poly(c.N, 0));
    return z;
}

Ct materialize(orc_ctx& c, const XCt& x) {
    const unsigned N = c.N, L = c.L, nB = c.nB;
    Ct o = x.add;
    if (x.pending) {
        std::vector<Poly> tq[3], tb[3];
        for (int t = 0; t < 3; ++t) {
            tq[t].assign(x.T.t[t].begin(), x.T.t[t].begin() + L);
            tb[t].assign(x.T.t[t].begin() + L, x.T.t[t].end());
            for (unsigned i = 0; i < L; ++i) ntt_inv(tq[t][i], c.pr[i]);
            for (unsigned k = 0; k < nB; ++k) ntt_inv(tb[t][k], c.pr[c.bidx(k)]);
        }
        std::vector<Poly> e0 = scale_round(c, tq[0], tb[0]);
        std::vector<Poly> e1 = scale_round(c, tq[1], tb[1]);
        std::vector<Poly> e2 = scale_round(c, tq[2], tb[2]);
        std::vector<Poly> u0, u1;
        key_switch(c, e2, 0, u0, u1);
        for (unsigned i = 0; i < L; ++i) {
            const u64 q = c.pr[i].q;
            ntt_fwd(e0[i], c.pr[i]); ntt_fwd(e1[i], c.pr[i]);
            for (unsigned j = 0; j < N; ++j) {
                o.c0[i][j] = addmod(addmod(e0[i][j], u0[i][j], q), o.c0[i][j], q);
                o.c1[i][j] = addmod(addmod(e1[i][j], u1[i][j], q), o.c1[i][j], q);
            }
        }
    }
    if (x.ks) {
        std::vector<Poly> m0, m1;
        moddown(c, x.A0, m0);
        moddown(c, x.A1, m1);
        for (unsigned i = 0; i < L; ++i) {
            const u64 q = c.pr[i].q;
            for (unsigned j = 0; j < N; ++j) {
                o.c0[i][j] = addmod(o.c0[i][j], m0[i][j], q);
                o.c1[i][j] = addmod(o.c1[i][j], m1[i][j], q);
            }
        }
    }
    return o;
}

XCt plain_x(const Ct& v) {
    XCt o;
    o.add = v;
    return o;
}

XCt mult_pending(const orc_ctx& c, const Ct& x, const Ct& y) {
    XCt o;
    o.pending = true;
    o.add = zero_ct(c);
    o.T = tensor_of(c, x, y);
    return o;
}

// rotation as a pending key switch (z = 0: the plain operand)
XCt rot_x(orc_ctx& c, const Ct& a, i64 z) {
    const i64 H = c.N / 2;
    const i64 zz = ((z % H) + H) % H;
    if (zz == 0) return plain_x(a);
    const u64 g = powmod(3, (u64)zz, 2 * (u64)c.N);
    std::vector<Poly> c0(c.L), c1(c.L);
    for (unsigned i = 0; i < c.L; ++i) {
        Poly t0 = a.c0[i], t1 = a.c1[i];
        ntt_inv(t0, c.pr[i]); ntt_inv(t1, c.pr[i]);
        c0[i] = automorph_coeff(t0, g, c.pr[i].q);
        c1[i] = automorph_coeff(t1, g, c.pr[i].q);
        ntt_fwd(c0[i], c.pr[i]);
    }
    XCt o;
    o.add = zero_ct(c);
    o.ks = true;
    ks_acc(c, c1, g, o.A0, o.A1);
    for (unsigned i = 0; i < c.L; ++i) {  // + P phi(c0): ModDown(A + P y) = ModDown(A) + y
        const u64 q = c.pr[i].q;
        for (unsigned j = 0; j < c.N; ++j) o.A0[i][j] = addmod(o.A0[i][j], mulmod(c.P_mod_r[i], c0[i][j], q), q);
    }
    return o;
}

// mask over Q ++ P (NTT domain) for masking pending key switches
std::vector<Poly> mask_qp(const orc_ctx& c, const int64_t* mask, size_t S) { return *mask_ntt(c, mask, S); }

XCt cmult_x(orc_ctx& c, const XCt& v, const int64_t* mask, size_t S) {
    XCt o;
    if (v.pending) {  // a pending product is materialised (with every other part) first
        o.add = cmult(c, materialize(c, v), mask, S);
        return o;
    }
    o.add = cmult(c, v.add, mask, S);
    if (v.ks) {
        const std::vector<Poly> m = mask_qp(c, mask, S);
        o.ks = true;
        o.A0 = v.A0;
        o.A1 = v.A1;
        for (unsigned r = 0; r < c.R(); ++r) {
            const u64 q = c.pr[r].q;
            for (unsigned j = 0; j < c.N; ++j) {
                o.A0[r][j] = mulmod(o.A0[r][j], m[r][j], q);
                o.A1[r][j] = mulmod(o.A1[r][j], m[r][j], q);
            }
        }
    }
    return o;
}

XCt add_any(const orc_ctx& c, const XCt& a, const XCt& b) {
    XCt o;
    o.add = add(c, a.add, b.add);
    o.pending = a.pending || b.pending;
    if (o.pending) {
        const unsigned L = c.L, D = c.L + c.nB;
        const XCt& p = a.pending ? a : b;
        o.T = p.T;
        if (a.pending && b.pending)
            for (int t = 0; t < 3; ++t)
                for (unsigned r = 0; r < D; ++r) {
                    const u64 q = r < L ? c.pr[r].q : c.pr[c.bidx(r - L)].q;
                    for (unsigned j = 0; j < c.N; ++j) o.T.t[t][r][j] = addmod(a.T.t[t][r][j], b.T.t[t][r][j], q);
                }
    }
    o.ks = a.ks || b.ks;
    if (o.ks) {
        const XCt& p = a.ks ? a : b;
        o.A0 = p.A0;
        o.A1 = p.A1;
        if (a.ks && b.ks)
            for (unsigned r = 0; r < c.R(); ++r) {
                const u64 q = c.pr[r].q;
                for (unsigned j = 0; j < c.N; ++j) {
                    o.A0[r][j] = addmod(a.A0[r][j], b.A0[r][j], q);
                    o.A1[r][j] = addmod(a.A1[r][j], b.A1[r][j], q);
                }
            }
    }
    return o;
}

// Eager product / rotation (a pending value materialised at once).
Ct mult(orc_ctx& c, const Ct& x, const Ct& y) { return materialize(c, mult_pending(c, x, y)); }
Ct rot(orc_ctx& c, const Ct& a, i64 z) { return materialize(c, rot_x(c, a, z)); }

// value buffer: [X: 2 L N][T: 3 (L + nB) N, if kind & 1][A: 2 R N, if kind & 2]
size_t pending_words(const orc_ctx& c) {
    return (size_t)2 * c.L * c.N + (size_t)3 * (c.L + c.nB) * c.N + (size_t)2 * c.R() * c.N;
}
size_t kind_words(const orc_ctx& c, int kind) {
    return (size_t)2 * c.L * c.N + ((kind & kPartT) ? (size_t)3 * (c.L + c.nB) * c.N : 0) +
           ((kind & kPartA) ? (size_t)2 * c.R() * c.N : 0);
}
XCt load_x(const orc_ctx& c, const uint64_t* buf, int kind) {
    XCt x;
    x.add = load(c, buf);
    x.pending = (kind & kPartT) != 0;
    x.ks = (kind & kPartA) != 0;
    const unsigned D = c.L + c.nB, R = c.R();
    const uint64_t* t = buf + (size_t)2 * c.L * c.N;
    if (x.pending)
        for (int k = 0; k < 3; ++k) {
            x.T.t[k].resize(D);
            for (unsigned r = 0; r < D; ++r) {
                const uint64_t* p = t + ((size_t)k * D + r) * c.N;
                x.T.t[k][r].assign(p, p + c.N);
            }
        }
    const uint64_t* a = t + (x.pending ? (size_t)3 * D * c.N : 0);
    if (x.ks) {
        x.A0.resize(R);
        x.A1.resize(R);
        for (unsigned r = 0; r < R; ++r) {
            x.A0[r].assign(a + (size_t)r * c.N, a + (size_t)(r + 1) * c.N);
            x.A1[r].assign(a + (size_t)(R + r) * c.N, a + (size_t)(R + r + 1) * c.N);
        }
    }
    return x;
}
void store_x(const orc_ctx& c, const XCt& x, uint64_t* buf) {
    store(c, x.add, buf);
    if (!x.pending && !x.ks) return;
    const unsigned D = c.L + c.nB, R = c.R();
    uint64_t* t = buf + (size_t)2 * c.L * c.N;
    if (x.pending)
        for (int k = 0; k < 3; ++k)
            for (unsigned r = 0; r < D; ++r) std::memcpy(t + ((size_t)k * D + r) * c.N, x.T.t[k][r].data(), c.N * 8);
    uint64_t* a = t + (x.pending ? (size_t)3 * D * c.N : 0);
    if (x.ks)
        for (unsigned r = 0; r < R; ++r) {
            std::memcpy(a + (size_t)r * c.N, x.A0[r].data(), c.N * 8);
            std::memcpy(a + (size_t)(R + r) * c.N, x.A1[r].data(), c.N * 8);
        }
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::length_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

}  // namespace

extern "C" {

orc_ctx* orc_create(int param_id, uint64_t seed) {
    auto c = std::make_unique<orc_ctx>();
    c->seed = seed;
    try {
        build(*c, param_id);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
    return c.release();
}
void orc_destroy(orc_ctx* c) { delete c; }
const char* orc_last_error(void) { return g_err.c_str(); }

int orc_info(const orc_ctx* c, uint64_t* info, size_t cap) {
    const size_t need = 8 + c->pr.size();
    if (cap < need) return 1;
    info[0] = c->N; info[1] = c->L; info[2] = c->K; info[3] = c->nB; info[4] = c->dnum;
    info[5] = kT; info[6] = c->alpha; info[7] = c->seed;
    for (size_t i = 0; i < c->pr.size(); ++i) info[8 + i] = c->pr[i].q;
    return 0;
}
size_t orc_ct_words(const orc_ctx* c) { return (size_t)2 * c->L * c->N; }

int orc_encrypt(orc_ctx* c, const int64_t* values, size_t S, uint64_t counter, uint64_t* out) {
    return guarded([&] { check_segment(*c, S); store(*c, encrypt(*c, values, S, counter), out); });
}
int orc_decrypt(orc_ctx* c, const uint64_t* ct, size_t S, int64_t* out) {
    return guarded([&] {
        check_segment(*c, S);
        auto v = decrypt(*c, load(*c, ct), S);
        std::memcpy(out, v.data(), S * 8);
    });
}
int orc_add(orc_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out) {
    return guarded([&] { store(*c, add(*c, load(*c, a), load(*c, b)), out); });
}
int orc_cmult(orc_ctx* c, const uint64_t* a, const int64_t* mask, size_t S, uint64_t* out) {
    return guarded([&] { check_segment(*c, S); store(*c, cmult(*c, load(*c, a), mask, S), out); });
}
int orc_rot(orc_ctx* c, const uint64_t* a, int64_t z, uint64_t* out) {
    return guarded([&] { store(*c, rot(*c, load(*c, a), z), out); });
}
int orc_mult(orc_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out) {
    return guarded([&] { store(*c, mult(*c, load(*c, a), load(*c, b)), out); });
}
size_t orc_pending_words(const orc_ctx* c) { return pending_words(*c); }
size_t orc_kind_words(const orc_ctx* c, int kind) { return kind_words(*c, kind); }
int orc_mult_pending(orc_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out) {
    return guarded([&] { store_x(*c, mult_pending(*c, load(*c, a), load(*c, b)), out); });
}
int orc_add_any(orc_ctx* c, const uint64_t* a, int a_kind, const uint64_t* b, int b_kind, uint64_t* out) {
    return guarded([&] { store_x(*c, add_any(*c, load_x(*c, a, a_kind), load_x(*c, b, b_kind)), out); });
}
int orc_rot_x(orc_ctx* c, const uint64_t* a, int64_t z, uint64_t* out, int* out_kind) {
    return guarded([&] {
        const XCt x = rot_x(*c, load(*c, a), z);
        store_x(*c, x, out);
        *out_kind = x.kind();
    });
}
int orc_cmult_x(orc_ctx* c, const uint64_t* a, int a_kind, const int64_t* mask, size_t S, uint64_t* out,
                int* out_kind) {
    return guarded([&] {
        check_segment(*c, S);
        const XCt x = cmult_x(*c, load_x(*c, a, a_kind), mask, S);
        store_x(*c, x, out);
        *out_kind = x.kind();
    });
}
int orc_materialize_kind(orc_ctx* c, const uint64_t* x, int kind, uint64_t* out) {
    return guarded([&] { store(*c, materialize(*c, load_x(*c, x, kind)), out); });
}
int orc_materialize(orc_ctx* c, const uint64_t* x, uint64_t* out) { return orc_materialize_kind(c, x, kPartT, out); }

double orc_noise_budget(orc_ctx* c, const uint64_t* ct) {
    std::vector<u128> ph = scaled_phase(*c, load(*c, ct));
    u64 worst = 0;
    for (u128 s : ph) {
        u64 frac = (u64)s;  // fractional part in units of 2^-64
        u64 dist = frac >= (1ULL << 63) ? (u64)(0 - frac) : frac;
        if (dist > worst) worst = dist;
    }
    if (worst == 0) return 64.0;
    // v = worst / 2^64 ; budget = -log2(2 v)
    double v = (double)worst / 18446744073709551616.0;
    return -__builtin_log2(2.0 * v);
}

int orc_ntt_fwd(orc_ctx* c, int r, uint64_t* a) {
    return guarded([&] {
        const Prime& P = r < 0 ? c->tp : c->pr.at(r);
        Poly v(a, a + c->N);
        ntt_fwd(v, P);
        std::memcpy(a, v.data(), c->N * 8);
    });
}
int orc_ntt_inv(orc_ctx* c, int r, uint64_t* a) {
    return guarded([&] {
        const Prime& P = r < 0 ? c->tp : c->pr.at(r);
        Poly v(a, a + c->N);
        ntt_inv(v, P);
        std::memcpy(a, v.data(), c->N * 8);
    });
}
int orc_encode(orc_ctx* c, const int64_t* values, size_t S, uint64_t* m_out) {
    return guarded([&] {
        check_segment(*c, S);
        Poly m = encode(*c, values, S);
        std::memcpy(m_out, m.data(), c->N * 8);
    });
}
size_t orc_key_words(const orc_ctx* c, int kind) {
    switch (kind) {
        case 0: return (size_t)c->R() * c->N;
        case 1: return (size_t)2 * c->L * c->N;
        case 2: return (size_t)c->dnum * 2 * c->R() * c->N;
        default: return 0;
    }
}

int orc_key_export(orc_ctx* c, int kind, uint32_t elt, uint64_t* w) {
    return guarded([&] {
        const size_t N = c->N;
        if (kind == 0) {
            for (unsigned r = 0; r < c->R(); ++r) std::memcpy(w + r * N, c->s_ntt[r].data(), N * 8);
        } else if (kind == 1) {
            for (unsigned i = 0; i < c->L; ++i) {
                std::memcpy(w + i * N, c->pk0[i].data(), N * 8);
                std::memcpy(w + (c->L + i) * N, c->pk1[i].data(), N * 8);
            }
        } else if (kind == 2) {
            const KsKey& k = get_key(*c, elt);
            const unsigned R = c->R();
            for (unsigned d = 0; d < c->dnum; ++d)
                for (unsigned r = 0; r < R; ++r) {
                    std::memcpy(w + (((size_t)d * 2 + 0) * R + r) * N, k.k0[d][r].data(), N * 8);
                    std::memcpy(w + (((size_t)d * 2 + 1) * R + r) * N, k.k1[d][r].data(), N * 8);
                }
        } else {
            throw std::invalid_argument("key kind");
        }
    });
}

// Installs key material produced elsewhere (the layouts of orc_key_export).
// An imported secret key also replaces the coefficient form the oracle derives
// Galois and relinearisation keys from (centred INTT of its first limb).
int orc_key_import(orc_ctx* c, int kind, uint32_t elt, const uint64_t* w) {
    return guarded([&] {
        const size_t N = c->N;
        if (kind == 0) {
            for (unsigned r = 0; r < c->R(); ++r) c->s_ntt[r].assign(w + r * N, w + (r + 1) * N);
            Poly s0 = c->s_ntt[0];
            ntt_inv(s0, c->pr[0]);
            const u64 q = c->pr[0].q;
            for (size_t j = 0; j < N; ++j) c->s_coeff[j] = s0[j] > q / 2 ? -(i64)(q - s0[j]) : (i64)s0[j];
            c->keys.clear();  // keys derived from the old secret
        } else if (kind == 1) {
            for (unsigned i = 0; i < c->L; ++i) {
                c->pk0[i].assign(w + i * N, w + (i + 1) * N);
                c->pk1[i].assign(w + (c->L + i) * N, w + (c->L + i + 1) * N);
            }
        } else if (kind == 2) {
            const unsigned R = c->R();
            auto k = std::make_unique<KsKey>();
            k->k0.assign(c->dnum, std::vector<Poly>(R));
            k->k1.assign(c->dnum, std::vector<Poly>(R));
            for (unsigned d = 0; d < c->dnum; ++d)
                for (unsigned r = 0; r < R; ++r) {
                    const uint64_t* a = w + (((size_t)d * 2 + 0) * R + r) * N;
                    const uint64_t* b = w + (((size_t)d * 2 + 1) * R + r) * N;
                    k->k0[d][r].assign(a, a + N);
                    k->k1[d][r].assign(b, b + N);
                }
            c->keys[elt] = std::move(k);
        } else {
            throw std::invalid_argument("key kind");
        }
    });
}

int orc_encrypt_noise(orc_ctx* c, const int64_t* values, size_t S, const int64_t* u, const int64_t* e0,
                      const int64_t* e1, uint64_t* out) {
    return guarded([&] {
        check_segment(*c, S);
        const size_t N = c->N;
        std::vector<i64> U(u, u + N), E0(e0, e0 + N), E1(e1, e1 + N);
        store(*c, encrypt_with(*c, values, S, U, E0, E1), out);
    });
}

uint64_t orc_prng(uint64_t seed, uint64_t stream, uint64_t idx) { return prng(seed, stream, idx); }
int64_t orc_gauss(uint64_t seed, uint64_t stream, uint64_t idx) { return gauss(seed, stream, idx); }

}  // extern "C"
