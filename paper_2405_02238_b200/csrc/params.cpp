// params.cpp -- prime selection, NTT tables and RNS conversion constants.
//
// Selection rules (shared, by specification, with oracle/bfv_oracle.cpp):
//  * primes are taken in descending order q = 2^bits - k*2^32 + 1, k = 1, 2, ...
//    (q = 1 mod 2^32: NTT-friendly for every N here, and q's low word is 1, so
//    every quotient-times-q product on the device is one 32-bit IMAD);
//    first L for Q, next K for P, next nB for the auxiliary base B;
//  * psi = x^((q-1)/2N) for the smallest x >= 2 with psi^N = -1;
//  * the NTT is negacyclic, natural order in, bit-reversed order out, so the
//    output index k holds the evaluation at psi^(2 brv(k) + 1);
//  * slot (row r, column i) sits at the NTT index of the exponent 3^i (row 0)
//    or -3^i (row 1) mod 2N, which makes X -> X^(3^z) a left rotation by z of
//    each N/2-slot row (reference he_rot, proj/src/backend.cpp:185-197).
#include "params.hpp"

#include <stdexcept>

namespace hgm {

namespace {

using u128 = unsigned __int128;

u64 mulmod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
u64 powmod(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    for (; e; e >>= 1) {
        if (e & 1) r = mulmod(r, a, q);
        a = mulmod(a, a, q);
    }
    return r;
}
u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }
u64 shoup_of(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }

bool is_prime(u64 n) {
    static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (u64 p : bases)
        if (n % p == 0) return n == p;
    u64 d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; ++s; }
    for (u64 a : bases) {
        u64 x = powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool composite = true;
        for (int r = 1; r < s && composite; ++r) {
            x = mulmod(x, x, n);
            if (x == n - 1) composite = false;
        }
        if (composite) return false;
    }
    return true;
}

u32 bitrev(u32 x, u32 bits) {
    u32 r = 0;
    for (u32 i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1);
    return r;
}

Frac frac_of(u64 a, u64 q) {
    u128 num = (u128)a << 64;
    Frac f;
    f.hi = (u64)(num / q);
    u64 rem = (u64)(num % q);
    f.lo = (u64)(((u128)rem << 64) / q);
    return f;
}

Prime prime_of(u64 q, unsigned N) {
    Prime p{};
    p.q = q;
    p.s = 64 - __builtin_clzll(q);
    p.mu = (u64)(((u128)1 << (62 + p.s)) / q);
    // ntt.cu Canon: x < 16q is canonicalised as x - floor(x / 2^s) q, then one
    // conditional subtraction; that needs 16 (2^s - q) < q (t = 65537 has its own kernel)
    if (q != kT && (p.s < 33 || (((u128)1 << p.s) - q) * 16 >= q))
        throw std::invalid_argument("prime too far below a power of two for the table reduction");
    p.ninv = invmod(N % q, q);
    p.ninv_sh = shoup_of(p.ninv, q);
    return p;
}

const ParamSpec kSpecs[] = {{13, 60, 3, 1, 3, 4}, {15, 55, 8, 4, 2, 9}, {12, 60, 3, 1, 3, 4}};

}  // namespace

const u64 kGaussCdt[20] = {
    0x0ff52b40a5917e80ULL, 0x2e5a25d4bf0e3e00ULL, 0x489ae26955b04800ULL, 0x5d2bc20f621bf000ULL,
    0x6bc8694c3cc81000ULL, 0x7532d89ac6ba8000ULL, 0x7ab396cb74436c00ULL, 0x7d9e4e916643f000ULL,
    0x7f05495819eb2400ULL, 0x7fa1ce9c0039ac00ULL, 0x7fdfb3f212e8c800ULL, 0x7ff5e6f9d2315400ULL,
    0x7ffd1f97bc440c00ULL, 0x7fff40fa0088d800ULL, 0x7fffd2e835e1cc00ULL, 0x7ffff65243870400ULL,
    0x7ffffe1db476a400ULL, 0x7fffffac0a1dd000ULL, 0x7ffffff428673c00ULL, 0x8000000000000000ULL};

const ParamSpec& param_spec(int id) {
    if (id < 0 || id > 2) throw std::invalid_argument("unknown parameter set " + std::to_string(id));
    return kSpecs[id];
}

HostParams make_params(int id, u64 seed) {
    HostParams h;
    h.spec = param_spec(id);
    h.id = id;
    h.seed = seed;
    h.logN = h.spec.logN;
    h.N = 1u << h.logN;
    h.L = h.spec.L;
    h.K = h.spec.K;
    h.nB = h.spec.nB;
    h.dnum = h.spec.dnum;
    h.alpha = h.L / h.dnum;
    h.R = h.L + h.K;
    const unsigned N = h.N, L = h.L, K = h.K, nB = h.nB, R = h.R, A = h.alpha;
    const unsigned total = L + K + nB;
    for (u64 k = 1; h.primes.size() < total; ++k) {
        const u64 c = (1ULL << h.spec.qbits) - (k << 32) + 1;  // = 1 mod 2^32, hence mod 2N
        if (is_prime(c)) h.primes.push_back(c);
    }
    // the device reductions compute quotient * q as x + (x_lo c) 2^32 (common.cuh mul_lo_q)
    for (u64 q : h.primes)
        if ((u32)q != 1u) throw std::logic_error("ciphertext primes must be 1 mod 2^32");
    // the lazy NTT butterflies keep values below 16q and the column accumulator
    // splits residues into two digits of at most 30 bits: both need q < 2^60
    for (u64 q : h.primes)
        if (q >> 60) throw std::logic_error("prime above 2^60 breaks the lazy NTT / digit bounds");
    // tables: slot t lives at kTIndex
    h.tw.assign((size_t)(kMaxPrimes + 1) * 4 * N, 0);
    auto fill = [&](unsigned slot, u64 q) {
        u64 psi = 0;
        for (u64 x = 2;; ++x) {
            psi = powmod(x, (q - 1) / (2 * N), q);
            if (powmod(psi, N, q) == q - 1) break;
        }
        h.psi.push_back(psi);
        const u64 ipsi = invmod(psi, q);
        u64* base = h.tw.data() + (size_t)slot * 4 * N;
        // interleaved Shoup pairs: [2i] = w, [2i+1] = w' (forward), then the inverse at +2N
        for (u32 i = 0; i < N; ++i) {
            const u32 e = bitrev(i, h.logN);
            base[2 * i] = powmod(psi, e, q);
            base[2 * i + 1] = shoup_of(base[2 * i], q);
            base[2 * N + 2 * i] = powmod(ipsi, e, q);
            base[2 * N + 2 * i + 1] = shoup_of(base[2 * N + 2 * i], q);
        }
    };
    for (unsigned r = 0; r < total; ++r) fill(r, h.primes[r]);
    fill(kTIndex, kT);

    h.slot_ntt.resize(N);
    u64 ex = 1;
    for (u32 i = 0; i < N / 2; ++i) {
        h.slot_ntt[i] = bitrev((u32)((ex - 1) / 2), h.logN);
        const u64 ex2 = 2 * (u64)N - ex;
        h.slot_ntt[N / 2 + i] = bitrev((u32)((ex2 - 1) / 2), h.logN);
        ex = ex * 3 % (2 * (u64)N);
    }

    DevParams& d = h.dev;
    d.N = N; d.logN = h.logN; d.L = L; d.K = K; d.nB = nB; d.dnum = h.dnum; d.alpha = A; d.R = R;
    d.seed = seed;
    for (unsigned r = 0; r < total; ++r) d.pr[r] = prime_of(h.primes[r], N);
    d.pr[kTIndex] = prime_of(kT, N);

    auto qv = [&](unsigned i) { return h.primes[i]; };
    auto bv = [&](unsigned j) { return h.primes[L + K + j]; };
    auto prod_mod = [&](const std::vector<u64>& xs, u64 m) {
        u64 r = 1 % m;
        for (u64 x : xs) r = mulmod(r, x % m, m);
        return r;
    };
    std::vector<u64> Qs(h.primes.begin(), h.primes.begin() + L);
    std::vector<u64> Ps(h.primes.begin() + L, h.primes.begin() + L + K);
    std::vector<u64> Bs(h.primes.begin() + L + K, h.primes.end());
    auto without = [](std::vector<u64> v, size_t i) { v.erase(v.begin() + i); return v; };

    const u64 Q_mod_t = prod_mod(Qs, kT);
    for (unsigned i = 0; i < L; ++i) {
        const u64 q = qv(i);
        const u64 qhat = prod_mod(without(Qs, i), q);
        d.qhat_inv[i] = invmod(qhat, q);
        d.qhat_inv_sh[i] = shoup_of(d.qhat_inv[i], q);
        d.delta[i] = mulmod((q - Q_mod_t % q) % q, invmod(kT % q, q), q);
        d.delta_sh[i] = shoup_of(d.delta[i], q);
        d.t_over_q[i] = frac_of(kT, q);
        d.one_over_q[i] = frac_of(1, q);
        const u64 Bq = prod_mod(Bs, q);
        d.dhat_inv[i] = invmod(mulmod(qhat, Bq, q), q);
        d.dhat_inv_sh[i] = shoup_of(d.dhat_inv[i], q);
        const u64 tB = mulmod(kT % q, Bq, q);
        d.F[i] = frac_of(tB, q);
        for (unsigned j = 0; j < nB; ++j) {
            const u64 b = bv(j);
            d.W[i][j] = mulmod((b - tB % b) % b, invmod(q % b, b), b);
            d.W_sh[i][j] = shoup_of(d.W[i][j], b);
            d.qhat_mod_b[i][j] = prod_mod(without(Qs, i), b);
            d.qhat_mod_b_sh[i][j] = shoup_of(d.qhat_mod_b[i][j], b);
            {  // digit width of the kernels' shape for this set (bfv.cu: L = 3 -> ShapeQ3, else ShapeQ8)
                const unsigned S = L == 3 ? 30 : 28;
                const u64 v = d.qhat_mod_b[i][j];
                d.qhat_mod_b_pk[i][j] = (v & ((1ULL << S) - 1)) | ((v >> S) << 32);
            }
        }
        d.B_mod_q[i] = Bq;
        d.B_mod_q_sh[i] = shoup_of(Bq, q);
        d.neg_B_mod_q[i] = (q - Bq) % q;
        const u64 Pq = prod_mod(Ps, q);
        d.P_mod_q[i] = Pq;
        d.P_mod_q_sh[i] = shoup_of(Pq, q);
        d.P_inv_q[i] = invmod(Pq, q);
        d.P_inv_q_sh[i] = shoup_of(d.P_inv_q[i], q);
    }
    for (unsigned j = 0; j < nB; ++j) {
        const u64 b = bv(j);
        d.Q_mod_b[j] = prod_mod(Qs, b);
        d.Q_mod_b_sh[j] = shoup_of(d.Q_mod_b[j], b);
        d.neg_Q_mod_b[j] = (b - d.Q_mod_b[j]) % b;
        d.T[j] = mulmod(kT % b, invmod(d.Q_mod_b[j], b), b);
        d.T_sh[j] = shoup_of(d.T[j], b);
        d.bhat_inv[j] = invmod(prod_mod(without(Bs, j), b), b);
        d.bhat_inv_sh[j] = shoup_of(d.bhat_inv[j], b);
        d.one_over_b[j] = frac_of(1, b);
        for (unsigned i = 0; i < L; ++i) {
            const u64 q = qv(i);
            d.bhat_mod_q[j][i] = prod_mod(without(Bs, j), q);
            d.bhat_mod_q_sh[j][i] = shoup_of(d.bhat_mod_q[j][i], q);
        }
    }
    for (unsigned dg = 0; dg < h.dnum; ++dg) {
        std::vector<u64> digit(Qs.begin() + dg * A, Qs.begin() + (dg + 1) * A);
        for (unsigned a = 0; a < A; ++a) {
            const unsigned i = dg * A + a;
            const u64 q = qv(i);
            d.dg_hat_inv[i] = invmod(prod_mod(without(digit, a), q), q);
            d.dg_hat_inv_sh[i] = shoup_of(d.dg_hat_inv[i], q);
            for (unsigned r = 0; r < R; ++r) {
                const u64 m = h.primes[r];
                d.dg_hat[i][r] = prod_mod(without(digit, a), m);
                d.dg_hat_sh[i][r] = shoup_of(d.dg_hat[i][r], m);
            }
        }
    }
    for (unsigned k = 0; k < K; ++k) {
        const u64 p = h.primes[L + k];
        d.phat_inv[k] = invmod(prod_mod(without(Ps, k), p), p);
        d.phat_inv_sh[k] = shoup_of(d.phat_inv[k], p);
        for (unsigned i = 0; i < L; ++i) {
            const u64 q = qv(i);
            d.phat_mod_q[k][i] = prod_mod(without(Ps, k), q);
            d.phat_mod_q_sh[k][i] = shoup_of(d.phat_mod_q[k][i], q);
        }
    }
    // fx_add_small: the reciprocals' integer parts fit 32 bits
    for (unsigned i = 0; i < L; ++i)
        if (d.one_over_q[i].hi >> 32) throw std::logic_error("1/q integer part above 2^32");
    for (unsigned j = 0; j < nB; ++j)
        if (d.one_over_b[j].hi >> 32) throw std::logic_error("1/b integer part above 2^32");
    // N^-1 folded into the first multiplier of each unscaled-INTT consumer
    auto with_ninv = [&](u64 c, unsigned r) { return mulmod(c, d.pr[r].ninv, h.primes[r]); };
    for (unsigned i = 0; i < L; ++i) {
        d.qhat_inv_n[i] = with_ninv(d.qhat_inv[i], i);
        d.qhat_inv_n_sh[i] = shoup_of(d.qhat_inv_n[i], qv(i));
        d.dhat_inv_n[i] = with_ninv(d.dhat_inv[i], i);
        d.dhat_inv_n_sh[i] = shoup_of(d.dhat_inv_n[i], qv(i));
    }
    for (unsigned j = 0; j < nB; ++j) d.T_n[j] = with_ninv(d.T[j], L + K + j);
    for (unsigned i = 0; i < L; ++i) {
        d.dg_hat_inv_n[i] = with_ninv(d.dg_hat_inv[i], i);
        d.dg_hat_inv_n_sh[i] = shoup_of(d.dg_hat_inv_n[i], qv(i));
    }
    for (unsigned k = 0; k < K; ++k) {
        d.phat_inv_n[k] = with_ninv(d.phat_inv[k], L + k);
        d.phat_inv_n_sh[k] = shoup_of(d.phat_inv_n[k], h.primes[L + k]);
    }
    return h;
}

}  // namespace hgm
