// common.cuh -- integer arithmetic and the device-side parameter block.
//
// All ciphertext arithmetic is 64-bit RNS modular arithmetic over NTT-friendly
// primes q = c 2^32 + 1 < 2^60.  Fixed multiplicands (twiddles, base-conversion constants)
// use Shoup's precomputed quotient; products of two variables use a shifted
// Barrett reduction.  Nothing here is floating point: the scale-and-round steps
// use 128-bit fixed-point fractions (see Frac) so that every result is an exact
// integer function of its inputs and matches oracle/bfv_oracle.cpp bit for bit.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define HD __host__ __device__ __forceinline__
#else
#define HD inline
#endif

namespace hgm {

using u64 = std::uint64_t;
using u32 = std::uint32_t;
using i64 = std::int64_t;

constexpr int kMaxL = 8;       // ciphertext primes
constexpr int kMaxK = 4;       // special primes
constexpr int kMaxB = 10;      // auxiliary base for the tensor product
constexpr int kMaxR = kMaxL + kMaxK;
constexpr int kMaxPrimes = kMaxL + kMaxK + kMaxB;
constexpr int kTIndex = kMaxPrimes;  // table slot of the plaintext modulus t
constexpr u64 kT = 65537;

// sampler stream tags: identical to oracle/bfv_oracle.cpp
constexpr u64 kStreamSk = 1ULL << 56, kStreamPkA = 2ULL << 56, kStreamPkE = 3ULL << 56,
              kStreamKsA = 4ULL << 56, kStreamKsE = 5ULL << 56, kStreamEncU = 6ULL << 56,
              kStreamEncE0 = 7ULL << 56, kStreamEncE1 = 8ULL << 56;

struct Frac {
    u64 hi, lo;  // floor(a * 2^128 / q) for a < q
};

struct Prime {
    u64 q;
    u64 mu;      // floor(2^(62+s) / q), shifted Barrett
    u32 s;       // bit length of q
    u32 pad;
    u64 ninv, ninv_sh;
};

// Everything a kernel needs, stored once in device memory per context and
// passed by pointer (uniform loads through the constant/L1 path).
struct DevParams {
    u32 N, logN, L, K, nB, dnum, alpha, R;  // R = L + K
    u64 seed;
    Prime pr[kMaxPrimes + 1];  // Q ++ P ++ B, then t at kTIndex
    const u64* tw;             // [(kMaxPrimes+1)][4][N]: psi_rev, sh, ipsi_rev, sh
    const u32* slot_ntt;       // slot (row*N/2+col) -> NTT index, N entries
    const u64* cdt;            // 20-entry Gaussian CDT
    // encrypt / decrypt
    u64 delta[kMaxL], delta_sh[kMaxL];
    u64 qhat_inv[kMaxL], qhat_inv_sh[kMaxL];  // (Q/q_i)^-1 mod q_i
    Frac t_over_q[kMaxL];
    // exact Q -> B
    Frac one_over_q[kMaxL];
    u64 qhat_mod_b[kMaxL][kMaxB], qhat_mod_b_sh[kMaxL][kMaxB];
    u64 qhat_mod_b_pk[kMaxL][kMaxB];  // packed digits (l | h << 32) at the set's digit width
    u64 Q_mod_b[kMaxB], Q_mod_b_sh[kMaxB];
    u64 neg_Q_mod_b[kMaxB];  // b_j - (Q mod b_j)
    // scale-and-round Q++B -> B
    u64 dhat_inv[kMaxL], dhat_inv_sh[kMaxL];
    u64 W[kMaxL][kMaxB], W_sh[kMaxL][kMaxB];
    Frac F[kMaxL];
    u64 T[kMaxB], T_sh[kMaxB];
    // exact B -> Q
    u64 bhat_inv[kMaxB], bhat_inv_sh[kMaxB];
    Frac one_over_b[kMaxB];
    u64 bhat_mod_q[kMaxB][kMaxL], bhat_mod_q_sh[kMaxB][kMaxL];
    u64 B_mod_q[kMaxL], B_mod_q_sh[kMaxL];
    u64 neg_B_mod_q[kMaxL];  // q_i - (B mod q_i)
    // key switching (digit d holds primes d*alpha .. d*alpha+alpha-1)
    u64 dg_hat_inv[kMaxL], dg_hat_inv_sh[kMaxL];               // by prime i
    u64 dg_hat[kMaxL][kMaxR], dg_hat_sh[kMaxL][kMaxR];         // [i][r] (Q_d/q_i) mod r
    u64 P_mod_q[kMaxL], P_mod_q_sh[kMaxL];
    u64 P_inv_q[kMaxL], P_inv_q_sh[kMaxL];
    u64 phat_inv[kMaxK], phat_inv_sh[kMaxK];
    u64 phat_mod_q[kMaxK][kMaxL], phat_mod_q_sh[kMaxK][kMaxL];
    // the same with N^-1 folded in, for inputs from unscaled INTTs (NttJobs::unscaled)
    u64 qhat_inv_n[kMaxL], qhat_inv_n_sh[kMaxL];
    u64 dhat_inv_n[kMaxL], dhat_inv_n_sh[kMaxL];
    u64 T_n[kMaxB];
    u64 phat_inv_n[kMaxK], phat_inv_n_sh[kMaxK];
    u64 dg_hat_inv_n[kMaxL], dg_hat_inv_n_sh[kMaxL];
};

// Per-context values passed by value to every kernel (the parameter-set
// constants live in __constant__ memory, one slot per set, see kParamSets).
constexpr int kParamSets = 3;
struct DevCtx {
    const u64* tw;        // twiddle tables of this context
    const u32* slot_ntt;  // slot -> NTT index
    const u64* cdt;       // Gaussian CDT
    u64 seed;
    u32 pid;              // parameter-set slot in c_dp
    u32 csprng;           // 1: keys and noise from ChaCha (OS-seeded sessions), 0: the parity PRF
    u32 ck[8];            // ChaCha key (256 bits from the OS CSPRNG), csprng == 1
};

// ------------------------------------------------------------------ scalar ops
#ifdef __CUDACC__
HD u64 mulhi64(u64 a, u64 b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (u64)(((unsigned __int128)a * b) >> 64);
#endif
}
#else
inline u64 mulhi64(u64 a, u64 b) { return (u64)(((unsigned __int128)a * b) >> 64); }
#endif

HD u64 neg_mod(u64 a, u64 q) { return a ? q - a : 0; }
// Every ciphertext prime (Q, P and B) has the form q = c 2^32 + 1 (params.cpp),
// so the low 64 bits of x q are x + (x_lo c) 2^32: one 32-bit IMAD instead of
// an IMAD.WIDE and two IMADs.  Every quotient-times-q product of a Shoup or
// Barrett reduction below goes through this; the plaintext modulus t = 65537 is
// not of that form and never reaches these helpers (its transforms have their
// own kernel, ntt.cu k_ntt_t).
HD u64 mul_lo_q(u64 x, u64 q) {
#ifdef __CUDA_ARCH__
    u32 hi;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(hi) : "r"((u32)x), "r"((u32)(q >> 32)), "r"((u32)(x >> 32)));
    return ((u64)hi << 32) | (u32)x;
#else
    return x * q;
#endif
}
// Harvey's lazy Shoup product: a * w mod q in [0, 2q), any a < 2^64
HD u64 shoup_lazy(u64 a, u64 w, u64 ws, u64 q) { return a * w - mul_lo_q(mulhi64(a, ws), q); }
// Shoup product whose quotient drops the a_lo*ws_lo partial product: the
// quotient is low by at most 1, so the result lies in [0, 3q) for any a < 2^64.
// On sm_100a the quotient is 2 IMAD.WIDE + 1 IMAD.HI instead of 4 IMAD.WIDE
// (the NTT is bound by the integer multiply pipe).
HD u64 mulhi64_approx(u64 a, u64 b) {
#ifdef __CUDA_ARCH__
    const u32 a0 = (u32)a, a1 = (u32)(a >> 32), b0 = (u32)b, b1 = (u32)(b >> 32);
    u32 x0, x1, x2, r0, r1;
    asm("mul.lo.u32 %0, %5, %7;\n\t"
        "mul.hi.u32 %1, %5, %7;\n\t"
        "mad.lo.cc.u32 %0, %6, %8, %0;\n\t"
        "madc.hi.cc.u32 %1, %6, %8, %1;\n\t"
        "addc.u32 %2, 0, 0;\n\t"
        "mad.lo.cc.u32 %3, %5, %8, %1;\n\t"
        "madc.hi.u32 %4, %5, %8, %2;"
        : "=&r"(x0), "=&r"(x1), "=&r"(x2), "=&r"(r0), "=&r"(r1)
        : "r"(a1), "r"(a0), "r"(b0), "r"(b1));
    return ((u64)r1 << 32) | r0;
#else
    const u64 a_lo = (u32)a, a_hi = a >> 32, b_lo = (u32)b, b_hi = b >> 32;
    const u64 m1 = a_hi * b_lo, m2 = a_lo * b_hi;
    return a_hi * b_hi + (m1 >> 32) + (m2 >> 32) + (((m1 & 0xffffffffULL) + (m2 & 0xffffffffULL)) >> 32);
#endif
}
// a * w - qh * q (mod 2^64) for the special primes.  Code-generation variants
// (same value; they differ in SASS and in register pressure inside the
// unrolled NTT rounds): 0 generic 64-bit product, 1 qh*q hi word by mad.lo,
// 2 plain C, 3 whole expression in PTX with mul.lo/mul.hi, 4 the same with
// mul.wide (IMAD.WIDE + 3 IMAD).
template <int V>
HD u64 shoup_rem(u64 a, u64 w, u64 qh, u64 q) {
#ifdef __CUDA_ARCH__
    if constexpr (V == 0) {
        return a * w - qh * q;
    } else if constexpr (V == 1) {
        return a * w - mul_lo_q(qh, q);
    } else if constexpr (V == 2) {
        return a * w - (qh + ((u64)((u32)qh * (u32)(q >> 32)) << 32));
    } else if constexpr (V == 3) {
        u32 r0, r1;
        asm("{\n\t.reg .u32 t;\n\t"
            "mul.lo.u32 %0, %2, %4;\n\t"
            "mul.hi.u32 %1, %2, %4;\n\t"
            "mad.lo.u32 %1, %2, %5, %1;\n\t"
            "mad.lo.u32 %1, %3, %4, %1;\n\t"
            "mad.lo.u32 t, %6, %8, %7;\n\t"
            "sub.cc.u32 %0, %0, %6;\n\t"
            "subc.u32 %1, %1, t;\n\t}"
            : "=&r"(r0), "=&r"(r1)
            : "r"((u32)a), "r"((u32)(a >> 32)), "r"((u32)w), "r"((u32)(w >> 32)), "r"((u32)qh),
              "r"((u32)(qh >> 32)), "r"((u32)(q >> 32)));
        return ((u64)r1 << 32) | r0;
    } else {
        u32 r0, r1;
        asm("{\n\t.reg .u32 t;\n\t.reg .u64 p;\n\t"
            "mul.wide.u32 p, %2, %4;\n\t"
            "mov.b64 {%0, %1}, p;\n\t"
            "mad.lo.u32 %1, %2, %5, %1;\n\t"
            "mad.lo.u32 %1, %3, %4, %1;\n\t"
            "mad.lo.u32 t, %6, %8, %7;\n\t"
            "sub.cc.u32 %0, %0, %6;\n\t"
            "subc.u32 %1, %1, t;\n\t}"
            : "=&r"(r0), "=&r"(r1)
            : "r"((u32)a), "r"((u32)(a >> 32)), "r"((u32)w), "r"((u32)(w >> 32)), "r"((u32)qh),
              "r"((u32)(qh >> 32)), "r"((u32)(q >> 32)));
        return ((u64)r1 << 32) | r0;
    }
#else
    return a * w - qh * q;
#endif
}
#ifndef HGM_SHOUP_V
#define HGM_SHOUP_V 4
#endif
template <int V = HGM_SHOUP_V>
HD u64 shoup_lazy3(u64 a, u64 w, u64 ws, u64 q) { return shoup_rem<V>(a, w, mulhi64_approx(a, ws), q); }
// x in [0, 2m) -> [0, m)   (m = q or 2q).  On the device the subtraction's
// borrow selects the result: IADD3 + IADD3.X (carry out) + 2 SEL, where the
// compare-then-subtract form costs two ISETP, two SEL and the subtraction.
#ifndef HGM_RED_BORROW
#define HGM_RED_BORROW 1
#endif
#ifndef HGM_ADD128_PTX
#define HGM_ADD128_PTX 1
#endif
#ifndef HGM_MAC_PTX
#define HGM_MAC_PTX 1
#endif
HD u64 reduce_once(u64 x, u64 m) {
#if defined(__CUDA_ARCH__) && HGM_RED_BORROW
    u32 lo, hi, b;
    asm("sub.cc.u32 %0, %3, %5;\n\t"
        "subc.cc.u32 %1, %4, %6;\n\t"
        "subc.u32 %2, 0, 0;"
        : "=r"(lo), "=r"(hi), "=r"(b)
        : "r"((u32)x), "r"((u32)(x >> 32)), "r"((u32)m), "r"((u32)(m >> 32)));
    return b ? x : ((u64)hi << 32) | lo;
#else
    return x >= m ? x - m : x;
#endif
}
// a + b, a - b mod q for a, b < q (q < 2^63), through the borrow-select reduction
HD u64 add_mod(u64 a, u64 b, u64 q) { return reduce_once(a + b, q); }
HD u64 sub_mod(u64 a, u64 b, u64 q) { return reduce_once(a + q - b, q); }
// a * w mod q with ws = floor(w 2^64 / q); any a < 2^64, result in [0, q)
HD u64 shoup_mul(u64 a, u64 w, u64 ws, u64 q) {
    u64 r = shoup_lazy3(a, w, ws, q);  // [0, 3q)
    r = reduce_once(r, q);
    return reduce_once(r, q);
}
// a * b mod q for a, b < q < 2^61 (shifted Barrett, two corrections)
HD u64 mul_mod(u64 a, u64 b, const Prime& p) {
    const u64 lo = a * b, hi = mulhi64(a, b);
    const u64 x = (hi << (66 - p.s)) | (lo >> (p.s - 2));
    const u64 qh = mulhi64_approx(x, p.mu);  // low by at most 3: r < 4q
    const u64 r = lo - mul_lo_q(qh, p.q);
    return reduce_once(reduce_once(r, 2 * p.q), p.q);
}
// 128-bit lazy accumulator of products of residues, reduced once; valid while
// the sum stays below 2^(s+62) (4 products of 60-bit residues, 9 of 55-bit).
// (hi:lo) += (bh:bl): on the device one carry chain (add.cc / addc: IADD3 +
// IADD3.X with carry-out), where the C form derives the carry by a 64-bit
// compare and a select.
HD void add128(u64& lo, u64& hi, u64 bl, u64 bh) {
#if defined(__CUDA_ARCH__) && HGM_ADD128_PTX
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(bl), "l"(bh));
#else
    lo += bl;
    hi += bh + (lo < bl);
#endif
}
struct Acc {
    u64 lo = 0, hi = 0;
    HD void add(u64 v) { add128(lo, hi, v, 0); }
    HD void mac(u64 a, u64 b) { add128(lo, hi, a * b, mulhi64(a, b)); }
};
// Shifted Barrett on x < 2^(s+62) (s = bit length of q <= 60): x >> (s-2)
// fits 64 bits; the quotient estimate is low by at most 2 (+1 for the
// 3-partial-product high half), so r < 4q and two corrections suffice.
HD u64 reduce_acc(const Acc& a, const Prime& p) {
    const u64 x = (a.hi << (66 - p.s)) | (a.lo >> (p.s - 2));
    const u64 qh = mulhi64_approx(x, p.mu);
    const u64 r = a.lo - mul_lo_q(qh, p.q);
    return reduce_once(reduce_once(r, 2 * p.q), p.q);
}
// The same on x < 2^(s+63) (8 products of 60-bit residues and a residue): x >> (s-1)
// fits 64 bits and 2 mu stands in for floor(2^(63+s) / q) (low by less than 2), so the
// quotient estimate is low by less than 3 (+1 for the 3-partial-product high half):
// r < 5q, three corrections.
HD u64 reduce_acc_wide(const Acc& a, const Prime& p) {
    const u64 x = (a.hi << (65 - p.s)) | (a.lo >> (p.s - 1));
    const u64 qh = mulhi64_approx(x, p.mu << 1);
    const u64 r = a.lo - mul_lo_q(qh, p.q);
    return reduce_once(reduce_once(reduce_once(r, 4 * p.q), 2 * p.q), p.q);
}
// Column accumulator for sums of residue products.  Operands are split into
// S-bit digits (residues < 2^(2S): S = 30 for 60-bit primes, 28 for 55-bit)
// and multiplied Karatsuba-style: c0 += a_l b_l, c2 += a_h b_h,
// c1 += (a_l + a_h)(b_l + b_h), the middle column being c1 - c0 - c2 at fold
// time.  Each partial product accumulates with one IMAD.WIDE (multiply + 64-bit
// add) and no carry handling, so a 64x64 product costs 3 IMAD.WIDE instead of
// 5 IMAD.WIDE + 2 IMAD + carries.  Digit sums are < 2^(S+1): c1 holds up to
// 2^(62-2S) products between folds (4 at S = 30, 64 at S = 28).  Plain
// additions go to a separate 128-bit word (x, xh), outside the columns.
template <int S>
struct Dig {
    u32 l, h, s;  // s = l + h
};
template <int S>
HD Dig<S> split(u64 a) {
    const u32 l = (u32)a & ((1u << S) - 1u), h = (u32)(a >> S);
    return Dig<S>{l, h, l + h};
}
// digits of a value stored packed as l | h << 32 (k_mask_digits)
template <int S>
HD Dig<S> packed_dig(u64 p) {
    const u32 l = (u32)p, h = (u32)(p >> 32);
    return Dig<S>{l, h, l + h};
}
struct Cols {
    u64 c0 = 0, c1 = 0, c2 = 0, x = 0, xh = 0;
    template <int S>
    HD void mac(Dig<S> a, Dig<S> b) {
#if defined(__CUDA_ARCH__) && HGM_MAC_PTX
        // one IMAD.WIDE.U32 per column with the 64-bit accumulator as its addend
        // (parameter set 1's long unrolled conversions, S = 28, keep the C form:
        // the asm operands pushed k_scale_round<ShapeQ8> into 1.4 KB of spills)
        if constexpr (S == 28) {
            c0 += (u64)a.l * b.l;
            c1 += (u64)a.s * b.s;
            c2 += (u64)a.h * b.h;
            return;
        }
        asm("mad.wide.u32 %0, %3, %4, %0;\n\t"
            "mad.wide.u32 %1, %5, %6, %1;\n\t"
            "mad.wide.u32 %2, %7, %8, %2;"
            : "+l"(c0), "+l"(c1), "+l"(c2)
            : "r"(a.l), "r"(b.l), "r"(a.s), "r"(b.s), "r"(a.h), "r"(b.h));
#else
        c0 += (u64)a.l * b.l;
        c1 += (u64)a.s * b.s;
        c2 += (u64)a.h * b.h;
#endif
    }
    // adds a full 64-bit value
    template <int S>
    HD void add(u64 v) {
        add128(x, xh, v, 0);
    }
    // x + c0 + (c1 - c0 - c2) 2^S + c2 2^(2S) as a 128-bit accumulator
    template <int S>
    HD Acc fold() const {
        const u64 mid = c1 - c0 - c2;
        Acc a;
        a.lo = x;
        a.hi = xh;
        add128(a.lo, a.hi, c0, 0);
        add128(a.lo, a.hi, mid << S, mid >> (64 - S));
        add128(a.lo, a.hi, c2 << (2 * S), c2 >> (64 - 2 * S));
        return a;
    }
};

HD u64 from_signed(i64 v, u64 q) { return v >= 0 ? (u64)v % q : q - 1 - ((u64)(-(v + 1)) % q); }
HD u64 centred_neg(u64 y, u64 q) { return y > (q - 1) / 2; }
// y (canonical mod src) viewed as its centred representative, reduced mod dst.
// Requires src < 2^62 and src, dst odd primes.
HD u64 centred_to(u64 y, u64 src, u64 dst) {
    if (y > (src - 1) / 2) {
        u64 m = (src - y) % dst;  // |centred value| mod dst
        return m ? dst - m : 0;
    }
    return y % dst;
}

// 128-bit accumulator in units of 2^-64
struct Acc128 {
    u64 lo, hi;
};
HD void fx_add(Acc128& s, u64 y, const Frac& f) {
    // y*f.hi (128 bit) + mulhi(y, f.lo)
    u64 plo = y * f.hi, phi = mulhi64(y, f.hi);
    add128(plo, phi, mulhi64(y, f.lo), 0);
    add128(s.lo, s.hi, plo, phi);
}
// fx_add for a fraction whose integer part f.hi < 2^32 (1/q, 1/b: f.hi = 2^64/q):
// y * f.hi from two 32x32 products instead of a full 64x64 one; same sum exactly
HD void fx_add_small(Acc128& s, u64 y, const Frac& f) {
    const u64 p0 = (u64)(u32)y * f.hi, p1 = (y >> 32) * f.hi;  // f.hi < 2^32
    u64 plo = p0, phi = 0;
    add128(plo, phi, p1 << 32, p1 >> 32);
    add128(plo, phi, mulhi64(y, f.lo), 0);
    add128(s.lo, s.hi, plo, phi);
}
HD u64 fx_round(const Acc128& s) {
    // (s + 2^63) >> 64
    u64 lo = s.lo, hi = s.hi;
    add128(lo, hi, 1ULL << 63, 0);
    return hi;
}

// ------------------------------------------------------------------ sampler
HD u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
HD u64 prng(u64 seed, u64 stream, u64 idx) {
    u64 h = mix64(seed ^ 0x5851f42d4c957f2dULL);
    h = mix64(h ^ stream);
    return mix64(h + (idx + 1) * 0x9e3779b97f4a7c15ULL);
}
// ChaCha block function (Bernstein's original layout: 64-bit block counter,
// 64-bit nonce), `rounds` rounds.  OS-seeded sessions draw every secret-key,
// key-switching and encryption sample from ChaCha12(key, nonce = stream,
// counter = index): the parity PRF above is a public bijection chain, so one
// output (e.g. a public key's uniform `a`) would give back its 64-bit seed.
HD u32 rotl32(u32 x, int r) { return (x << r) | (x >> (32 - r)); }
#define HGM_QR(a, b, c, d) \
    a += b; d = rotl32(d ^ a, 16); c += d; b = rotl32(b ^ c, 12); \
    a += b; d = rotl32(d ^ a, 8);  c += d; b = rotl32(b ^ c, 7);
HD void chacha_block(const u32 key[8], u64 nonce, u64 counter, int rounds, u32 out[16]) {
    u32 x[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                 key[0], key[1], key[2], key[3], key[4], key[5], key[6], key[7],
                 (u32)counter, (u32)(counter >> 32), (u32)nonce, (u32)(nonce >> 32)};
    u32 in[16];
    for (int i = 0; i < 16; ++i) in[i] = x[i];
    for (int r = 0; r < rounds; r += 2) {
        HGM_QR(x[0], x[4], x[8], x[12]) HGM_QR(x[1], x[5], x[9], x[13])
        HGM_QR(x[2], x[6], x[10], x[14]) HGM_QR(x[3], x[7], x[11], x[15])
        HGM_QR(x[0], x[5], x[10], x[15]) HGM_QR(x[1], x[6], x[11], x[12])
        HGM_QR(x[2], x[7], x[8], x[13]) HGM_QR(x[3], x[4], x[9], x[14])
    }
    for (int i = 0; i < 16; ++i) out[i] = x[i] + in[i];
}
#undef HGM_QR
constexpr int kChachaRounds = 12;
// one 64-bit sample of (stream, idx): the first two words of its block
HD u64 chacha_u64(const u32 key[8], u64 stream, u64 idx) {
    u32 b[16];
    chacha_block(key, stream, idx, kChachaRounds, b);
    return (u64)b[0] | ((u64)b[1] << 32);
}
// the session's sampler: ChaCha for OS-seeded sessions, the parity PRF (shared
// bit for bit with the CPU oracle) for caller-seeded ones
HD u64 draw(const DevCtx& cx, u64 stream, u64 idx) {
    return cx.csprng ? chacha_u64(cx.ck, stream, idx) : prng(cx.seed, stream, idx);
}
HD i64 ternary(const DevCtx& cx, u64 stream, u64 idx) { return (i64)mulhi64(draw(cx, stream, idx), 3) - 1; }
HD u64 uniform(const DevCtx& cx, u64 stream, u64 idx, u64 q) { return mulhi64(draw(cx, stream, idx), q); }
HD i64 gauss(const DevCtx& cx, u64 stream, u64 idx, const u64* cdt) {
    u64 r = draw(cx, stream, idx);
    u64 mag = r & 0x7fffffffffffffffULL;
    i64 k = 0;
    while (mag >= cdt[k]) ++k;
    return (r >> 63) ? -k : k;
}

// index of the NTT slot read by the automorphism X -> X^g at NTT index k
HD u32 galois_src(u32 k, u32 g, u32 logN) {
#ifdef __CUDA_ARCH__
    const u32 bk = __brev(k) >> (32 - logN);
#else
    u32 bk = 0;
    for (u32 i = 0, x = k; i < logN; ++i, x >>= 1) bk = (bk << 1) | (x & 1);
#endif
    const u32 twoN_mask = (2u << logN) - 1;
    const u32 e = (g * (2 * bk + 1)) & twoN_mask;  // mod 2^32 then mod 2N (2N | 2^32)
#ifdef __CUDA_ARCH__
    return __brev((e - 1) >> 1) >> (32 - logN);
#else
    u32 v = (e - 1) >> 1, r = 0;
    for (u32 i = 0; i < logN; ++i, v >>= 1) r = (r << 1) | (v & 1);
    return r;
#endif
}

}  // namespace hgm
