// bfv.cu -- RNS-BFV primitive kernels and the Context that launches them.
//
// Semantics are defined by oracle/bfv_oracle.cpp (bit-exact); the comments
// name the oracle routine each kernel reproduces.  Shapes: n items per launch,
// thread per (item, coefficient), loops over RNS limbs inside the thread so a
// warp's loads are coalesced within each limb.
#include <algorithm>
#include <cstring>
#include <stdexcept>

#include "context.hpp"

#include <type_traits>
#include "parallel.hpp"

namespace hgm {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

__constant__ DevParams c_dp[kParamSets];

constexpr int kThreads = 256;

// RNS shapes of the parameter sets, as compile-time constants so per-thread
// residue arrays unroll into registers (set 0 and 2: L 3 / K 1 / B 4 / dnum 3;
// set 1: L 8 / K 4 / B 9 / dnum 2).
// S: digit width of the column accumulator (residues < 2^(2S)).
struct ShapeQ3 {
    static constexpr u32 L = 3, K = 1, nB = 4, dnum = 3, A = 1, R = 4;
    static constexpr int S = 30;  // 60-bit primes
};
struct ShapeQ8 {
    static constexpr u32 L = 8, K = 4, nB = 9, dnum = 2, A = 4, R = 12;
    static constexpr int S = 28;  // 55-bit primes
};
// items per launch sequence: bounds temporaries and staging uploads
constexpr int kChunkEnc = 1024, kChunkDec = 1024, kChunkLin = 8192, kChunkKs = 8192, kChunkMult = 4096;
// key-switch and multiplication batches are also capped by their temporaries:
// large batches fill the GPU (3 NTT CTAs per SM, >= 1 wave of limbs per launch)
constexpr size_t kChunkBytes = (size_t)24 << 30;
// the tensor pass applies the INTT's first stage (HGM_TENSOR_S1=0 disables)
bool tensor_first_stage() {
    static const bool on = [] {
        const char* e = std::getenv("HGM_TENSOR_S1");
        return !e || e[0] != '0';
    }();
    return on;
}

int chunk_for(size_t words_per_item, int cap) {
    // 24 GB, or a sixth of the device's memory on smaller parts (the stream-ordered
    // pool keeps freed blocks, so "free" memory is not a useful bound here)
    static const size_t budget = [] {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || total_b == 0) return kChunkBytes;
        return std::min(kChunkBytes, total_b / 6);
    }();
    const size_t n = budget / (words_per_item * 8);
    return (int)std::max<size_t>(1, std::min<size_t>(n, (size_t)cap));
}

// values with |v| < q (noise, ternary, small messages)
__device__ __forceinline__ u64 small_to_mod(i64 v, u64 q) { return v >= 0 ? (u64)v : q + v; }
// y < src < 2*dst (all primes of a set share their bit length): centred y mod dst
__device__ __forceinline__ u64 centred_lift(u64 y, u64 src, u64 dst) {
    if (y > (src - 1) / 2) {
        u64 m = src - y;
        if (m >= dst) m -= dst;
        return m ? dst - m : 0;
    }
    return y >= dst ? y - dst : y;
}

#define ITEM_LOOP for (u32 item = blockIdx.y; item < n; item += gridDim.y)
#define COEF_LOOP for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x)

// ---------------------------------------------------------------- encoding
// oracle encode(): slot values mod t scattered to their NTT positions
// vals: slot values already reduced to [0, t) on the host (to_slot_residue),
// stride H per item
__global__ void k_encode_scatter(DevCtx cx, u32 n, const u32* vals,
                                 const u32* S, u64* out) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, H = N / 2;
    ITEM_LOOP {
        COEF_LOOP {
            u64 v = 0;
            if (j < S[item]) v = vals[(size_t)item * H + j];
            out[(size_t)item * N + cx.slot_ntt[j]] = v;
        }
    }
}
// canonical residue mod t of a signed slot value (SlotBackend semantics)
inline u32 to_slot_residue(i64 x) {
    return (u32)(x >= 0 ? (u64)x % kT : kT - 1 - ((u64)(-(x + 1)) % kT));
}

// oracle encrypt(): sample u, e0, e1; c0 = e0 + Delta m, c1 = e1 (coefficient form)
// noise (optional): host-sampled [n][3][N] signed coefficients (u, e0, e1) in
// place of the counter PRNG (hgm_encrypt_noise)
template <typename SH>
__global__ void __launch_bounds__(kThreads, 4) k_enc_lift(DevCtx cx, u32 n, const u64* m, const u64* ctr,
                           const i64* noise, u64* U, u64* const* out) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L;
    ITEM_LOOP {
        const u64 c = noise ? 0 : ctr[item];
        const i64* nz = noise ? noise + (size_t)item * 3 * N : nullptr;
        u64* o = out[item];
        COEF_LOOP {
            const i64 u = nz ? nz[j] : ternary(cx, kStreamEncU | c, j);
            const i64 e0 = nz ? nz[N + j] : gauss(cx, kStreamEncE0 | c, j, cx.cdt);
            const i64 e1 = nz ? nz[2 * N + j] : gauss(cx, kStreamEncE1 | c, j, cx.cdt);
            const u64 mj = m[(size_t)item * N + j];
            for (u32 i = 0; i < L; ++i) {
                const u64 q = dp->pr[i].q;
                U[((size_t)item * L + i) * N + j] = small_to_mod(u, q);
                o[(size_t)i * N + j] =
                    add_mod(small_to_mod(e0, q), shoup_mul(mj, dp->delta[i], dp->delta_sh[i], q), q);
                o[(size_t)(L + i) * N + j] = small_to_mod(e1, q);
            }
        }
    }
}

template <typename SH>
__global__ void k_enc_finish(DevCtx cx, u32 n, const u64* U, const u64* pk,
                             u64* const* out) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L;
    ITEM_LOOP {
        u64* o = out[item];
        COEF_LOOP {
            for (u32 i = 0; i < L; ++i) {
                const Prime& P = dp->pr[i];
                const u64 u = U[((size_t)item * L + i) * N + j];
                const size_t w0 = (size_t)i * N + j, w1 = (size_t)(L + i) * N + j;
                o[w0] = add_mod(mul_mod(pk[w0], u, P), o[w0], P.q);
                o[w1] = add_mod(mul_mod(pk[w1], u, P), o[w1], P.q);
            }
        }
    }
}

// ---------------------------------------------------------------- decryption
template <typename SH>
__global__ void k_dec_phase(DevCtx cx, u32 n, const u64* const* in,
                            const u64* sk, u64* X) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L;
    ITEM_LOOP {
        const u64* c = in[item];
        COEF_LOOP {
            for (u32 i = 0; i < L; ++i) {
                const Prime& P = dp->pr[i];
                X[((size_t)item * L + i) * N + j] =
                    add_mod(c[(size_t)i * N + j], mul_mod(c[(size_t)(L + i) * N + j], sk[(size_t)i * N + j], P), P.q);
            }
        }
    }
}

// oracle decrypt(): m = round(t x / Q) mod t via sum_i [x_i (Q/q_i)^-1]_{q_i} t/q_i
template <typename SH>
__global__ void __launch_bounds__(kThreads, 4) k_dec_round(DevCtx cx, u32 n, const u64* X, u64* M) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L;
    ITEM_LOOP {
        COEF_LOOP {
            Acc128 s{0, 0};
            for (u32 i = 0; i < L; ++i) {
                const u64 q = dp->pr[i].q;
                const u64 y = shoup_mul(X[((size_t)item * L + i) * N + j], dp->qhat_inv[i], dp->qhat_inv_sh[i], q);
                fx_add(s, y, dp->t_over_q[i]);
            }
            M[(size_t)item * N + j] = fx_round(s) % kT;
        }
    }
}

// out: decrypted slots in [0, t) as u32, stride H per item
__global__ void k_dec_gather(DevCtx cx, u32 n, const u64* M, const u32* S,
                             u32* out) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, H = N / 2;
    ITEM_LOOP {
        for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < S[item]; i += gridDim.x * blockDim.x)
            out[(size_t)item * H + i] = (u32)M[(size_t)item * N + cx.slot_ntt[i]];
    }
}

// ---------------------------------------------------------------- linear ops
template <typename SH>
__global__ void k_add(DevCtx cx, u32 n, const u64* const* a,
                      const u64* const* b, u64* const* out) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L;
    const size_t W = (size_t)2 * L * N;
    ITEM_LOOP {
        const u64 *x = a[item], *y = b[item];
        u64* o = out[item];
        for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < W; w += (size_t)gridDim.x * blockDim.x) {
            const u64 q = dp->pr[(w / N) % L].q;
            o[w] = add_mod(x[w], y[w], q);
        }
    }
}

__global__ void k_copy(u32 n, size_t W, const u64* const* in, u64* const* out) {
    ITEM_LOOP {
        const ulonglong2* x = reinterpret_cast<const ulonglong2*>(in[item]);
        ulonglong2* o = reinterpret_cast<ulonglong2*>(out[item]);
        for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < W / 2; w += (size_t)gridDim.x * blockDim.x)
            o[w] = x[w];
    }
}

// out[o] = sum_t in[t] (.* mask[t]) : oracle cmult() followed by add()
// Masks are stored in packed digit form (mask_digits: l | h << 32).  Each
// thread takes two adjacent words (16-byte loads) of one limb.
#ifndef HGM_LC_U
#define HGM_LC_U 2
#endif
#ifndef HGM_LC_MINB
#define HGM_LC_MINB 4
#endif
// RL = limbs per component: L (ciphertexts), or R = L + K for pending key
// switches over Q ++ P (the masks hold R limbs; limb r uses prime r).
template <typename SH, u32 RL = SH::L>
__global__ void __launch_bounds__(kThreads, HGM_LC_MINB) k_lincomb(DevCtx cx, u32 n, const u32* off,
                          const u64* const* in, const u64* const* mask, u64* const* out) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, logN = dp->logN, L = RL;
    const size_t LN = (size_t)L * N, W2 = LN;  // word pairs per ciphertext
    ITEM_LOOP {
        const u32 t0 = off[item], t1 = off[item + 1];
        ulonglong2* o = reinterpret_cast<ulonglong2*>(out[item]);
        for (size_t w2 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w2 < W2; w2 += (size_t)gridDim.x * blockDim.x) {
            const size_t wl2 = w2 < LN / 2 ? w2 : w2 - LN / 2;  // pair index within the component
            const Prime& P = dp->pr[(wl2 * 2) >> logN];
            // exact accumulation; reduced after every 3 masked products
            // (the sum stays below 2^(s+62), reduce_acc's range).  Terms are
            // taken kU at a time with all their loads issued first, so a
            // long plain sum (an add tree of 64 products) is not a chain of
            // dependent load latencies.
            Cols a0, a1;
            u32 pending = 0;
            constexpr u32 kU = HGM_LC_U;
            for (u32 t = t0; t < t1; t += kU) {
                const u32 nt = t1 - t < kU ? t1 - t : kU;
                ulonglong2 v[kU], m[kU];
                bool hm[kU];
#pragma unroll
                for (u32 u = 0; u < kU; ++u) {
                    hm[u] = false;
                    if (u < nt) {
                        const u64* mt = mask[t + u];
                        hm[u] = mt != nullptr;
                        v[u] = reinterpret_cast<const ulonglong2*>(in[t + u])[w2];
                        if (mt) m[u] = __ldg(reinterpret_cast<const ulonglong2*>(mt) + wl2);
                    }
                }
#pragma unroll
                for (u32 u = 0; u < kU; ++u) {
                    if (u >= nt) break;
                    if (hm[u]) {
                        a0.mac(split<SH::S>(v[u].x), packed_dig<SH::S>(m[u].x));
                        a1.mac(split<SH::S>(v[u].y), packed_dig<SH::S>(m[u].y));
                        if (++pending == 3) {
                            const u64 r0 = reduce_acc(a0.fold<SH::S>(), P), r1 = reduce_acc(a1.fold<SH::S>(), P);
                            a0 = Cols{};
                            a1 = Cols{};
                            a0.x = r0;
                            a1.x = r1;
                            pending = 0;
                        }
                    } else {
                        a0.add<SH::S>(v[u].x);
                        a1.add<SH::S>(v[u].y);
                    }
                }
            }
            ulonglong2 r;
            r.x = reduce_acc(a0.fold<SH::S>(), P);
            r.y = reduce_acc(a1.fold<SH::S>(), P);
            o[w2] = r;
        }
    }
}

// The same sum when every term carries a mask (the masked sums of rotations of
// an apply_plan / eps / omega plan): terms are taken three at a time -- the
// most masked products the 128-bit column sum holds with the running residue
// (3 q^2 + q < 2^(s+62)) -- with all their loads issued first, the chunk's
// columns start from its first product (no zeroed accumulators to carry
// through the loop) and each chunk folds the previous chunk's residue in.
template <typename SH, u32 RL = SH::L>
__global__ void __launch_bounds__(kThreads, HGM_LC_MINB) k_lincomb_masked(DevCtx cx, u32 n, const u32* off,
                          const u64* const* in, const u64* const* mask, u64* const* out) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, logN = dp->logN, L = RL;
    const size_t LN = (size_t)L * N, W2 = LN;  // word pairs per output
    ITEM_LOOP {
        const u32 t0 = off[item], t1 = off[item + 1];
        ulonglong2* o = reinterpret_cast<ulonglong2*>(out[item]);
        for (size_t w2 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w2 < W2; w2 += (size_t)gridDim.x * blockDim.x) {
            const size_t wl2 = w2 < LN / 2 ? w2 : w2 - LN / 2;  // pair index within the component
            const Prime& P = dp->pr[(wl2 * 2) >> logN];
            u64 r0 = 0, r1 = 0;
            // one straight-line block per chunk size: with the term count a
            // compile-time constant the column accumulators stay in aligned
            // register pairs and every product is a single IMAD.WIDE (a shared,
            // predicated block split each into IMAD.WIDE + IADD3 + IMAD.X + moves)
            auto chunk = [&](auto nt_c, u32 t) {
                constexpr u32 NT = decltype(nt_c)::value;
                ulonglong2 v[NT], m[NT];
#pragma unroll
                for (u32 u = 0; u < NT; ++u) {
                    v[u] = reinterpret_cast<const ulonglong2*>(in[t + u])[w2];
                    m[u] = __ldg(reinterpret_cast<const ulonglong2*>(mask[t + u]) + wl2);
                }
                Cols a0, a1;
                a0.x = r0;
                a1.x = r1;
#pragma unroll
                for (u32 u = 0; u < NT; ++u) {
                    a0.mac(split<SH::S>(v[u].x), packed_dig<SH::S>(m[u].x));
                    a1.mac(split<SH::S>(v[u].y), packed_dig<SH::S>(m[u].y));
                }
                r0 = reduce_acc(a0.fold<SH::S>(), P);
                r1 = reduce_acc(a1.fold<SH::S>(), P);
            };
            for (u32 t = t0; t < t1; t += 3) {
                const u32 nt = t1 - t;
                if (nt >= 3)
                    chunk(std::integral_constant<u32, 3>{}, t);
                else if (nt == 2)
                    chunk(std::integral_constant<u32, 2>{}, t);
                else
                    chunk(std::integral_constant<u32, 1>{}, t);
            }
            ulonglong2 r;
            r.x = r0;
            r.y = r1;
            o[w2] = r;
        }
    }
}

// canonical residues -> packed digit form (l | h << 32) for k_lincomb (masks) and
// k_ks_inner (keys); launch on a 1-D grid (every word converted exactly once)
template <typename SH>
__global__ void k_mask_digits(u64* m, size_t words) {
    for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (size_t)gridDim.x * blockDim.x) {
        const Dig<SH::S> d = split<SH::S>(m[w]);
        m[w] = (u64)d.l | ((u64)d.h << 32);
    }
}

// centred lift of the mod-t mask polynomial to each q_i (oracle cmult())
template <typename SH>
__global__ void k_mask_lift(DevCtx cx, const u64* m, u64* out) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L;
    const u32 n = 1;
    ITEM_LOOP {
        COEF_LOOP {
            const u64 v = m[j];
            for (u32 i = 0; i < SH::R; ++i) out[(size_t)i * N + j] = centred_lift(v, kT, dp->pr[i].q);
        }
    }
}

// ---------------------------------------------------------------- key switching
// c1 limbs of each ct into a contiguous [n][L][N] buffer
template <typename SH>
__global__ void k_gather_c1(DevCtx cx, u32 n, const u64* const* ct, u64* C) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L;
    const size_t LN = (size_t)L * N;
    ITEM_LOOP {
        const u64* c = ct[item] + LN;
        for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < LN; w += (size_t)gridDim.x * blockDim.x)
            C[item * LN + w] = c[w];
    }
}

// oracle key_switch() ModUp: digit dg of the coefficient-domain poly C, lifted
// to every limb of Q ++ P with centred residues.  D: [n][dnum][R][N]
// from_intt: C is an unscaled, lazy INTT (N * c1 in [0, 4q)); N^-1 is folded
// into dg_hat_inv_n and the digit's own limbs are not written (the caller
// copies them from the NTT-domain ciphertext, so they need no forward NTT).
template <typename SH>
__global__ void k_modup_lift(DevCtx cx, u32 n, const u64* C, size_t c_stride,
                             u64* D, int from_intt, u64* const* Dp = nullptr) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, R = SH::R, A = SH::A, dnum = SH::dnum;
    const u64* ghi = from_intt ? dp->dg_hat_inv_n : dp->dg_hat_inv;
    const u64* ghs = from_intt ? dp->dg_hat_inv_n_sh : dp->dg_hat_inv_sh;
    ITEM_LOOP {
        const u64* c = C + item * c_stride;
        u64* d = Dp ? Dp[item] : D + (size_t)item * dnum * R * N;  // per-item outputs, or one block
        COEF_LOOP {
            u64 x[kMaxL];
            for (u32 i = 0; i < L; ++i) x[i] = c[(size_t)i * N + j];
            for (u32 dg = 0; dg < dnum; ++dg) {
                u64 y[kMaxL];
                for (u32 a = 0; a < A; ++a) {
                    const u32 i = dg * A + a;
                    y[a] = shoup_mul(x[i], ghi[i], ghs[i], dp->pr[i].q);
                }
                for (u32 r = 0; r < R; ++r) {
                    u64 v;
                    if (r < L && r / A == dg) {
                        if (from_intt) continue;
                        v = x[r];
                    } else {
                        const u64 qr = dp->pr[r].q;
                        if (A == 1) {
                            v = centred_lift(y[0], dp->pr[dg].q, qr);  // (Q_d/q_i) = 1
                        } else {
                            Cols s;
                            for (u32 a = 0; a < A; ++a) {
                                const u32 i = dg * A + a;
                                s.mac(split<SH::S>(centred_lift(y[a], dp->pr[i].q, qr)), split<SH::S>(dp->dg_hat[i][r]));
                            }
                            v = reduce_acc(s.fold<SH::S>(), dp->pr[r]);
                        }
                    }
                    d[((size_t)dg * R + r) * N + j] = v;
                }
            }
        }
    }
}

// acc[c][r] = sum_dg D[dg][r][galois_src(k)] * key[dg][c][r][k]  ([n][2][R][N];
// keys stored in packed digit form, k_mask_digits)
// Items are grouped by Galois key (the engine sorts rotations by element): a
// block serves up to kKeyReuse consecutive items and reads each key element
// once for all items of the group that share it.
constexpr int kKeyReuse = 8;
template <typename SH>
// c0 (optional, per item): NTT-domain c0 of the rotated ciphertext; P phi_g(c0)
// is folded into acc's component 0 over Q (a pending key switch, oracle rot_x:
// ModDown(acc + P y) = ModDown(acc) + y).
__global__ void k_ks_inner(DevCtx cx, u32 n, const u64* const* D,
                           const u64* const* key, const u32* g, u64* const* acc, const u64* const* c0) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, R = SH::R, dnum = SH::dnum, logN = dp->logN;
    for (u32 grp = blockIdx.y; grp * kKeyReuse < n; grp += gridDim.y) {
        const u32 i0 = grp * kKeyReuse;
        const u32 cnt = min((u32)kKeyReuse, n - i0);
        const u64* k = key[i0];
        const u32 ge = g[i0];
        u32 same = 1;  // leading items that share key and element with i0
        while (same < cnt && key[i0 + same] == k && g[i0 + same] == ge) ++same;
        COEF_LOOP {
            const u32 src = ge == 1 ? j : galois_src(j, ge, logN);
            for (u32 r = 0; r < R; ++r) {
                const Prime& P = dp->pr[r];
                Dig<SH::S> k0[4], k1[4];
                for (u32 dg = 0; dg < dnum; ++dg) {
                    k0[dg] = packed_dig<SH::S>(__ldg(k + (((size_t)dg * 2 + 0) * R + r) * N + j));
                    k1[dg] = packed_dig<SH::S>(__ldg(k + (((size_t)dg * 2 + 1) * R + r) * N + j));
                }
                const Dig<SH::S> pm = split<SH::S>(dp->P_mod_q[r < SH::L ? r : 0]);
                for (u32 u = 0; u < same; ++u) {
                    const u64* d = D[i0 + u];
                    Cols a0, a1;  // column accumulation, one reduction per output
                    for (u32 dg = 0; dg < dnum; ++dg) {
                        const Dig<SH::S> x = split<SH::S>(d[((size_t)dg * R + r) * N + src]);
                        a0.mac(x, k0[dg]);
                        a1.mac(x, k1[dg]);
                    }
                    if (c0 && r < SH::L) a0.mac(split<SH::S>(c0[i0 + u][(size_t)r * N + src]), pm);
                    u64* a = acc[i0 + u];
                    a[(size_t)r * N + j] = reduce_acc(a0.fold<SH::S>(), P);
                    a[((size_t)R + r) * N + j] = reduce_acc(a1.fold<SH::S>(), P);
                }
            }
            for (u32 u = same; u < cnt; ++u) {  // rest of the group: own key
                const u64* kk = key[i0 + u];
                const u32 gu = g[i0 + u];
                const u32 su = gu == 1 ? j : galois_src(j, gu, logN);
                const u64* d = D[i0 + u];
                u64* a = acc[i0 + u];
                for (u32 r = 0; r < R; ++r) {
                    Cols a0, a1;
                    for (u32 dg = 0; dg < dnum; ++dg) {
                        const Dig<SH::S> x = split<SH::S>(d[((size_t)dg * R + r) * N + su]);
                        a0.mac(x, packed_dig<SH::S>(__ldg(kk + (((size_t)dg * 2 + 0) * R + r) * N + j)));
                        a1.mac(x, packed_dig<SH::S>(__ldg(kk + (((size_t)dg * 2 + 1) * R + r) * N + j)));
                    }
                    if (c0 && r < SH::L)
                        a0.mac(split<SH::S>(c0[i0 + u][(size_t)r * N + su]), split<SH::S>(dp->P_mod_q[r]));
                    a[(size_t)r * N + j] = reduce_acc(a0.fold<SH::S>(), dp->pr[r]);
                    a[((size_t)R + r) * N + j] = reduce_acc(a1.fold<SH::S>(), dp->pr[r]);
                }
            }
        }
    }
}

// Masked key of one term of a masked sum of rotations:
//   mk[dg][c][r][j] = key_g[dg][c][r][j] * m[r][j] mod q_r     (packed digits)
//   mp[r][j]        = (P mod q_r) * m[r][j] mod q_r, r < L     (packed digits)
// with m = the sum mod q_r of the term's NTT-domain mask lifts (several masks
// on one rotation add up: a x m1 + a x m2 = a x (m1 + m2) mod q).  Since
// mask (.) (sum_dg D_dg key_dg + P phi(c0)) = sum_dg D_dg (mask (.) key_dg) + phi(c0) (mask P),
// k_ks_plan computes a whole masked sum of rotations as one longer inner
// product, with neither the rotations' accumulators nor a separate masked sum.
template <typename SH>
// pre: the Q limbs' mask is multiplied by P^-1 mod q_r first, so the sum k_ks_plan
// computes over Q is P^-1 (acc + P phi(c0)) and ModDown's finishing pass adds it
// without its Shoup product (exact: the same canonical residue).
__global__ void k_mask_key(DevCtx cx, const u64* key, const u64* const* masks, u32 n_masks, u64* out, u32 pre) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, R = SH::R, L = SH::L, dnum = SH::dnum;
    auto unpack = [](u64 p) { return (u64)(u32)p + ((p >> 32) << SH::S); };
    auto pack = [](u64 v) {
        const Dig<SH::S> d = split<SH::S>(v);
        return (u64)d.l | ((u64)d.h << 32);
    };
    for (u32 w = blockIdx.x * blockDim.x + threadIdx.x; w < R * N; w += gridDim.x * blockDim.x) {
        const u32 r = w / N, j = w - r * N;
        const Prime& P = dp->pr[r];
        u64 m = 0;
        for (u32 i = 0; i < n_masks; ++i) m = add_mod(m, unpack(masks[i][w]), P.q);
        if (pre && r < L) m = mul_mod(m, dp->P_inv_q[r], P);
        for (u32 dg = 0; dg < dnum; ++dg)
            for (u32 c = 0; c < 2; ++c) {
                const size_t o = (((size_t)dg * 2 + c) * R + r) * N + j;
                out[o] = pack(mul_mod(unpack(key[o]), m, P));
            }
        if (r < L) out[(size_t)dnum * 2 * R * N + w] = pack(mul_mod(dp->P_mod_q[r], m, P));
    }
}

// out[c][r][j] = sum_t ( sum_dg D_t[dg][r][src_t(j)] mk_t[dg][c][r][j]
//                        + [c = 0, r < L] c0_t[r][src_t(j)] mp_t[r][j] )   over Q ++ P
// = sum_t mask_t (.) RotAcc(ct_t, g_t): the value k_ks_inner + k_lincomb_masked
// produce, bit for bit (canonical residues of the same sum mod q_r).
// A group is a tile of lockstep instances of one sum: each thread keeps its
// coefficient's masked-key elements of up to kPlanTerms terms in shared memory
// (its own slots: no barrier) and walks the group's instances, so a masked key
// is read once per group.  Terms are taken one at a time on top of the running
// residue (4 products + a residue stay inside the 128-bit column sum:
// 4 q^2 + q < 2^(s+62) for every prime of the sets); sums of more than
// kPlanTerms terms continue from the stored output.
// resident CTAs per SM the register allocation of the three largest elementwise kernels
// is bounded for (A/B knobs; 4 measured best)
#ifndef HGM_PLAN_MINB
#define HGM_PLAN_MINB 4
#endif
#ifndef HGM_QTOB2_MINB
#define HGM_QTOB2_MINB 4
#endif
#ifndef HGM_TACC_MINB
#define HGM_TACC_MINB 4
#endif
constexpr u32 kPlanTerms = 2;
#ifndef HGM_PLAN_WIDE
#define HGM_PLAN_WIDE 1
#endif
template <typename SH, u32 NT>
__device__ __forceinline__ void plan_terms(const Prime& P, const u64* sk, u32 tid, u32 r, u32 N, const u32* src,
                                           const u64* const* Dt, const u64* const* Ct, u64& r0, u64& r1) {
    constexpr u32 dnum = SH::dnum, R = SH::R, E = 2 * SH::dnum + 1;
    u64 x[NT][SH::dnum], c[NT];
#pragma unroll
    for (u32 t = 0; t < NT; ++t) {  // every load of the chunk first
        const u64* d = Dt[t];
#pragma unroll
        for (u32 dg = 0; dg < dnum; ++dg) x[t][dg] = d[((size_t)dg * R + r) * N + src[t]];
        c[t] = r < SH::L ? Ct[t][(size_t)r * N + src[t]] : 0;
    }
#if HGM_PLAN_WIDE
    if constexpr (NT == 2) {
        // both terms' column sums folded into one 128-bit sum, reduced once
        // (8 q^2 + q < 2^(s+63), reduce_acc_wide): one Barrett reduction per output
        // instead of one per term
        Acc s0{r0, 0}, s1{r1, 0};
#pragma unroll
        for (u32 t = 0; t < NT; ++t) {
            Cols a0, a1;
#pragma unroll
            for (u32 dg = 0; dg < dnum; ++dg) {
                const Dig<SH::S> xd = split<SH::S>(x[t][dg]);
                a0.mac(xd, packed_dig<SH::S>(sk[((t * E) + 2 * dg) * kThreads + tid]));
                a1.mac(xd, packed_dig<SH::S>(sk[((t * E) + 2 * dg + 1) * kThreads + tid]));
            }
            if (r < SH::L) a0.mac(split<SH::S>(c[t]), packed_dig<SH::S>(sk[((t * E) + 2 * dnum) * kThreads + tid]));
            const Acc f0 = a0.fold<SH::S>(), f1 = a1.fold<SH::S>();
            add128(s0.lo, s0.hi, f0.lo, f0.hi);
            add128(s1.lo, s1.hi, f1.lo, f1.hi);
        }
        r0 = reduce_acc_wide(s0, P);
        r1 = reduce_acc_wide(s1, P);
        return;
    }
#endif
#pragma unroll
    for (u32 t = 0; t < NT; ++t) {
        Cols a0, a1;
        a0.x = r0;
        a1.x = r1;
#pragma unroll
        for (u32 dg = 0; dg < dnum; ++dg) {
            const Dig<SH::S> xd = split<SH::S>(x[t][dg]);
            a0.mac(xd, packed_dig<SH::S>(sk[((t * E) + 2 * dg) * kThreads + tid]));
            a1.mac(xd, packed_dig<SH::S>(sk[((t * E) + 2 * dg + 1) * kThreads + tid]));
        }
        if (r < SH::L) a0.mac(split<SH::S>(c[t]), packed_dig<SH::S>(sk[((t * E) + 2 * dnum) * kThreads + tid]));
        r0 = reduce_acc(a0.fold<SH::S>(), P);
        r1 = reduce_acc(a1.fold<SH::S>(), P);
    }
}
template <typename SH>
__global__ void __launch_bounds__(kThreads, HGM_PLAN_MINB) k_ks_plan(DevCtx cx, u32 n_groups, const PlanGroup* groups,
                                                         const u64* const* mkey, const u32* g,
                                                         const u64* const* D, const u64* const* c0,
                                                         u64* const* out) {
    extern __shared__ u64 sk[];  // [chunk terms][2 dnum + 1][kThreads]
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, R = SH::R, dnum = SH::dnum, logN = dp->logN, tid = threadIdx.x;
    constexpr u32 E = 2 * SH::dnum + 1;
    for (u32 grp = blockIdx.y; grp < n_groups; grp += gridDim.y) {
        const PlanGroup G = groups[grp];
        COEF_LOOP {
            for (u32 t0 = 0; t0 < G.nterms; t0 += kPlanTerms) {
                const u32 nt = min(kPlanTerms, G.nterms - t0);
                u32 src[kPlanTerms];
#pragma unroll
                for (u32 t = 0; t < kPlanTerms; ++t) {
                    const u32 ge = t < nt ? g[G.term0 + t0 + t] : 1;
                    src[t] = ge == 1 ? j : galois_src(j, ge, logN);
                }
                for (u32 r = 0; r < R; ++r) {
                    const Prime& P = dp->pr[r];
                    for (u32 t = 0; t < nt; ++t) {
                        const u64* k = mkey[G.term0 + t0 + t];
#pragma unroll
                        for (u32 dg = 0; dg < dnum; ++dg) {
                            sk[((t * E) + 2 * dg) * kThreads + tid] = __ldg(k + (((size_t)dg * 2 + 0) * R + r) * N + j);
                            sk[((t * E) + 2 * dg + 1) * kThreads + tid] = __ldg(k + (((size_t)dg * 2 + 1) * R + r) * N + j);
                        }
                        if (r < SH::L) sk[((t * E) + 2 * dnum) * kThreads + tid] = __ldg(k + ((size_t)dnum * 2 * R + r) * N + j);
                    }
                    for (u32 u = 0; u < G.cnt; ++u) {
                        u64* a = out[G.item0 + u];
                        u64 r0 = 0, r1 = 0;
                        if (t0) {
                            r0 = a[(size_t)r * N + j];
                            r1 = a[((size_t)R + r) * N + j];
                        }
                        const u64* const* Dt = D + G.dbase + (size_t)u * G.nterms + t0;
                        const u64* const* Ct = c0 + G.dbase + (size_t)u * G.nterms + t0;
                        if (nt == 1)
                            plan_terms<SH, 1>(P, sk, tid, r, N, src, Dt, Ct, r0, r1);
                        else
                            plan_terms<SH, 2>(P, sk, tid, r, N, src, Dt, Ct, r0, r1);
                        a[(size_t)r * N + j] = r0;
                        a[((size_t)R + r) * N + j] = r1;
                    }
                }
            }
        }
    }
}

// ModDown correction: V[c][i] = sum_k centred([w_k (P/p_k)^-1]_{p_k}) (P/p_k) mod q_i
// V[c][i] = ecoef[c][i] - P^-1 conv[c][i]  (coefficient domain; ecoef optional)
// so that NTT(V) + P^-1 acc = (acc - NTT(conv)) P^-1 + NTT(ecoef) exactly (the NTT
// is linear mod q_i): relinearisation adds e0, e1 without transforming them apart.
template <typename SH>
// Pc (optional): the P limbs' coefficients [n][2][K][N] (an out-of-place INTT, acc
// left intact); otherwise they are read from acc's P limbs, inverse-transformed in place.
__global__ void __launch_bounds__(kThreads, 4) k_moddown_conv(DevCtx cx, u32 n, const u64* const* acc, const u64* const* ecoef, u64* V,
                                                               const u64* Pc) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, K = SH::K, R = SH::R;
    ITEM_LOOP {
        const u32 c = blockIdx.z;
        // P limb k: Pc's [item][c][k], or acc's limb L + k
        const u64* pl = Pc ? Pc + ((size_t)item * 2 + c) * K * N : acc[item] + ((size_t)c * R + L) * N;
        const u64* ec = ecoef ? ecoef[item] + (size_t)c * L * N : nullptr;
        u64* v = V + ((size_t)item * 2 + c) * L * N;
        COEF_LOOP {
            u64 z[kMaxK];
            for (u32 k = 0; k < K; ++k) {
                const u64 p = dp->pr[L + k].q;
                z[k] = shoup_mul(pl[(size_t)k * N + j], dp->phat_inv_n[k], dp->phat_inv_n_sh[k], p);
            }
            for (u32 i = 0; i < L; ++i) {
                const u64 q = dp->pr[i].q;
                u64 conv;
                if (K == 1) {  // P/p_0 = 1: the conversion is the centred lift itself
                    conv = centred_lift(z[0], dp->pr[L].q, q);
                } else {
                    Cols s;
                    for (u32 k = 0; k < K; ++k)
                        s.mac(split<SH::S>(centred_lift(z[k], dp->pr[L + k].q, q)), split<SH::S>(dp->phat_mod_q[k][i]));
                    conv = reduce_acc(s.fold<SH::S>(), dp->pr[i]);
                }
                const u64 scaled = shoup_mul(conv, dp->P_inv_q[i], dp->P_inv_q_sh[i], q);
                v[(size_t)i * N + j] = sub_mod(ec ? ec[(size_t)i * N + j] : 0, scaled, q);
            }
        }
    }
}

// out_c = NTT(V_c) + P^-1 acc_c  (+ addn[galois_src] for c = 0)
template <typename SH>
__global__ void k_ks_finish(DevCtx cx, u32 n, const u64* const* acc, const u64* V, const u64* const* addn,
                            const u32* g, u64* const* out, u32 pre) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, R = SH::R, logN = dp->logN;
    ITEM_LOOP {
        const u64* a = acc[item];
        const u64* v = V + (size_t)item * 2 * L * N;
        const u64* x0 = addn ? addn[item] : nullptr;
        const u32 ge = g[item];
        u64* o = out[item];
        COEF_LOOP {
            const u32 src = ge == 1 ? j : galois_src(j, ge, logN);
            for (u32 i = 0; i < L; ++i) {
                const u64 q = dp->pr[i].q;
                const u64 pi = dp->P_inv_q[i], pis = dp->P_inv_q_sh[i];
                const u64 a0 = a[(size_t)i * N + j], a1 = a[((size_t)R + i) * N + j];
                u64 r0 = add_mod(v[(size_t)i * N + j], pre ? a0 : shoup_mul(a0, pi, pis, q), q);
                const u64 r1 = add_mod(v[((size_t)L + i) * N + j], pre ? a1 : shoup_mul(a1, pi, pis, q), q);
                if (x0) r0 = add_mod(r0, x0[(size_t)i * N + src], q);
                o[(size_t)i * N + j] = r0;
                o[((size_t)L + i) * N + j] = r1;
            }
        }
    }
}

// ---------------------------------------------------------------- tensoring
// oracle q_to_b(): exact centred conversion of 4 polys per item, X: [n][4][L][N]
template <typename SH>
__global__ void __launch_bounds__(kThreads, 6) k_q_to_b(DevCtx cx, u32 n, const u64* X, u64* XB) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, K = SH::K, nB = SH::nB;
    ITEM_LOOP {
        const u32 p = blockIdx.z;
        const u64* x = X + ((size_t)item * 4 + p) * L * N;
        u64* xb = XB + ((size_t)item * 4 + p) * nB * N;
        COEF_LOOP {
            u64 y[kMaxL];
            Acc128 s{0, 0};
            for (u32 i = 0; i < L; ++i) {
                y[i] = shoup_mul(x[(size_t)i * N + j], dp->qhat_inv_n[i], dp->qhat_inv_n_sh[i], dp->pr[i].q);
                fx_add_small(s, y[i], dp->one_over_q[i]);  // 1/q_i: integer part < 2^32
            }
            const u64 v = fx_round(s);
            Dig<SH::S> yd[kMaxL];
            for (u32 i = 0; i < L; ++i) yd[i] = split<SH::S>(y[i]);
            for (u32 k = 0; k < nB; ++k) {
                // sum_i y_i (Q/q_i) - v Q  (mod b_k), one reduction
                Cols a;
                for (u32 i = 0; i < L; ++i) a.mac(yd[i], packed_dig<SH::S>(dp->qhat_mod_b_pk[i][k]));
                a.add<SH::S>(v * dp->neg_Q_mod_b[k]);  // v <= L: < 2^63, a plain addend
                xb[(size_t)k * N + j] = reduce_acc(a.fold<SH::S>(), dp->pr[L + K + k]);
            }
        }
    }
}

// The same with two adjacent coefficients per thread: 16-byte loads and stores,
// and the conversion constants (uniform loads) and addressing shared by both.
#ifndef HGM_QTOB_PAIR
#define HGM_QTOB_PAIR 1
#endif
template <typename SH>
__global__ void __launch_bounds__(kThreads, HGM_QTOB2_MINB) k_q_to_b2(DevCtx cx, u32 n, const u64* X, u64* XB) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, K = SH::K, nB = SH::nB;
    ITEM_LOOP {
        const u32 p = blockIdx.z;
        const ulonglong2* x = reinterpret_cast<const ulonglong2*>(X + ((size_t)item * 4 + p) * L * N);
        ulonglong2* xb = reinterpret_cast<ulonglong2*>(XB + ((size_t)item * 4 + p) * nB * N);
        const u32 N2 = N / 2;
        for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < N2; j += gridDim.x * blockDim.x) {
            ulonglong2 xv[kMaxL];
            for (u32 i = 0; i < L; ++i) xv[i] = x[(size_t)i * N2 + j];
            u64 y0[kMaxL], y1[kMaxL];
            Acc128 s0{0, 0}, s1{0, 0};
            for (u32 i = 0; i < L; ++i) {
                const u64 qi = dp->pr[i].q, hi = dp->qhat_inv_n[i], hs = dp->qhat_inv_n_sh[i];
                const Frac f = dp->one_over_q[i];
                y0[i] = shoup_mul(xv[i].x, hi, hs, qi);
                y1[i] = shoup_mul(xv[i].y, hi, hs, qi);
                fx_add_small(s0, y0[i], f);
                fx_add_small(s1, y1[i], f);
            }
            const u64 v0 = fx_round(s0), v1 = fx_round(s1);
            for (u32 k = 0; k < nB; ++k) {
                Cols a0, a1;
                for (u32 i = 0; i < L; ++i) {
                    const Dig<SH::S> c = packed_dig<SH::S>(dp->qhat_mod_b_pk[i][k]);
                    a0.mac(split<SH::S>(y0[i]), c);
                    a1.mac(split<SH::S>(y1[i]), c);
                }
                const u64 nq = dp->neg_Q_mod_b[k];
                a0.add<SH::S>(v0 * nq);
                a1.add<SH::S>(v1 * nq);
                const Prime& P = dp->pr[L + K + k];
                ulonglong2 r;
                r.x = reduce_acc(a0.fold<SH::S>(), P);
                r.y = reduce_acc(a1.fold<SH::S>(), P);
                xb[(size_t)k * N2 + j] = r;
            }
        }
    }
}

// tensor over Q ++ B in the NTT domain; T: [n][3][L+nB][N]
template <typename SH>
__global__ void k_tensor(DevCtx cx, u32 n, const u64* const* A,
                         const u64* const* B, const u64* XB, u64* T) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, K = SH::K, nB = SH::nB, D = L + nB;
    ITEM_LOOP {
        const u32 d = blockIdx.z;
        u64 *t0 = T + (((size_t)item * 3 + 0) * D + d) * N, *t1 = T + (((size_t)item * 3 + 1) * D + d) * N,
            *t2 = T + (((size_t)item * 3 + 2) * D + d) * N;
        const u64 *a0, *a1, *b0, *b1;
        const Prime* P;
        if (d < L) {
            a0 = A[item] + (size_t)d * N; a1 = A[item] + (size_t)(L + d) * N;
            b0 = B[item] + (size_t)d * N; b1 = B[item] + (size_t)(L + d) * N;
            P = &dp->pr[d];
        } else {
            const size_t base = (size_t)item * 4 * nB * N + (size_t)(d - L) * N;
            a0 = XB + base; a1 = XB + base + (size_t)nB * N;
            b0 = XB + base + (size_t)2 * nB * N; b1 = XB + base + (size_t)3 * nB * N;
            P = &dp->pr[L + K + (d - L)];
        }
        COEF_LOOP {
            const Dig<SH::S> x0 = split<SH::S>(a0[j]), x1 = split<SH::S>(a1[j]), y0 = split<SH::S>(b0[j]),
                             y1 = split<SH::S>(b1[j]);
            Cols s0, s1, s2;
            s0.mac(x0, y0);
            s1.mac(x0, y1);
            s1.mac(x1, y0);
            s2.mac(x1, y1);
            t0[j] = reduce_acc(s0.fold<SH::S>(), *P);
            t1[j] = reduce_acc(s1.fold<SH::S>(), *P);
            t2[j] = reduce_acc(s2.fold<SH::S>(), *P);
        }
    }
}

// k_tensor with the first Gentleman-Sande stage of the following INTT applied
// to each output pair (2i, 2i+1): the same arithmetic load_first_stage does,
// so the INTT (NttJobs::first_done) starts from plain loads.  One thread per
// coefficient pair, 16-byte loads and stores.
template <typename SH>
__global__ void k_tensor_s1(DevCtx cx, u32 n, const u64* const* A, const u64* const* B, const u64* XB, u64* T) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, K = SH::K, nB = SH::nB, D = L + nB;
    ITEM_LOOP {
        const u32 d = blockIdx.z;
        const u32 pi = d < L ? d : L + K + (d - L);
        const ulonglong2 *a0, *a1, *b0, *b1;
        if (d < L) {
            a0 = reinterpret_cast<const ulonglong2*>(A[item] + (size_t)d * N);
            a1 = reinterpret_cast<const ulonglong2*>(A[item] + (size_t)(L + d) * N);
            b0 = reinterpret_cast<const ulonglong2*>(B[item] + (size_t)d * N);
            b1 = reinterpret_cast<const ulonglong2*>(B[item] + (size_t)(L + d) * N);
        } else {
            const u64* base = XB + (size_t)item * 4 * nB * N + (size_t)(d - L) * N;
            a0 = reinterpret_cast<const ulonglong2*>(base);
            a1 = reinterpret_cast<const ulonglong2*>(base + (size_t)nB * N);
            b0 = reinterpret_cast<const ulonglong2*>(base + (size_t)2 * nB * N);
            b1 = reinterpret_cast<const ulonglong2*>(base + (size_t)3 * nB * N);
        }
        const Prime& P = dp->pr[pi];
        const u64 q = P.q;
        const ulonglong2* tw = reinterpret_cast<const ulonglong2*>(cx.tw + (size_t)pi * 4 * N + 2 * N) + (N >> 1);
        ulonglong2* t0 = reinterpret_cast<ulonglong2*>(T + (((size_t)item * 3 + 0) * D + d) * N);
        ulonglong2* t1 = reinterpret_cast<ulonglong2*>(T + (((size_t)item * 3 + 1) * D + d) * N);
        ulonglong2* t2 = reinterpret_cast<ulonglong2*>(T + (((size_t)item * 3 + 2) * D + d) * N);
        for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < N / 2; i += gridDim.x * blockDim.x) {
            const ulonglong2 x0 = a0[i], x1 = a1[i], y0 = b0[i], y1 = b1[i];
            const ulonglong2 w = __ldg(tw + i);
            u64 r[3][2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const Dig<SH::S> p0 = split<SH::S>(e ? x0.y : x0.x), p1 = split<SH::S>(e ? x1.y : x1.x),
                                 q0 = split<SH::S>(e ? y0.y : y0.x), q1 = split<SH::S>(e ? y1.y : y1.x);
                Cols s0, s1, s2;
                s0.mac(p0, q0);
                s1.mac(p0, q1);
                s1.mac(p1, q0);
                s2.mac(p1, q1);
                r[0][e] = reduce_acc(s0.fold<SH::S>(), P);
                r[1][e] = reduce_acc(s1.fold<SH::S>(), P);
                r[2][e] = reduce_acc(s2.fold<SH::S>(), P);
            }
            ulonglong2* outs[3] = {t0, t1, t2};
#pragma unroll
            for (int p = 0; p < 3; ++p) {
                ulonglong2 v;
                v.x = reduce_once(r[p][0] + r[p][1], q << 1);
                v.y = shoup_lazy3(r[p][0] - r[p][1] + (q << 1), w.x, w.y, q);
                outs[p][i] = v;
            }
        }
    }
}

// Pending products (oracle XCt): T[d] (+)= sum over the items i of
// d's range [off[d], off[d+1]) of tensor(a_i, b_i) over Q ++ B, NTT domain,
// T: [3][L+nB][N] per destination.  a_i, b_i give the Q limbs; their B
// extensions are XB + i * 4 nB N (k_q_to_b's layout).  init[d]: T[d] already
// holds a partial sum to add to.  One thread per coefficient of one limb.
// Karatsuba on the tensor: x0 y1 + x1 y0 = (x0 + x1)(y0 + y1) - x0 y0 - x1 y1,
// three products per item instead of four; products accumulate in Karatsuba
// columns, reduced every kGroup items (the Cols / reduce_acc bounds: 4 products
// of 60-bit residues, 16 of 55-bit ones) into running sums mod q.
template <typename SH>
__global__ void __launch_bounds__(kThreads, HGM_TACC_MINB) k_tensor_acc(DevCtx cx, u32 n, const u32* off, const u64* const* A,
                                                             const u64* const* B, const u64* XB, u64* const* T,
                                                             const unsigned char* init) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, K = SH::K, nB = SH::nB, D = L + nB;
    constexpr u32 kGroup = SH::S == 30 ? 4 : 16;
    ITEM_LOOP {
        const u32 d = blockIdx.z;
        const Prime& P = dp->pr[d < L ? d : L + K + (d - L)];
        const u64 q = P.q;
        const u32 i0 = off[item], i1 = off[item + 1];
        u64* t0 = T[item] + (size_t)d * N;
        u64* t1 = t0 + (size_t)D * N;
        u64* t2 = t1 + (size_t)D * N;
        const bool acc = init[item] != 0;
        COEF_LOOP {
            // chunks of kGroup products (the column sums' range), each chunk's
            // columns starting from the running residues (folded in as x)
            u64 p0 = 0, pm = 0, p2 = 0;
            for (u32 ic = i0; ic < i1; ic += kGroup) {
                const u32 ni = i1 - ic < kGroup ? i1 - ic : kGroup;
                Cols s0, sm, s2;
                s0.x = p0;
                sm.x = pm;
                s2.x = p2;
#pragma unroll
                for (u32 u = 0; u < kGroup; ++u) {
                    if (u >= ni) break;
                    const u32 i = ic + u;
                    const u64 *a0, *a1, *b0, *b1;
                    if (d < L) {
                        a0 = A[i] + (size_t)d * N; a1 = A[i] + (size_t)(L + d) * N;
                        b0 = B[i] + (size_t)d * N; b1 = B[i] + (size_t)(L + d) * N;
                    } else {
                        a0 = XB + ((size_t)i * 4 * nB + (d - L)) * N; a1 = a0 + (size_t)nB * N;
                        b0 = a1 + (size_t)nB * N; b1 = b0 + (size_t)nB * N;
                    }
                    const u64 x0 = a0[j], x1 = a1[j], y0 = b0[j], y1 = b1[j];
                    s0.mac(split<SH::S>(x0), split<SH::S>(y0));
                    s2.mac(split<SH::S>(x1), split<SH::S>(y1));
                    sm.mac(split<SH::S>(add_mod(x0, x1, q)), split<SH::S>(add_mod(y0, y1, q)));
                }
                p0 = reduce_acc(s0.fold<SH::S>(), P);
                pm = reduce_acc(sm.fold<SH::S>(), P);
                p2 = reduce_acc(s2.fold<SH::S>(), P);
            }
            u64 p1 = sub_mod(sub_mod(pm, p0, q), p2, q);
            if (acc) {
                p0 = add_mod(p0, t0[j], q);
                p1 = add_mod(p1, t1[j], q);
                p2 = add_mod(p2, t2[j], q);
            }
            t0[j] = p0;
            t1[j] = p1;
            t2[j] = p2;
        }
    }
}

// out[o] (+)= sum over t in [off[o], off[o+1]) of in[t], over the T region of
// pending buffers ([3][L+nB][N]); init[o]: add to out[o]'s current value.
template <typename SH>
__global__ void k_tsum(DevCtx cx, u32 n, const u32* off, const u64* const* in, u64* const* out,
                       const unsigned char* init) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, K = SH::K, nB = SH::nB, D = L + nB;
    ITEM_LOOP {
        const u32 r = blockIdx.z;  // limb of [3][D]
        const u32 d = r % D;
        const u64 q = dp->pr[d < L ? d : L + K + (d - L)].q;
        u64* o = out[item] + (size_t)r * N;
        const bool acc = init[item] != 0;
        COEF_LOOP {
            u64 s = acc ? o[j] : 0;
            for (u32 t = off[item]; t < off[item + 1]; ++t) s = add_mod(s, in[t][(size_t)r * N + j], q);
            o[j] = s;
        }
    }
}

// oracle scale_round(): round(t x / Q) from Q ++ B residues, then exact B -> Q
template <typename SH>
// Dg (optional, alpha = 1): component 2 is not stored in E but lifted straight
// into the relinearisation digits [n][dnum][R][N] (k_modup_lift's output: digit
// dg = limb dg, centred into every other limb).
__global__ void __launch_bounds__(kThreads, 6) k_scale_round(DevCtx cx, u32 n, const u64* T, u64* E, u64* Dg) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, K = SH::K, nB = SH::nB, D = L + nB;
    ITEM_LOOP {
        const u32 p = blockIdx.z;
        const u64* t = T + ((size_t)item * 3 + p) * D * N;
        u64* e = E + ((size_t)item * 3 + p) * L * N;
        COEF_LOOP {
            u64 a[kMaxL];
            Acc128 s{0, 0};
            for (u32 i = 0; i < L; ++i) {
                a[i] = shoup_mul(t[(size_t)i * N + j], dp->dhat_inv_n[i], dp->dhat_inv_n_sh[i], dp->pr[i].q);
                fx_add(s, a[i], dp->F[i]);
            }
            const u64 rr = fx_round(s);
            Dig<SH::S> ad[kMaxL];
            for (u32 i = 0; i < L; ++i) ad[i] = split<SH::S>(a[i]);
            Dig<SH::S> cb[kMaxB];
            Acc128 s2{0, 0};
            for (u32 k = 0; k < nB; ++k) {
                const u64 b = dp->pr[L + K + k].q;
                // rr + sum_i a_i floor(tB/q_i) + x_b [t/Q]  (mod b_k), one reduction
                Cols acc;
                acc.x = rr;  // rr < L * 2^60
                for (u32 i = 0; i < L; ++i) acc.mac(ad[i], split<SH::S>(dp->W[i][k]));
                const u64 tb = reduce_once(reduce_once(t[(size_t)(L + k) * N + j], b << 1), b);  // [0, 4b) -> [0, b)
                acc.mac(split<SH::S>(tb), split<SH::S>(dp->T_n[k]));
                const u64 c = shoup_mul(reduce_acc(acc.fold<SH::S>(), dp->pr[L + K + k]), dp->bhat_inv[k],
                                        dp->bhat_inv_sh[k], b);
                cb[k] = split<SH::S>(c);
                fx_add_small(s2, c, dp->one_over_b[k]);  // 1/b_k: integer part < 2^32
            }
            const u64 v = fx_round(s2);
            for (u32 i = 0; i < L; ++i) {
                // sum_k c_k (B/b_k) - v B  (mod q_i), one reduction
                Cols acc;
                for (u32 k = 0; k < nB; ++k) acc.mac(cb[k], split<SH::S>(dp->bhat_mod_q[k][i]));
                acc.add<SH::S>(v * dp->neg_B_mod_q[i]);  // v <= nB: < 2^64, a plain addend
                const u64 r = reduce_acc(acc.fold<SH::S>(), dp->pr[i]);
                if (SH::A == 1 && Dg && p == 2) {
                    u64* dgi = Dg + ((size_t)item * SH::dnum + i) * SH::R * N;
                    for (u32 rr2 = 0; rr2 < SH::R; ++rr2)
                        dgi[(size_t)rr2 * N + j] = rr2 == i ? r : centred_lift(r, dp->pr[i].q, dp->pr[rr2].q);
                } else {
                    e[(size_t)i * N + j] = r;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- key generation
template <typename SH>
__global__ void k_keygen_sk(DevCtx cx, u64* S) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, R = SH::R;
    const u32 n = 1;
    ITEM_LOOP {
        COEF_LOOP {
            const i64 s = ternary(cx, kStreamSk, j);
            for (u32 r = 0; r < R; ++r) S[(size_t)r * N + j] = small_to_mod(s, dp->pr[r].q);
        }
    }
}

// Gaussian error for a stream, lifted to `limbs` limbs: E[l][j]
__global__ void k_keygen_err(DevCtx cx, u64 stream, u32 limbs, u64* E) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N;
    const u32 n = 1;
    ITEM_LOOP {
        COEF_LOOP {
            const i64 e = gauss(cx, stream, j, cx.cdt);
            for (u32 r = 0; r < limbs; ++r) E[(size_t)r * N + j] = small_to_mod(e, dp->pr[r].q);
        }
    }
}

template <typename SH>
__global__ void k_keygen_pk(DevCtx cx, const u64* S, const u64* E, u64* pk) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L;
    const u32 n = 1;
    ITEM_LOOP {
        COEF_LOOP {
            for (u32 i = 0; i < L; ++i) {
                const Prime& P = dp->pr[i];
                const u64 a = uniform(cx, kStreamPkA, (u64)i * N + j, P.q);
                pk[(size_t)i * N + j] = sub_mod(E[(size_t)i * N + j], mul_mod(a, S[(size_t)i * N + j], P), P.q);
                pk[(size_t)(L + i) * N + j] = a;
            }
        }
    }
}

// oracle make_key(): key[dg][0][r] = -a s + e + [r in digit dg] P s'; key[dg][1][r] = a
template <typename SH>
__global__ void k_keygen_ks(DevCtx cx, u32 kid, u32 g, const u64* S,
                            const u64* E, u64* key) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, L = SH::L, R = SH::R, A = SH::A, logN = dp->logN;
    const u32 dg = blockIdx.y;
    const u32 n = 1;
    (void)n;
    COEF_LOOP {
        const u32 src = kid == 0 ? j : galois_src(j, g, logN);
        for (u32 r = 0; r < R; ++r) {
            const Prime& P = dp->pr[r];
            const u64 sr = S[(size_t)r * N + j];
            const u64 a = uniform(cx, kStreamKsA | ((u64)kid << 8) | dg, (u64)r * N + j, P.q);
            u64 v = sub_mod(E[((size_t)dg * R + r) * N + j], mul_mod(a, sr, P), P.q);
            if (r < L && r / A == dg) {
                const u64 sp = kid == 0 ? mul_mod(sr, sr, P) : S[(size_t)r * N + src];
                v = add_mod(v, mul_mod(dp->P_mod_q[r], sp, P), P.q);
            }
            key[(((size_t)dg * 2 + 0) * R + r) * N + j] = v;
            key[(((size_t)dg * 2 + 1) * R + r) * N + j] = a;
        }
    }
}

dim3 grid_of(u32 N, u32 n, u32 z = 1) {
    const u32 gx = (N + kThreads - 1) / kThreads;
    return dim3(gx, n < 65535 ? n : 65535, z);
}

u64 mask_hash(const i64* m, size_t S) {
    u64 h = 0x243f6a8885a308d3ULL ^ S;
    for (size_t i = 0; i < S; ++i) h = (h ^ (u64)m[i]) * 0x100000001b3ULL;  // collisions: content compared
    return mix64(h);
}

}  // namespace

// ==================================================================== PinnedRing
PinnedRing::PinnedRing(size_t bytes) : cap_(bytes) {
    HGM_CUDA(cudaMallocHost(&host_, cap_));
    HGM_CUDA(cudaMalloc(&dev_, cap_));
}
PinnedRing::~PinnedRing() {
    for (auto& m : marks_) cudaEventDestroy(m.ev);
    for (auto e : free_events_) cudaEventDestroy(e);
    cudaFreeHost(host_);
    cudaFree(dev_);
}
char* PinnedRing::reserve(size_t bytes) {
    const size_t need = (bytes + 255) & ~size_t(255);
    if (need > cap_) throw std::length_error("staging ring too small for an upload of " + std::to_string(bytes));
    size_t b = head_;
    if (b + need > cap_) b = 0;
    const size_t e = b + need;
    // retire (wait for) any in-flight copy whose host range intersects [b, e)
    for (size_t i = 0; i < marks_.size();) {
        const size_t mb = marks_[i].end >> 32, me = marks_[i].end & 0xffffffffULL;
        if (mb < e && b < me) {
            HGM_CUDA(cudaEventSynchronize(marks_[i].ev));
            free_events_.push_back(marks_[i].ev);
            marks_.erase(marks_.begin() + i);
        } else {
            // drop completed marks opportunistically
            if (cudaEventQuery(marks_[i].ev) == cudaSuccess) {
                free_events_.push_back(marks_[i].ev);
                marks_.erase(marks_.begin() + i);
            } else {
                ++i;
            }
        }
    }
    head_ = e;
    return host_ + b;
}

void* PinnedRing::commit(char* host, size_t bytes, cudaStream_t s) {
    const size_t b = (size_t)(host - host_), e = b + ((bytes + 255) & ~size_t(255));
    HGM_CUDA(cudaMemcpyAsync(dev_ + b, host, bytes, cudaMemcpyHostToDevice, s));
    cudaEvent_t ev;
    if (free_events_.empty()) {
        HGM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    } else {
        ev = free_events_.back();
        free_events_.pop_back();
    }
    HGM_CUDA(cudaEventRecord(ev, s));
    marks_.push_back(Mark{((size_t)b << 32) | e, ev});
    return dev_ + b;
}

void* PinnedRing::upload(const void* src, size_t bytes, cudaStream_t s) {
    char* h = reserve(bytes);
    std::memcpy(h, src, bytes);
    return commit(h, bytes, s);
}

// ==================================================================== Context
namespace {
// Makes the context's device current for a scope and restores the caller's.
struct DeviceScope {
    int prev = -1, want;
    explicit DeviceScope(int d) : want(d) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != want) cudaSetDevice(want);
    }
    ~DeviceScope() {
        if (prev >= 0 && prev != want) cudaSetDevice(prev);
    }
};
}  // namespace

Context::Context(int param_id, u64 seed, int device, bool keyless, const u32* csprng_key)
    : device_(device), keyless_(keyless) {
    hp_ = make_params(param_id, seed);
    // all primes of one set share their bit length (centred_lift relies on it)
    for (size_t r = 1; r < hp_.primes.size(); ++r)
        if (64 - __builtin_clzll(hp_.primes[r]) != 64 - __builtin_clzll(hp_.primes[0]))
            throw std::logic_error("prime set has mixed bit lengths");
    HGM_CUDA(cudaSetDevice(device_));
    HGM_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    HGM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device_));
    u64 threshold = ~0ULL;
    HGM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    ring_ = std::make_unique<PinnedRing>((size_t)64 << 20);

    const size_t N = hp_.N;
    HGM_CUDA(cudaMalloc(&d_tw_, hp_.tw.size() * 8));
    HGM_CUDA(cudaMemcpy(d_tw_, hp_.tw.data(), hp_.tw.size() * 8, cudaMemcpyHostToDevice));
    HGM_CUDA(cudaMalloc(&d_slot_, N * 4));
    HGM_CUDA(cudaMemcpy(d_slot_, hp_.slot_ntt.data(), N * 4, cudaMemcpyHostToDevice));
    HGM_CUDA(cudaMalloc(&d_cdt_, sizeof(kGaussCdt)));
    HGM_CUDA(cudaMemcpy(d_cdt_, kGaussCdt, sizeof(kGaussCdt), cudaMemcpyHostToDevice));
    hp_.dev.tw = d_tw_;
    hp_.dev.slot_ntt = d_slot_;
    hp_.dev.cdt = d_cdt_;
    HGM_CUDA(cudaMalloc(&dp_, sizeof(DevParams)));
    HGM_CUDA(cudaMemcpy(dp_, &hp_.dev, sizeof(DevParams), cudaMemcpyHostToDevice));
    // parameter-set constants -> __constant__ (identical for every context of the set)
    HGM_CUDA(cudaMemcpyToSymbol(c_dp, &hp_.dev, sizeof(DevParams), (size_t)param_id * sizeof(DevParams)));
    ntt_upload_params(param_id, hp_.dev);
    HGM_CUDA(cudaGetLastError());
    cx_.tw = d_tw_;
    cx_.slot_ntt = d_slot_;
    cx_.cdt = d_cdt_;
    cx_.seed = seed;
    cx_.pid = (u32)param_id;
    if (csprng_key) {
        cx_.csprng = 1;
        for (int i = 0; i < 8; ++i) cx_.ck[i] = csprng_key[i];
    }
    if (!keyless_) build_keys();
}

Context::~Context() {
    DeviceScope dev(device_);
    cudaStreamSynchronize(stream_);
    for (auto& kv : keys_) cudaFree(kv.second);
    for (auto& kv : masks_)
        for (auto& e : kv.second) cudaFreeAsync(e.dev, stream_);
    for (auto& kv : mkeys_) cudaFreeAsync(kv.second.dev, stream_);
    cudaStreamSynchronize(stream_);
    cudaFree(d_sk_);
    cudaFree(d_pk_);
    cudaFree(dp_);
    cudaFree(d_tw_);
    cudaFree(d_slot_);
    cudaFree(d_cdt_);
    ring_.reset();
    if (dl_host_) cudaFreeHost(dl_host_);
    for (u32* p : slot_host_)
        if (p) cudaFreeHost(p);
    cudaStreamDestroy(stream_);
}

u64* Context::alloc(size_t words) {
    void* p = nullptr;
    HGM_CUDA(cudaMallocAsync(&p, words * 8, stream_));
    return static_cast<u64*>(p);
}
void Context::release(void* p) {
    if (p) HGM_CUDA(cudaFreeAsync(p, stream_));
}
void Context::sync() { HGM_CUDA(cudaStreamSynchronize(stream_)); }

void Context::ntt(bool forward, const NttJobs& jobs) {
    if (jobs.count == 0) return;
    launches_ += hp_.logN > 13 ? 2 : 1;
    if (forward)
        ntt_forward(cx_, hp_.dev, jobs, stream_);
    else
        ntt_inverse(cx_, hp_.dev, jobs, stream_);
    HGM_CUDA(cudaGetLastError());
}

void Context::build_keys() {
    const u32 N = hp_.N, L = hp_.L, R = hp_.R;
    HGM_CUDA(cudaMalloc(&d_sk_, (size_t)R * N * 8));
    HGM_CUDA(cudaMalloc(&d_pk_, (size_t)2 * L * N * 8));
    if (hp_.L == 3) k_keygen_sk<ShapeQ3><<<grid_of(N, 1), kThreads, 0, stream_>>>(cx_, d_sk_); else k_keygen_sk<ShapeQ8><<<grid_of(N, 1), kThreads, 0, stream_>>>(cx_, d_sk_); ++launches_;
    ntt(true, jobs_contig(d_sk_, R, 0, R));
    u64* E = alloc((size_t)L * N);
    k_keygen_err<<<grid_of(N, 1), kThreads, 0, stream_>>>(cx_, kStreamPkE, L, E); ++launches_;
    ntt(true, jobs_contig(E, L, 0, L));
    if (hp_.L == 3) k_keygen_pk<ShapeQ3><<<grid_of(N, 1), kThreads, 0, stream_>>>(cx_, d_sk_, E, d_pk_); else k_keygen_pk<ShapeQ8><<<grid_of(N, 1), kThreads, 0, stream_>>>(cx_, d_sk_, E, d_pk_); ++launches_;
    release(E);
    HGM_CUDA(cudaGetLastError());
    ks_key(0);  // relinearisation key
}

u32 Context::galois_of(i64 z, u32 N) {
    const i64 H = N / 2;
    const i64 zz = ((z % H) + H) % H;
    u64 g = 1;
    for (i64 i = 0; i < zz; ++i) g = g * 3 % (2 * (u64)N);
    return (u32)g;
}

const u64* Context::ks_key(u32 kid) {
    {
        std::lock_guard<std::mutex> lk(key_mu_);
        auto it = keys_.find(kid);
        if (it != keys_.end()) return it->second;
    }
    if (!d_sk_)
        throw std::invalid_argument("no key-switching key for Galois element " + std::to_string(kid) +
                                    (kid == 0 ? " (relinearisation)" : "") +
                                    " and no secret key to generate it: upload it with hgm_key_upload");
    const u32 N = hp_.N, R = hp_.R, dnum = hp_.dnum;
    u64* key = nullptr;
    HGM_CUDA(cudaMallocAsync((void**)&key, (size_t)dnum * 2 * R * N * 8, stream_));
    u64* E = alloc((size_t)dnum * R * N);
    for (u32 dg = 0; dg < dnum; ++dg) {
        k_keygen_err<<<grid_of(N, 1), kThreads, 0, stream_>>>(cx_, kStreamKsE | ((u64)kid << 8) | dg, R,
                                                             E + (size_t)dg * R * N);
        ++launches_;
    }
    ntt(true, jobs_contig(E, dnum * R, 0, R));
    if (hp_.L == 3) k_keygen_ks<ShapeQ3><<<dim3((N + kThreads - 1) / kThreads, dnum), kThreads, 0, stream_>>>(cx_, kid, kid, d_sk_, E, key); else k_keygen_ks<ShapeQ8><<<dim3((N + kThreads - 1) / kThreads, dnum), kThreads, 0, stream_>>>(cx_, kid, kid, d_sk_, E, key); ++launches_;
    // k_ks_inner (the only reader) takes the key in packed digit form
    const size_t kw = (size_t)dnum * 2 * R * N;
    const dim3 kg((unsigned)((kw + 4 * kThreads - 1) / (4 * kThreads)));  // 1-D: each word converted once
    if (hp_.L == 3) k_mask_digits<ShapeQ3><<<kg, kThreads, 0, stream_>>>(key, kw); else k_mask_digits<ShapeQ8><<<kg, kThreads, 0, stream_>>>(key, kw);
    ++launches_;
    release(E);
    HGM_CUDA(cudaGetLastError());
    std::lock_guard<std::mutex> lk(key_mu_);
    keys_.emplace(kid, key);
    return key;
}

void Context::ensure_galois_keys(const std::vector<u32>& elements) {
    for (u32 g : elements)
        if (g != 1) ks_key(g);
}

size_t Context::key_words(int kind) const {
    const size_t N = hp_.N;
    switch (kind) {
        case 0: return (size_t)hp_.R * N;
        case 1: return (size_t)2 * hp_.L * N;
        case 2: return (size_t)hp_.dnum * 2 * hp_.R * N;
        default: throw std::invalid_argument("key kind must be 0 (secret), 1 (public) or 2 (switching)");
    }
}

namespace {
// every word of a [..][limbs][N] key image canonical under its limb's prime
void check_canonical(const HostParams& hp, const u64* w, size_t words, u32 limbs) {
    for (size_t i = 0; i < words; ++i)
        if (w[i] >= hp.primes[(i / hp.N) % limbs]) throw std::invalid_argument("non-canonical key residue");
}
}  // namespace

void Context::upload_key(int kind, u32 elt, const u64* host, size_t words) {
    const size_t W = key_words(kind);
    if (words != W) throw std::invalid_argument("key size mismatch: " + std::to_string(words) + " words, expected " +
                                                std::to_string(W));
    if (kind == 2 && elt != 0 && (elt % 2 == 0 || elt >= 2 * hp_.N))
        throw std::invalid_argument("Galois element must be odd and below 2N (0 = relinearisation)");
    check_canonical(hp_, host, W, kind == 1 ? hp_.L : hp_.R);
    u64* dst = nullptr;
    HGM_CUDA(cudaMalloc((void**)&dst, W * 8));
    HGM_CUDA(cudaMemcpyAsync(dst, host, W * 8, cudaMemcpyHostToDevice, stream_));
    if (kind == 2) {  // k_ks_inner reads keys in packed digit form
        const dim3 kg((unsigned)((W + 4 * kThreads - 1) / (4 * kThreads)));
        if (hp_.L == 3) k_mask_digits<ShapeQ3><<<kg, kThreads, 0, stream_>>>(dst, W); else k_mask_digits<ShapeQ8><<<kg, kThreads, 0, stream_>>>(dst, W);
        ++launches_;
    }
    HGM_CUDA(cudaGetLastError());
    sync();
    u64* old = nullptr;
    if (kind == 0) {
        old = d_sk_;
        d_sk_ = dst;
    } else if (kind == 1) {
        old = d_pk_;
        d_pk_ = dst;
    } else {
        std::lock_guard<std::mutex> lk(key_mu_);
        auto it = keys_.find(elt);
        if (it != keys_.end()) old = it->second;
        keys_[elt] = dst;
    }
    if (kind == 2 && old) drop_masked_keys();  // masked keys derive from the replaced key
    if (old) HGM_CUDA(cudaFree(old));
}

void Context::export_key(int kind, u32 elt, u64* host) {
    const size_t W = key_words(kind);
    const u64* src = kind == 0 ? d_sk_ : kind == 1 ? d_pk_ : ks_key(elt);
    if (!src) throw std::invalid_argument(kind == 0 ? "context holds no secret key" : "context holds no public key");
    sync();
    HGM_CUDA(cudaMemcpy(host, src, W * 8, cudaMemcpyDeviceToHost));
    if (kind == 2) {  // unpack the digit form: v = l + h 2^S
        const int S = hp_.L == 3 ? ShapeQ3::S : ShapeQ8::S;
        for (size_t i = 0; i < W; ++i) host[i] = (host[i] & 0xffffffffULL) + ((host[i] >> 32) << S);
    }
}

void Context::drop_secret() {
    sync();
    if (d_sk_) {
        // overwrite before freeing: the allocation may be handed out again
        HGM_CUDA(cudaMemset(d_sk_, 0, (size_t)hp_.R * hp_.N * 8));
        HGM_CUDA(cudaFree(d_sk_));
    }
    d_sk_ = nullptr;
}

size_t Context::key_count() const {
    std::lock_guard<std::mutex> lk(key_mu_);
    return keys_.size();
}

const u64* Context::mask_plain(const i64* mask, size_t S, u64 stable_id) {
    if (stable_id) {
        std::lock_guard<std::mutex> lk(mask_mu_);
        auto it = masks_by_id_.find(stable_id);
        if (it != masks_by_id_.end()) {
            it->second->tick = ++mask_tick_;
            return it->second->dev;
        }
    }
    const u64 h = mask_hash(mask, S);
    std::lock_guard<std::mutex> lk(mask_mu_);
    auto& bucket = masks_[h];
    for (auto& e : bucket)
        if (e.content.size() == S && std::equal(e.content.begin(), e.content.end(), mask)) {
            e.tick = ++mask_tick_;
            if (stable_id) {
                masks_by_id_.emplace(stable_id, &e);
                e.ids.push_back(stable_id);
            }
            return e.dev;
        }
    const u32 N = hp_.N, L = hp_.L;
    std::vector<u32> padded(N / 2, 0);
    for (size_t j = 0; j < S; ++j) padded[j] = to_slot_residue(mask[j]);
    const u32* dvals = upload(padded);
    std::vector<u32> Sv{(u32)S};
    const u32* dS = upload(Sv);
    u64* m = alloc(N);
    k_encode_scatter<<<grid_of(N, 1), kThreads, 0, stream_>>>(cx_, 1, dvals, dS, m); ++launches_;
    NttJobs tj = jobs_contig(m, 1, kTIndex, 1);
    ntt(false, tj);
    u64* out = nullptr;
    // over Q ++ P: the P limbs mask pending key switches (k_lincomb over R limbs)
    const u32 R = hp_.R;
    HGM_CUDA(cudaMallocAsync((void**)&out, (size_t)R * N * 8, stream_));
    if (hp_.L == 3) k_mask_lift<ShapeQ3><<<grid_of(N, 1), kThreads, 0, stream_>>>(cx_, m, out); else k_mask_lift<ShapeQ8><<<grid_of(N, 1), kThreads, 0, stream_>>>(cx_, m, out); ++launches_;
    ntt(true, jobs_contig(out, R, 0, R));
    if (hp_.L == 3) k_mask_digits<ShapeQ3><<<grid_of(N, 1), kThreads, 0, stream_>>>(out, (size_t)R * N); else k_mask_digits<ShapeQ8><<<grid_of(N, 1), kThreads, 0, stream_>>>(out, (size_t)R * N);
    ++launches_;
    release(m);
    HGM_CUDA(cudaGetLastError());
    bucket.push_back(MaskEntry{std::vector<i64>(mask, mask + S), out, ++mask_tick_, {}});
    mask_bytes_ += (size_t)R * N * 8;
    if (stable_id) {
        masks_by_id_.emplace(stable_id, &bucket.back());
        bucket.back().ids.push_back(stable_id);
    }
    return out;
}

size_t Context::mask_budget() const {
    static const size_t env = [] {
        const char* e = std::getenv("HGM_MASK_CACHE_MB");
        return e ? (size_t)std::atoll(e) << 20 : (size_t)0;
    }();
    if (env) return env;
    if (mask_budget_ == 0) {  // once per context (cudaMemGetInfo is not free)
        size_t free_b = 0, total_b = 0;
        mask_budget_ = (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || total_b == 0)
                           ? (size_t)4 << 30
                           : std::min<size_t>((size_t)8 << 30, total_b / 16);
    }
    return mask_budget_;
}

void Context::trim_mask_cache() {
    std::lock_guard<std::mutex> lk(mask_mu_);
    const size_t budget = mask_budget();
    if (mask_bytes_ <= budget) return;
    std::vector<std::pair<u64, std::pair<u64, MaskEntry*>>> all;  // (tick, (hash, entry))
    for (auto& kv : masks_)
        for (auto& e : kv.second) all.push_back({e.tick, {kv.first, &e}});
    std::sort(all.begin(), all.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    const size_t each = (size_t)hp_.R * hp_.N * 8;
    for (auto& a : all) {
        if (mask_bytes_ <= budget / 2) break;  // hysteresis: trim to half the budget
        MaskEntry* e = a.second.second;
        for (u64 id : e->ids) masks_by_id_.erase(id);
        HGM_CUDA(cudaFreeAsync(e->dev, stream_));
        auto& bucket = masks_[a.second.first];
        bucket.remove_if([e](const MaskEntry& x) { return &x == e; });
        if (bucket.empty()) masks_.erase(a.second.first);
        mask_bytes_ -= each;
    }
}

// ------------------------------------------------------------------ primitives
void Context::encrypt(int n, const i64* const* host_vals, const size_t* S, const u64* counters,
                      u64* const* out) {
    encrypt_impl(n, host_vals, S, counters, nullptr, out);
}

void Context::encrypt_noise(int n, const i64* const* host_vals, const size_t* S, const i64* noise,
                            u64* const* out) {
    const size_t N = hp_.N;
    for (size_t i = 0; i < (size_t)n * 3 * N; ++i) {
        const bool is_u = (i / N) % 3 == 0;
        const i64 v = noise[i];
        if (is_u ? (v < -1 || v > 1) : (v < -(i64)1e9 || v > (i64)1e9))
            throw std::invalid_argument(is_u ? "u must be ternary" : "noise coefficient out of range");
    }
    encrypt_impl(n, host_vals, S, nullptr, noise, out);
}

void Context::encrypt_impl(int n, const i64* const* host_vals, const size_t* S, const u64* counters,
                           const i64* noise, u64* const* out) {
    if (n <= 0) return;
    if (!d_pk_) throw std::invalid_argument("context holds no public key: upload it with hgm_key_upload");
    if (n > kChunkEnc) {
        for (int c0 = 0; c0 < n; c0 += kChunkEnc) {
            const int cn = std::min(kChunkEnc, n - c0);
            encrypt_impl(cn, host_vals + c0, S + c0, counters ? counters + c0 : nullptr,
                         noise ? noise + (size_t)c0 * 3 * hp_.N : nullptr, out + c0);
        }
        return;
    }
    const u32 N = hp_.N, L = hp_.L, H = N / 2;
    std::vector<u32> Sv(n);
    std::vector<u64> ctr(n, 0);
    if (counters) std::copy(counters, counters + n, ctr.begin());
    std::vector<u64*> outs(out, out + n);
    for (int i = 0; i < n; ++i) Sv[i] = (u32)S[i];
    // slot values -> residues mod t, written straight into pinned staging
    const size_t vbytes = (size_t)n * H * sizeof(u32);
    u32* hv = reinterpret_cast<u32*>(ring_->reserve(vbytes));
    parallel_for((size_t)n, [&](size_t i) {
        const i64* src = host_vals[i];
        u32* dst = hv + i * H;
        for (size_t j = 0; j < S[i]; ++j) dst[j] = to_slot_residue(src[j]);
    });
    const u32* dvals = static_cast<const u32*>(ring_->commit(reinterpret_cast<char*>(hv), vbytes, stream_));
    const u32* dS = upload(Sv);
    const u64* dctr = upload(ctr);
    u64* const* dout = upload(outs);
    u64* M = alloc((size_t)n * N);
    u64* U = alloc((size_t)n * L * N);
    i64* dnoise = nullptr;
    if (noise) {
        dnoise = reinterpret_cast<i64*>(alloc((size_t)n * 3 * N));
        HGM_CUDA(cudaMemcpyAsync(dnoise, noise, (size_t)n * 3 * N * 8, cudaMemcpyHostToDevice, stream_));
    }
    k_encode_scatter<<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, dvals, dS, M); ++launches_;
    ntt(false, jobs_contig(M, n, kTIndex, 1));
    if (hp_.L == 3) k_enc_lift<ShapeQ3><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, M, dctr, dnoise, U, dout); else k_enc_lift<ShapeQ8><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, M, dctr, dnoise, U, dout); ++launches_;
    ntt(true, jobs_contig(U, n * L, 0, L));
    NttJobs cj;
    std::vector<u64*> limbs((size_t)n * 2 * L);
    for (int i = 0; i < n; ++i)
        for (u32 w = 0; w < 2 * L; ++w) limbs[(size_t)i * 2 * L + w] = out[i] + (size_t)w * N;
    cj.ptrs = upload(limbs);
    cj.count = n * 2 * L;
    cj.period = L;
    for (u32 i = 0; i < L; ++i) cj.prime[i] = (unsigned char)i;
    ntt(true, cj);
    if (hp_.L == 3) k_enc_finish<ShapeQ3><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, U, d_pk_, dout); else k_enc_finish<ShapeQ8><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, U, d_pk_, dout); ++launches_;
    release(M);
    release(U);
    if (dnoise) {
        release(dnoise);
        sync();  // the caller's noise buffer was copied from pageable memory; keep the call synchronous
    }
    HGM_CUDA(cudaGetLastError());
}

void Context::decrypt_to(int n, const u64* const* in, const size_t* S, u32* host) {
    if (n <= 0) return;
    if (!d_sk_) throw std::invalid_argument("context holds no secret key (a cloud context cannot decrypt)");
    const u32 N = hp_.N, L = hp_.L, H = N / 2;
    for (int c0 = 0; c0 < n; c0 += kChunkDec) {
        const int cn = std::min(kChunkDec, n - c0);
        std::vector<const u64*> ins(in + c0, in + c0 + cn);
        std::vector<u32> Sv(cn);
        for (int i = 0; i < cn; ++i) Sv[i] = (u32)S[c0 + i];
        const u64* const* din = upload(ins);
        const u32* dS = upload(Sv);
        u64* X = alloc((size_t)cn * L * N);
        u64* M = alloc((size_t)cn * N);
        u32* O = reinterpret_cast<u32*>(alloc(((size_t)cn * H + 1) / 2));
        if (hp_.L == 3) k_dec_phase<ShapeQ3><<<grid_of(N, cn), kThreads, 0, stream_>>>(cx_, cn, din, d_sk_, X); else k_dec_phase<ShapeQ8><<<grid_of(N, cn), kThreads, 0, stream_>>>(cx_, cn, din, d_sk_, X); ++launches_;
        ntt(false, jobs_contig(X, cn * L, 0, L));
        if (hp_.L == 3) k_dec_round<ShapeQ3><<<grid_of(N, cn), kThreads, 0, stream_>>>(cx_, cn, X, M); else k_dec_round<ShapeQ8><<<grid_of(N, cn), kThreads, 0, stream_>>>(cx_, cn, X, M); ++launches_;
        ntt(true, jobs_contig(M, cn, kTIndex, 1));
        k_dec_gather<<<grid_of(H, cn), kThreads, 0, stream_>>>(cx_, cn, M, dS, O); ++launches_;
        HGM_CUDA(cudaMemcpyAsync(host + (size_t)c0 * H, O, (size_t)cn * H * sizeof(u32), cudaMemcpyDeviceToHost,
                                 stream_));
        release(X);
        release(M);
        release(O);
    }
    HGM_CUDA(cudaGetLastError());
}

void Context::decrypt(int n, const u64* const* in, const size_t* S, i64* const* host_out) {
    if (n <= 0) return;
    const u32 H = hp_.N / 2;
    const u32* host = static_cast<const u32*>(download_buffer((size_t)n * H * sizeof(u32)));
    decrypt_to(n, in, S, const_cast<u32*>(host));
    sync();
    parallel_for((size_t)n, [&](size_t i) {
        const u32* src = host + i * H;
        i64* dst = host_out[i];
        for (size_t j = 0; j < S[i]; ++j) dst[j] = (i64)src[j];
    });
}

u32* Context::pinned_slot(int i, size_t bytes) {
    if (bytes > slot_cap_[i]) {
        if (slot_host_[i]) HGM_CUDA(cudaFreeHost(slot_host_[i]));
        slot_host_[i] = nullptr;
        HGM_CUDA(cudaMallocHost((void**)&slot_host_[i], bytes));
        slot_cap_[i] = bytes;
    }
    return slot_host_[i];
}

void* Context::download_buffer(size_t bytes) {
    if (bytes > dl_cap_) {
        if (dl_host_) HGM_CUDA(cudaFreeHost(dl_host_));
        dl_host_ = nullptr;
        HGM_CUDA(cudaMallocHost(&dl_host_, bytes));
        dl_cap_ = bytes;
    }
    return dl_host_;
}

void Context::add(int n, const u64* const* a, const u64* const* b, u64* const* out) {
    if (n <= 0) return;
    if (n > kChunkLin) {
        for (int c0 = 0; c0 < n; c0 += kChunkLin) {
            const int cn = std::min(kChunkLin, n - c0);
            add(cn, a + c0, b + c0, out + c0);
        }
        return;
    }
    std::vector<const u64*> va(a, a + n), vb(b, b + n);
    std::vector<u64*> vo(out, out + n);
    if (hp_.L == 3) k_add<ShapeQ3><<<grid_of(hp_.N, n, 1), kThreads, 0, stream_>>>(cx_, n, upload(va), upload(vb), upload(vo)); else k_add<ShapeQ8><<<grid_of(hp_.N, n, 1), kThreads, 0, stream_>>>(cx_, n, upload(va), upload(vb), upload(vo)); ++launches_;
    HGM_CUDA(cudaGetLastError());
}

void Context::copy(int n, const u64* const* in, u64* const* out) {
    if (n <= 0) return;
    if (n > kChunkLin) {
        for (int c0 = 0; c0 < n; c0 += kChunkLin) {
            const int cn = std::min(kChunkLin, n - c0);
            copy(cn, in + c0, out + c0);
        }
        return;
    }
    std::vector<const u64*> vi(in, in + n);
    std::vector<u64*> vo(out, out + n);
    k_copy<<<grid_of(hp_.N, n), kThreads, 0, stream_>>>(n, ct_words(), upload(vi), upload(vo)); ++launches_;
    HGM_CUDA(cudaGetLastError());
}

namespace {
// every term of every output has a mask (k_lincomb_masked applies); HGM_LC_MASKED=0 disables
bool all_masked(const std::vector<const u64*>& masks) {
    static const bool on = [] {
        const char* e = std::getenv("HGM_LC_MASKED");
        return !(e && e[0] == '0');
    }();
    if (!on || masks.empty()) return false;
    for (const u64* m : masks)
        if (!m) return false;
    return true;
}
}  // namespace

void Context::lincomb(int n_out, const u32* off, const u64* const* in, const u64* const* mask,
                      u64* const* out) {
    if (n_out <= 0) return;
    if (n_out > kChunkLin) {
        for (int c0 = 0; c0 < n_out; c0 += kChunkLin) {
            const int cn = std::min(kChunkLin, n_out - c0);
            std::vector<u32> sub(cn + 1);
            for (int i = 0; i <= cn; ++i) sub[i] = off[c0 + i] - off[c0];
            lincomb(cn, sub.data(), in + off[c0], mask + off[c0], out + c0);
        }
        return;
    }
    const u32 nt = off[n_out];
    std::vector<u32> voff(off, off + n_out + 1);
    std::vector<const u64*> vin(in, in + nt), vm(mask, mask + nt);
    std::vector<u64*> vo(out, out + n_out);
    if (all_masked(vm)) {
        if (hp_.L == 3)
            k_lincomb_masked<ShapeQ3><<<grid_of(hp_.N, n_out, 1), kThreads, 0, stream_>>>(cx_, n_out, upload(voff), upload(vin), upload(vm), upload(vo));
        else
            k_lincomb_masked<ShapeQ8><<<grid_of(hp_.N, n_out, 1), kThreads, 0, stream_>>>(cx_, n_out, upload(voff), upload(vin), upload(vm), upload(vo));
        ++launches_;
        HGM_CUDA(cudaGetLastError());
        return;
    }
    if (hp_.L == 3) k_lincomb<ShapeQ3><<<grid_of(hp_.N, n_out, 1), kThreads, 0, stream_>>>(cx_, n_out, upload(voff), upload(vin),
                                                                  upload(vm), upload(vo)); else k_lincomb<ShapeQ8><<<grid_of(hp_.N, n_out, 1), kThreads, 0, stream_>>>(cx_, n_out, upload(voff), upload(vin),
                                                                  upload(vm), upload(vo)); ++launches_;
    HGM_CUDA(cudaGetLastError());
}

void Context::modup(int n, const u64* const* ct, u64* const* out) {
    if (n <= 0) return;
    const int chunk = chunk_for((size_t)(hp_.dnum * hp_.R + 2 * hp_.R + 2 * hp_.L) * hp_.N, kChunkKs);
    if (n > chunk) {
        for (int c0 = 0; c0 < n; c0 += chunk) {
            const int cn = std::min(chunk, n - c0);
            modup(cn, ct + c0, out + c0);
        }
        return;
    }
    const u32 N = hp_.N, L = hp_.L, R = hp_.R, dnum = hp_.dnum;
    std::vector<const u64*> vc(ct, ct + n);
    u64* C = alloc((size_t)n * L * N);
    // own_copy: a digit's own limbs are the ciphertext's NTT-domain c1 limbs, copied
    // instead of lifted and transformed back; then the c1 INTT can stay unscaled
    const bool own_copy = ntt_fusable_size(hp_.dev) && !ntt_fusable(hp_.dev, kFuseModUp);
    if (ntt_fusable_size(hp_.dev)) {  // out-of-place INTT of the c1 limbs
        std::vector<const u64*> src((size_t)n * L);
        for (int i = 0; i < n; ++i)
            for (u32 l = 0; l < L; ++l) src[(size_t)i * L + l] = ct[i] + (size_t)(L + l) * N;
        NttJobs cj = jobs_contig(C, n * L, 0, L);
        cj.src = upload(src);
        if (own_copy) cj.unscaled = kLazyOut;  // k_modup_lift: Shoup by dg_hat_inv_n
        ntt(false, cj);
    } else {
        if (hp_.L == 3) k_gather_c1<ShapeQ3><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, upload(vc), C); else k_gather_c1<ShapeQ8><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, upload(vc), C); ++launches_;
        ntt(false, jobs_contig(C, n * L, 0, L));
    }
    // the digits go straight to the per-item outputs (only the opt-in fused
    // ModUp needs one contiguous block, staged and scattered afterwards)
    const bool fused = ntt_fusable(hp_.dev, kFuseModUp);
    const size_t W = modup_words();
    bool contiguous = true;
    for (int i = 1; i < n; ++i)
        if (out[i] != out[0] + (size_t)i * W) contiguous = false;
    u64* const* dpd = upload(std::vector<u64*>(out, out + n));
    if (fused) {
        u64* D = contiguous ? out[0] : alloc((size_t)n * W);
        ntt_modup_fused(cx_, hp_.dev, n, C, (size_t)L * N, D, stream_);
        ++launches_;
        if (!contiguous) {
            std::vector<const u64*> src(n);
            for (int i = 0; i < n; ++i) src[i] = D + (size_t)i * W;
            k_copy<<<grid_of(N, n), kThreads, 0, stream_>>>(n, W, upload(src), dpd); ++launches_;
            release(D);
        }
    } else if (own_copy) {
        if (hp_.L == 3) k_modup_lift<ShapeQ3><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, C, (size_t)L * N, nullptr, 1, dpd); else k_modup_lift<ShapeQ8><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, C, (size_t)L * N, nullptr, 1, dpd); ++launches_;
        // forward NTT of the lifted (non-own) limbs only; own limbs copied from c1
        const u32 A = hp_.alpha, per = dnum * R - L;
        NttJobs dj;
        std::vector<u64*> dl((size_t)n * per);
        std::vector<const u64*> csrc((size_t)n * L);
        std::vector<u64*> cdst((size_t)n * L);
        u32 k = 0;
        for (u32 dg = 0; dg < dnum; ++dg)
            for (u32 r = 0; r < R; ++r)
                if (!(r < L && r / A == dg)) dj.prime[k++] = (unsigned char)r;
        for (int i = 0; i < n; ++i) {
            u64* base = out[i];
            u32 t = 0;
            for (u32 dg = 0; dg < dnum; ++dg)
                for (u32 r = 0; r < R; ++r) {
                    u64* limb = base + ((size_t)dg * R + r) * N;
                    if (r < L && r / A == dg) {
                        csrc[(size_t)i * L + r] = ct[i] + (size_t)(L + r) * N;
                        cdst[(size_t)i * L + r] = limb;
                    } else {
                        dl[(size_t)i * per + t++] = limb;
                    }
                }
        }
        dj.ptrs = upload(dl);
        dj.count = n * per;
        dj.period = per;
        ntt(true, dj);
        k_copy<<<grid_of(N, n * L), kThreads, 0, stream_>>>(n * L, N, upload(csrc), upload(cdst)); ++launches_;
    } else {
        if (hp_.L == 3) k_modup_lift<ShapeQ3><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, C, (size_t)L * N, nullptr, 0, dpd); else k_modup_lift<ShapeQ8><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, C, (size_t)L * N, nullptr, 0, dpd); ++launches_;
        NttJobs dj = jobs_contig(nullptr, n * dnum * R, 0, R);
        std::vector<u64*> dl((size_t)n * dnum * R);
        for (int i = 0; i < n; ++i)
            for (u32 w = 0; w < dnum * R; ++w) dl[(size_t)i * dnum * R + w] = out[i] + (size_t)w * N;
        dj.ptrs = upload(dl);
        ntt(true, dj);
    }
    release(C);
    HGM_CUDA(cudaGetLastError());
}

__global__ void k_fill_residues(DevCtx cx, u64* p, u32 limbs, u32 first_prime, u32 period, u64 seed) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const size_t N = dp->N, words = (size_t)limbs * N;
    for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (size_t)gridDim.x * blockDim.x) {
        const u64 q = dp->pr[first_prime + (u32)((w / N) % period)].q;
        p[w] = prng(seed, 0, w) % q;
    }
}

void Context::fill_residues(u64* p, u32 limbs, u32 first_prime, u32 period, u64 seed) {
    k_fill_residues<<<148 * 8, 256, 0, stream_>>>(cx_, p, limbs, first_prime, period, seed); ++launches_;
    HGM_CUDA(cudaGetLastError());
}

float Context::bench_inner_product(int items, int iters) {
    const u32 N = hp_.N, R = hp_.R, dnum = hp_.dnum;
    const size_t dw = (size_t)dnum * R * N, aw = ks_words();
    u64* D = alloc((size_t)items * dw);
    u64* A = alloc((size_t)items * aw);
    u64* C0 = alloc((size_t)items * ct_words());
    for (int i = 0; i < items; ++i) {
        fill_residues(D + i * dw, dnum * R, 0, R, 11 + i);
        fill_residues(C0 + i * ct_words(), 2 * hp_.L, 0, hp_.L, 7 + i);
    }
    // groups of kKeyReuse rotations share one Galois key (the engine's order)
    std::vector<u32> elts;
    for (int i = 0; i < (items + kKeyReuse - 1) / kKeyReuse; ++i) elts.push_back(galois_of(1 + i % 64, N));
    ensure_galois_keys(elts);
    std::vector<const u64*> dig(items), keys(items), c0(items);
    std::vector<u64*> acc(items);
    std::vector<u32> g(items);
    for (int i = 0; i < items; ++i) {
        dig[i] = D + i * dw;
        g[i] = elts[i / kKeyReuse];
        keys[i] = ks_key(g[i]);
        acc[i] = A + i * aw;
        c0[i] = C0 + i * ct_words();
    }
    inner_product(items, dig.data(), keys.data(), g.data(), acc.data(), c0.data());  // warm-up
    cudaEvent_t e0, e1;
    HGM_CUDA(cudaEventCreate(&e0));
    HGM_CUDA(cudaEventCreate(&e1));
    HGM_CUDA(cudaEventRecord(e0, stream_));
    for (int it = 0; it < iters; ++it)
        inner_product(items, dig.data(), keys.data(), g.data(), acc.data(), c0.data());
    HGM_CUDA(cudaEventRecord(e1, stream_));
    HGM_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    HGM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    release(D);
    release(A);
    release(C0);
    sync();
    return ms / iters;
}

// k_ks_plan in the arrangement the cloud step launches it: tiles of `tile`
// lockstep instances, `sums` masked sums of `terms` rotations per tile, every sum
// of an instance reading that instance's ModUp digits and c0 (one source
// ciphertext, as basic_mm's shifts of sigma(A)), masked keys shared by the tile.
float Context::bench_plan(int instances, int sums, int terms, int tile, int iters) {
    const u32 N = hp_.N, R = hp_.R, dnum = hp_.dnum;
    const size_t dw = (size_t)dnum * R * N, aw = ks_words(), kw = masked_key_words();
    u64* D = alloc((size_t)instances * dw);
    u64* C0 = alloc((size_t)instances * ct_words());
    u64* MK = alloc((size_t)sums * terms * kw);
    u64* A = alloc((size_t)instances * sums * aw);
    for (int i = 0; i < instances; ++i) {
        fill_residues(D + i * dw, dnum * R, 0, R, 11 + i);
        fill_residues(C0 + i * ct_words(), 2 * hp_.L, 0, hp_.L, 7 + i);
    }
    for (int k = 0; k < sums * terms; ++k) {  // random residues in packed digit form
        fill_residues(MK + k * kw, dnum * 2 * R, 0, R, 1000 + k);
        fill_residues(MK + k * kw + (size_t)dnum * 2 * R * N, hp_.L, 0, hp_.L, 5000 + k);
    }
    {
        const size_t words = (size_t)sums * terms * kw;
        const dim3 kg((unsigned)((words + 4 * kThreads - 1) / (4 * kThreads)));
        if (hp_.L == 3) k_mask_digits<ShapeQ3><<<kg, kThreads, 0, stream_>>>(MK, words);
        else k_mask_digits<ShapeQ8><<<kg, kThreads, 0, stream_>>>(MK, words);
        ++launches_;
    }
    std::vector<PlanGroup> groups;
    std::vector<const u64*> mkey, dig, c0;
    std::vector<u32> gs;
    std::vector<u64*> out;
    for (int k0 = 0; k0 < instances; k0 += tile)
        for (int s = 0; s < sums; ++s) {
            PlanGroup G{};
            G.item0 = (u32)out.size();
            G.cnt = (u32)(std::min(instances, k0 + tile) - k0);
            G.term0 = (u32)mkey.size();
            G.nterms = (u32)terms;
            G.dbase = (u32)dig.size();
            for (int t = 0; t < terms; ++t) {
                mkey.push_back(MK + ((size_t)s * terms + t) * kw);
                gs.push_back(galois_of(1 + (s * terms + t) % 2047, N));
            }
            for (u32 u = 0; u < G.cnt; ++u) {
                for (int t = 0; t < terms; ++t) {
                    dig.push_back(D + (size_t)(k0 + u) * dw);
                    c0.push_back(C0 + (size_t)(k0 + u) * ct_words());
                }
                out.push_back(A + ((size_t)(k0 + u) * sums + s) * aw);
            }
            groups.push_back(G);
        }
    rotate_plan(groups, mkey, gs, dig, c0, out);  // warm-up
    cudaEvent_t e0, e1;
    HGM_CUDA(cudaEventCreate(&e0));
    HGM_CUDA(cudaEventCreate(&e1));
    HGM_CUDA(cudaEventRecord(e0, stream_));
    for (int it = 0; it < iters; ++it) rotate_plan(groups, mkey, gs, dig, c0, out);
    HGM_CUDA(cudaEventRecord(e1, stream_));
    HGM_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    HGM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    release(D);
    release(C0);
    release(MK);
    release(A);
    sync();
    return ms / iters;
}

void Context::inner_product(int n, const u64* const* digits, const u64* const* keys, const u32* g,
                            u64* const* acc, const u64* const* c0) {
    std::vector<const u64*> vd(digits, digits + n), vk(keys, keys + n);
    std::vector<u32> vg(g, g + n);
    std::vector<u64*> va(acc, acc + n);
    const u64* const* dc0 = nullptr;
    if (c0) {
        std::vector<const u64*> v(c0, c0 + n);
        dc0 = upload(v);
    }
    if (hp_.L == 3) k_ks_inner<ShapeQ3><<<grid_of(hp_.N, (n + kKeyReuse - 1) / kKeyReuse), kThreads, 0, stream_>>>(cx_, n, upload(vd), upload(vk), upload(vg),
                                                           upload(va), dc0); else k_ks_inner<ShapeQ8><<<grid_of(hp_.N, (n + kKeyReuse - 1) / kKeyReuse), kThreads, 0, stream_>>>(cx_, n, upload(vd), upload(vk), upload(vg),
                                                           upload(va), dc0); ++launches_;
    HGM_CUDA(cudaGetLastError());
}

// ModDown of n accumulators, then out = (acc - conv) P^-1 + add0[g0] (+ add1)
// ModDown of n accumulators (P limbs inverse-transformed first), then
//   out = (acc - NTT(conv)) P^-1 + NTT(ecoef) + addn[galois]   (ecoef/addn optional)
// ecoef: per item [2][L][N] coefficient-domain addend (relinearisation's e0, e1);
// addn: per item NTT-domain c0 limbs added to component 0 (rotation's phi(c0)).
// key_switch_tail leaves acc intact: its P limbs are read by the fused
// conversion (MdConvIO), or inverse-transformed out of place for k_moddown_conv
bool Context::tail_keeps_acc() const {
    if (ntt_fusable(hp_.dev, kFuseModDown)) return false;  // opt-in ModDownIO: P limbs transformed in place
    return ntt_conv_fusable(hp_.dev) || ntt_out_of_place_ok(hp_.dev);
}

void Context::key_switch_tail(int n, u64* const* acc, const u64* const* ecoef, const u64* const* addn,
                              const u32* g, u64* const* out, bool prescaled) {
    if (prescaled && ntt_fusable(hp_.dev, kFuseModDown))
        throw std::logic_error("prescaled accumulators need the split ModDown path");
    const u32 N = hp_.N, L = hp_.L, K = hp_.K, R = hp_.R;
    std::vector<u64*> va(acc, acc + n);
    u64* const* dacc = upload(va);
    std::vector<u32> vg(g, g + n);
    std::vector<u64*> vo(out, out + n);
    const u64* const* dadd = nullptr;
    if (addn) {
        std::vector<const u64*> v(addn, addn + n);
        dadd = upload(v);
    }
    const u64* const* dec = nullptr;
    if (ecoef) {
        std::vector<const u64*> v(ecoef, ecoef + n);
        dec = upload(v);
    }
    const bool conv_fused = ntt_conv_fusable(hp_.dev) && !ntt_fusable(hp_.dev, kFuseModDown);
    // out of place where the transform allows it: acc's P limbs stay in the NTT domain,
    // so a pending key switch survives its own ModDown without a copy (moddown())
    u64* Pc = nullptr;
    if (!conv_fused && tail_keeps_acc()) {
        Pc = alloc((size_t)n * 2 * K * N);
        std::vector<const u64*> src((size_t)n * 2 * K);
        for (int i = 0; i < n; ++i)
            for (u32 c = 0; c < 2; ++c)
                for (u32 k = 0; k < K; ++k) src[((size_t)i * 2 + c) * K + k] = acc[i] + ((size_t)c * R + L + k) * N;
        NttJobs pj = jobs_contig(Pc, n * 2 * K, L, K);
        pj.src = upload(src);
        pj.unscaled = kLazyOut;  // k_moddown_conv: Shoup by phat_inv_n (N^-1 folded in)
        ntt(false, pj);
    } else if (!conv_fused) {  // P limbs back to the coefficient domain (N^-1 left to the conversion)
        NttJobs pj;
        std::vector<u64*> plimbs((size_t)n * 2 * K);
        for (int i = 0; i < n; ++i)
            for (u32 c = 0; c < 2; ++c)
                for (u32 k = 0; k < K; ++k) plimbs[((size_t)i * 2 + c) * K + k] = acc[i] + ((size_t)c * R + L + k) * N;
        pj.ptrs = upload(plimbs);
        pj.count = n * 2 * K;
        pj.period = K;
        for (u32 k = 0; k < K; ++k) pj.prime[k] = (unsigned char)(L + k);
        pj.unscaled = kLazyOut;  // k_moddown_conv / ModDownIO: Shoup by phat_inv_n (N^-1 folded in)
        ntt(false, pj);
    }
    if (ntt_fusable(hp_.dev, kFuseModDown)) {
        ntt_moddown_fused(cx_, hp_.dev, n, dacc, dec, dadd, upload(vg), upload(vo), stream_);
        ++launches_;
        HGM_CUDA(cudaGetLastError());
        return;
    }
    // conversion (V = ecoef - P^-1 conv), NTT of V, finishing pass
    u64* V = alloc((size_t)n * 2 * L * N);
    if (conv_fused) {
        ntt_moddown_conv_fused(cx_, hp_.dev, n, dacc, dec, V, stream_);
        ++launches_;
    } else {
        if (hp_.L == 3) k_moddown_conv<ShapeQ3><<<grid_of(N, n, 2), kThreads, 0, stream_>>>(cx_, n, dacc, dec, V, Pc); else k_moddown_conv<ShapeQ8><<<grid_of(N, n, 2), kThreads, 0, stream_>>>(cx_, n, dacc, dec, V, Pc); ++launches_;
        if (Pc) release(Pc);
    }
    if (ntt_finish_fusable(hp_.dev)) {
        ntt_finish_fused(cx_, hp_.dev, n, V, dacc, dadd, upload(vg), upload(vo), stream_, prescaled);
        ++launches_;
    } else {
        ntt(true, jobs_contig(V, n * 2 * L, 0, L));
        if (hp_.L == 3) k_ks_finish<ShapeQ3><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, dacc, V, dadd, upload(vg), upload(vo), prescaled ? 1u : 0u); else k_ks_finish<ShapeQ8><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, dacc, V, dadd, upload(vg), upload(vo), prescaled ? 1u : 0u); ++launches_;
    }
    release(V);
    HGM_CUDA(cudaGetLastError());
}

void Context::rotate(int n, const u64* const* modup, const u64* const* ct, const u32* g,
                     u64* const* out) {
    if (n <= 0) return;
    const int chunk = chunk_for((size_t)(hp_.dnum * hp_.R + 2 * hp_.R + 2 * hp_.L) * hp_.N, kChunkKs);
    if (n > chunk) {
        for (int c0 = 0; c0 < n; c0 += chunk) {
            const int cn = std::min(chunk, n - c0);
            rotate(cn, modup + c0, ct + c0, g + c0, out + c0);
        }
        return;
    }
    const u32 N = hp_.N, R = hp_.R;
    std::vector<const u64*> keys(n);
    for (int i = 0; i < n; ++i) keys[i] = ks_key(g[i]);
    u64* A = alloc((size_t)n * 2 * R * N);
    std::vector<u64*> accs(n);
    for (int i = 0; i < n; ++i) accs[i] = A + (size_t)i * 2 * R * N;
    inner_product(n, modup, keys.data(), g, accs.data());
    key_switch_tail(n, accs.data(), nullptr, ct, g, out);
    release(A);
}

// Exact B extension of (a.c0, a.c1, b.c0, b.c1), NTT domain over B:
// returns XB [n][4][nB][N] (k_q_to_b's layout; caller releases).
u64* Context::b_extend(int n, const u64* const* a, const u64* const* b) {
    const u32 N = hp_.N, L = hp_.L, K = hp_.K, nB = hp_.nB;
    const size_t LN = (size_t)L * N;
    // 1. to the coefficient domain (out-of-place INTT)
    u64* X = alloc((size_t)n * 4 * LN);
    if (ntt_fusable_size(hp_.dev)) {
        std::vector<const u64*> src((size_t)n * 4 * L);
        for (int i = 0; i < n; ++i)
            for (u32 w = 0; w < 4 * L; ++w)
                src[(size_t)i * 4 * L + w] = (w < 2 * L ? a[i] + (size_t)w * N : b[i] + (size_t)(w - 2 * L) * N);
        NttJobs xj = jobs_contig(X, n * 4 * L, 0, L);
        xj.src = upload(src);
        xj.unscaled = kLazyOut;  // k_q_to_b: Shoup by qhat_inv_n (N^-1 folded in)
        ntt(false, xj);
    } else {
        std::vector<const u64*> src((size_t)2 * n);
        std::vector<u64*> dst((size_t)2 * n);
        for (int i = 0; i < n; ++i) {
            src[2 * i] = a[i];
            src[2 * i + 1] = b[i];
            dst[2 * i] = X + (size_t)i * 4 * LN;
            dst[2 * i + 1] = X + (size_t)i * 4 * LN + 2 * LN;
        }
        k_copy<<<grid_of(N, 2 * n), kThreads, 0, stream_>>>(2 * n, ct_words(), upload(src), upload(dst)); ++launches_;
        NttJobs xj = jobs_contig(X, n * 4 * L, 0, L);
        xj.unscaled = 1;
        ntt(false, xj);
    }
    // 2. exact Q -> B and NTT over B
    u64* XB = alloc((size_t)n * 4 * nB * N);
    if (HGM_QTOB_PAIR && hp_.L == 3) {  // (ShapeQ8's pair kernel spills: parameter set 1 keeps one per thread)
        k_q_to_b2<ShapeQ3><<<grid_of(N / 2, n, 4), kThreads, 0, stream_>>>(cx_, n, X, XB);
    } else {
        if (hp_.L == 3) k_q_to_b<ShapeQ3><<<grid_of(N, n, 4), kThreads, 0, stream_>>>(cx_, n, X, XB); else k_q_to_b<ShapeQ8><<<grid_of(N, n, 4), kThreads, 0, stream_>>>(cx_, n, X, XB);
    }
    ++launches_;
    release(X);
    ntt(true, jobs_contig(XB, n * 4 * nB, L + K, nB));
    return XB;
}

// Scale-and-round of n coefficient-domain tensors T [n][3][L+nB][N] (unscaled
// INTT output, kLazyOut) and relinearisation: out[i] = (e0, e1) + KS(e2).
// Releases T.
void Context::scale_relin(int n, u64* T, u64* const* out) {
    const u32 N = hp_.N, L = hp_.L, R = hp_.R, dnum = hp_.dnum;
    const size_t LN = (size_t)L * N;
    // 4. scale and round back to Q (coefficient form)
    u64* E = alloc((size_t)n * 3 * LN);
    const bool fused = ntt_fusable(hp_.dev, kFuseModUp);
    u64* Dg = alloc((size_t)n * dnum * R * N);
    // alpha = 1: scale-and-round writes e2's ModUp digits itself
    const bool lift_in_sr = hp_.alpha == 1 && !fused;
    if (hp_.L == 3) k_scale_round<ShapeQ3><<<grid_of(N, n, 3), kThreads, 0, stream_>>>(cx_, n, T, E, lift_in_sr ? Dg : nullptr); else k_scale_round<ShapeQ8><<<grid_of(N, n, 3), kThreads, 0, stream_>>>(cx_, n, T, E, nullptr); ++launches_;
    release(T);
    // 5. relinearise e2: ModUp, inner product with rlk, ModDown, add (e0, e1)
    if (lift_in_sr) {
        ntt(true, jobs_contig(Dg, n * dnum * R, 0, R));
    } else if (fused) {
        ntt_modup_fused(cx_, hp_.dev, n, E + 2 * LN, 3 * LN, Dg, stream_);
        ++launches_;
    } else {
        if (hp_.L == 3) k_modup_lift<ShapeQ3><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, E + 2 * LN, 3 * LN, Dg, 0); else k_modup_lift<ShapeQ8><<<grid_of(N, n), kThreads, 0, stream_>>>(cx_, n, E + 2 * LN, 3 * LN, Dg, 0); ++launches_;
        ntt(true, jobs_contig(Dg, n * dnum * R, 0, R));
    }
    u64* A = alloc((size_t)n * 2 * R * N);
    std::vector<const u64*> digits(n), keys(n), ecoef(n);
    std::vector<u64*> accs(n);
    std::vector<u32> ones(n, 1);
    const u64* rlk = ks_key(0);
    for (int i = 0; i < n; ++i) {
        digits[i] = Dg + (size_t)i * dnum * R * N;
        keys[i] = rlk;
        accs[i] = A + (size_t)i * 2 * R * N;
        ecoef[i] = E + (size_t)i * 3 * LN;  // [e0 limbs | e1 limbs]
    }
    inner_product(n, digits.data(), keys.data(), ones.data(), accs.data());
    key_switch_tail(n, accs.data(), ecoef.data(), nullptr, ones.data(), out);
    release(Dg);
    release(A);
    release(E);
}

void Context::rotate_acc(int n, const u64* const* modup, const u64* const* ct, const u32* g, u64* const* acc) {
    if (n <= 0) return;
    for (int c0 = 0; c0 < n; c0 += kChunkKs) {
        const int cn = std::min(kChunkKs, n - c0);
        std::vector<const u64*> keys(cn);
        for (int i = 0; i < cn; ++i) keys[i] = ks_key(g[c0 + i]);
        inner_product(cn, modup + c0, keys.data(), g + c0, acc + c0, ct + c0);
    }
}

size_t Context::masked_key_budget() const {
    static const size_t env = [] {
        const char* e = std::getenv("HGM_MASKED_KEY_MB");
        return e ? (size_t)std::atoll(e) << 20 : (size_t)0;
    }();
    if (env) return env;
    return 2 * mask_budget();  // min(16 GB, an eighth of the device)
}

void Context::drop_masked_keys() {
    std::lock_guard<std::mutex> lk(mask_mu_);
    for (auto& kv : mkeys_) HGM_CUDA(cudaFreeAsync(kv.second.dev, stream_));
    mkeys_.clear();
}

void Context::trim_masked_keys(size_t needed) {
    std::lock_guard<std::mutex> lk(mask_mu_);
    const size_t each = masked_key_words() * 8, budget = masked_key_budget();
    if ((mkeys_.size() + needed) * each <= budget) return;
    // least recently used first, down to half the budget (or room for `needed`)
    std::vector<std::pair<u64, const std::vector<u64>*>> all;
    for (auto& kv : mkeys_) all.push_back({kv.second.tick, &kv.first});
    std::sort(all.begin(), all.end());
    const size_t keep = std::min(budget / 2, budget - std::min(budget, needed * each)) / each;
    std::vector<std::vector<u64>> victims;
    for (size_t i = 0; i < all.size() && mkeys_.size() - victims.size() > keep; ++i) victims.push_back(*all[i].second);
    for (auto& v : victims) {
        auto it = mkeys_.find(v);
        HGM_CUDA(cudaFreeAsync(it->second.dev, stream_));
        mkeys_.erase(it);
    }
}

const u64* Context::masked_key(u32 g, const std::vector<u64>& ids, const std::vector<const u64*>* mask_dev,
                               bool prescaled) {
    std::vector<u64> id(ids);
    std::sort(id.begin(), id.end());
    id.insert(id.begin(), (u64)g | ((u64)(prescaled ? 1 : 0) << 32));
    {
        std::lock_guard<std::mutex> lk(mask_mu_);
        auto it = mkeys_.find(id);
        if (it != mkeys_.end()) {
            it->second.tick = ++mask_tick_;
            return it->second.dev;
        }
        if (!mask_dev || (mkeys_.size() + 1) * masked_key_words() * 8 > masked_key_budget()) return nullptr;
    }
    const u64* key = ks_key(g);
    u64* out = nullptr;
    HGM_CUDA(cudaMallocAsync((void**)&out, masked_key_words() * 8, stream_));
    const u64* const* dm = upload(*mask_dev);
    const u32 words = hp_.R * hp_.N;
    const dim3 grid((words + kThreads - 1) / kThreads);
    if (hp_.L == 3)
        k_mask_key<ShapeQ3><<<grid, kThreads, 0, stream_>>>(cx_, key, dm, (u32)mask_dev->size(), out, prescaled ? 1u : 0u);
    else
        k_mask_key<ShapeQ8><<<grid, kThreads, 0, stream_>>>(cx_, key, dm, (u32)mask_dev->size(), out, prescaled ? 1u : 0u);
    ++launches_;
    HGM_CUDA(cudaGetLastError());
    std::lock_guard<std::mutex> lk(mask_mu_);
    mkeys_.emplace(std::move(id), MaskedKey{out, ++mask_tick_});
    return out;
}

void Context::rotate_plan(const std::vector<PlanGroup>& groups, const std::vector<const u64*>& mkey,
                          const std::vector<u32>& g, const std::vector<const u64*>& digits,
                          const std::vector<const u64*>& c0, const std::vector<u64*>& out) {
    if (groups.empty()) return;
    const u64* const* dk = upload(mkey);
    const u32* dg = upload(g);
    const u64* const* dd = upload(digits);
    const u64* const* dc = upload(c0);
    u64* const* dout = upload(out);
    const PlanGroup* dgrp = upload(groups);
    const u32 n = (u32)groups.size();
    u32 tmax = 1;
    for (const PlanGroup& G : groups) tmax = std::max(tmax, std::min(G.nterms, kPlanTerms));
    const size_t smem = (size_t)tmax * (2 * hp_.dnum + 1) * kThreads * 8;
    static const bool attr = [] {
        const int cap = (int)(kPlanTerms * (2 * 3 + 1) * kThreads * 8);
        HGM_CUDA(cudaFuncSetAttribute(k_ks_plan<ShapeQ3>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap));
        HGM_CUDA(cudaFuncSetAttribute(k_ks_plan<ShapeQ8>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap));
        return true;
    }();
    (void)attr;
    if (hp_.L == 3)
        k_ks_plan<ShapeQ3><<<grid_of(hp_.N, n), kThreads, smem, stream_>>>(cx_, n, dgrp, dk, dg, dd, dc, dout);
    else
        k_ks_plan<ShapeQ8><<<grid_of(hp_.N, n), kThreads, smem, stream_>>>(cx_, n, dgrp, dk, dg, dd, dc, dout);
    ++launches_;
    HGM_CUDA(cudaGetLastError());
}

bool Context::can_prescale() const {
    static const bool on = [] {
        const char* e = std::getenv("HGM_PRESCALE");
        return !(e && e[0] == '0');
    }();
    return on && !ntt_fusable(hp_.dev, kFuseModDown);
}

void Context::moddown(int n, const u64* const* acc, u64* const* out, bool prescaled) {
    if (n <= 0) return;
    const int chunk = chunk_for((size_t)(2 * hp_.R + 2 * hp_.L) * hp_.N, kChunkKs);
    for (int c0 = 0; c0 < n; c0 += chunk) {
        const int cn = std::min(chunk, n - c0);
        std::vector<u32> ones(cn, 1);
        const bool in_place = !tail_keeps_acc();
        if (in_place) {  // this key_switch_tail path inverse-transforms acc's P limbs in place: work on a copy
            u64* A = alloc((size_t)cn * ks_words());
            std::vector<const u64*> src(acc + c0, acc + c0 + cn);
            std::vector<u64*> dst(cn);
            for (int i = 0; i < cn; ++i) dst[i] = A + (size_t)i * ks_words();
            k_copy<<<grid_of(hp_.N, cn), kThreads, 0, stream_>>>(cn, ks_words(), upload(src), upload(dst)); ++launches_;
            key_switch_tail(cn, dst.data(), nullptr, nullptr, ones.data(), out + c0, prescaled);
            release(A);
        } else {
            std::vector<u64*> va(cn);
            for (int i = 0; i < cn; ++i) va[i] = const_cast<u64*>(acc[c0 + i]);
            key_switch_tail(cn, va.data(), nullptr, nullptr, ones.data(), out + c0, prescaled);
        }
    }
}

void Context::lincomb_qp(int n_out, const u32* off, const u64* const* in, const u64* const* mask, u64* const* out) {
    if (n_out <= 0) return;
    for (int c0 = 0; c0 < n_out; c0 += kChunkLin) {
        const int cn = std::min(kChunkLin, n_out - c0);
        std::vector<u32> sub(cn + 1);
        for (int i = 0; i <= cn; ++i) sub[i] = off[c0 + i] - off[c0];
        std::vector<const u64*> vin(in + off[c0], in + off[c0 + cn]), vm(mask + off[c0], mask + off[c0 + cn]);
        std::vector<u64*> vo(out + c0, out + c0 + cn);
        if (all_masked(vm)) {
            if (hp_.L == 3)
                k_lincomb_masked<ShapeQ3, ShapeQ3::R><<<grid_of(hp_.N, cn, 1), kThreads, 0, stream_>>>(cx_, cn, upload(sub), upload(vin), upload(vm), upload(vo));
            else
                k_lincomb_masked<ShapeQ8, ShapeQ8::R><<<grid_of(hp_.N, cn, 1), kThreads, 0, stream_>>>(cx_, cn, upload(sub), upload(vin), upload(vm), upload(vo));
        } else if (hp_.L == 3)
            k_lincomb<ShapeQ3, ShapeQ3::R><<<grid_of(hp_.N, cn, 1), kThreads, 0, stream_>>>(cx_, cn, upload(sub), upload(vin), upload(vm), upload(vo));
        else
            k_lincomb<ShapeQ8, ShapeQ8::R><<<grid_of(hp_.N, cn, 1), kThreads, 0, stream_>>>(cx_, cn, upload(sub), upload(vin), upload(vm), upload(vo));
        ++launches_;
        HGM_CUDA(cudaGetLastError());
    }
}

void Context::mult(int n, const u64* const* a, const u64* const* b, u64* const* out) {
    if (n <= 0) return;
    const u32 Lm = hp_.L, Rm = hp_.R, Dm = hp_.L + hp_.nB;
    const int chunk = chunk_for((size_t)(7 * Lm + 4 * hp_.nB + 3 * Dm + hp_.dnum * Rm + 2 * Rm) * hp_.N, kChunkMult);
    if (n > chunk) {
        for (int c0 = 0; c0 < n; c0 += chunk) {
            const int cn = std::min(chunk, n - c0);
            mult(cn, a + c0, b + c0, out + c0);
        }
        return;
    }
    const u32 N = hp_.N, L = hp_.L, K = hp_.K, nB = hp_.nB;
    u64* XB = b_extend(n, a, b);
    // 3. tensor over Q ++ B, INTT
    const u32 D = L + nB;
    u64* T = alloc((size_t)n * 3 * D * N);
    std::vector<const u64*> va(a, a + n), vb(b, b + n);
    if (ntt_tensor_fusable(hp_.dev)) {  // tensor computed inside its INTT's load
        ntt_tensor_fused(cx_, hp_.dev, n, upload(va), upload(vb), XB, T, stream_);
        ++launches_;
        release(XB);
    } else {
        const bool s1 = ntt_inverse_takes_first_stage(hp_.dev) && tensor_first_stage();
        if (s1) {
            if (hp_.L == 3) k_tensor_s1<ShapeQ3><<<grid_of(N / 2, n, D), kThreads, 0, stream_>>>(cx_, n, upload(va), upload(vb), XB, T); else k_tensor_s1<ShapeQ8><<<grid_of(N / 2, n, D), kThreads, 0, stream_>>>(cx_, n, upload(va), upload(vb), XB, T);
        } else {
            if (hp_.L == 3) k_tensor<ShapeQ3><<<grid_of(N, n, D), kThreads, 0, stream_>>>(cx_, n, upload(va), upload(vb), XB, T); else k_tensor<ShapeQ8><<<grid_of(N, n, D), kThreads, 0, stream_>>>(cx_, n, upload(va), upload(vb), XB, T);
        }
        ++launches_;
        release(XB);
        NttJobs tj = jobs_contig(T, n * 3 * D, 0, D);
        tj.first_done = s1 ? 1 : 0;
        for (u32 k = 0; k < nB; ++k) tj.prime[L + k] = (unsigned char)(L + K + k);
        tj.unscaled = kLazyOut;  // k_scale_round: Shoup by dhat_inv_n; B limbs reduced, times T_n
        ntt(false, tj);
    }
    scale_relin(n, T, out);
}

void Context::tensor_acc(int n_dest, const u32* off, const u64* const* a, const u64* const* b, u64* const* T,
                         const unsigned char* init) {
    if (n_dest <= 0) return;
    const u32 N = hp_.N, L = hp_.L, nB = hp_.nB, D = L + nB;
    const int chunk = chunk_for((size_t)(4 * L + 4 * nB) * N, kChunkMult);
    // segments: (destination, item range) pieces of at most `chunk` items per launch sequence
    std::vector<const u64*> ca, cb;
    std::vector<u32> soff{0};
    std::vector<u64*> sdst;
    std::vector<unsigned char> sinit;
    auto run = [&]() {
        const int n = (int)ca.size();
        if (n > 0) {
            u64* XB = b_extend(n, ca.data(), cb.data());
            const int ns = (int)sdst.size();
            if (hp_.L == 3) k_tensor_acc<ShapeQ3><<<grid_of(N, ns, D), kThreads, 0, stream_>>>(cx_, ns, upload(soff), upload(ca), upload(cb), XB, upload(sdst), upload(sinit)); else k_tensor_acc<ShapeQ8><<<grid_of(N, ns, D), kThreads, 0, stream_>>>(cx_, ns, upload(soff), upload(ca), upload(cb), XB, upload(sdst), upload(sinit));
            ++launches_;
            HGM_CUDA(cudaGetLastError());
            release(XB);
        } else if (!sdst.empty()) {  // destinations without items: zero (or unchanged)
            for (size_t s2 = 0; s2 < sdst.size(); ++s2)
                if (!sinit[s2]) HGM_CUDA(cudaMemsetAsync(sdst[s2], 0, (size_t)3 * D * N * 8, stream_));
        }
        ca.clear(); cb.clear(); sdst.clear(); sinit.clear();
        soff.assign(1, 0);
    };
    for (int d = 0; d < n_dest; ++d) {
        u32 i = off[d];
        bool first = true;
        do {
            if ((int)ca.size() >= chunk) run();
            const u32 take = std::min<u32>(off[d + 1] - i, (u32)(chunk - (int)ca.size()));
            for (u32 t = i; t < i + take; ++t) {
                ca.push_back(a[t]);
                cb.push_back(b[t]);
            }
            sdst.push_back(T[d]);
            sinit.push_back(first ? init[d] : 1);
            soff.push_back((u32)ca.size());
            first = false;
            i += take;
        } while (i < off[d + 1]);
    }
    run();
}

void Context::tsum(int n_out, const u32* off, const u64* const* in, u64* const* out, const unsigned char* init) {
    if (n_out <= 0) return;
    const u32 D = hp_.L + hp_.nB;
    for (int c0 = 0; c0 < n_out; c0 += kChunkLin) {
        const int cn = std::min(kChunkLin, n_out - c0);
        std::vector<u32> sub(cn + 1);
        for (int i = 0; i <= cn; ++i) sub[i] = off[c0 + i] - off[c0];
        std::vector<const u64*> vin(in + off[c0], in + off[c0 + cn]);
        std::vector<u64*> vo(out + c0, out + c0 + cn);
        std::vector<unsigned char> vi(init + c0, init + c0 + cn);
        if (hp_.L == 3) k_tsum<ShapeQ3><<<grid_of(hp_.N, cn, 3 * D), kThreads, 0, stream_>>>(cx_, cn, upload(sub), upload(vin), upload(vo), upload(vi)); else k_tsum<ShapeQ8><<<grid_of(hp_.N, cn, 3 * D), kThreads, 0, stream_>>>(cx_, cn, upload(sub), upload(vin), upload(vo), upload(vi));
        ++launches_;
        HGM_CUDA(cudaGetLastError());
    }
}

void Context::materialize(int n, const u64* const* T, const u64* const* addend, u64* const* out) {
    if (n <= 0) return;
    const u32 N = hp_.N, L = hp_.L, K = hp_.K, R = hp_.R, nB = hp_.nB, D = L + nB;
    const int chunk = chunk_for((size_t)(3 * D + 3 * L + hp_.dnum * R + 2 * R) * N, kChunkMult);
    if (n > chunk) {
        for (int c0 = 0; c0 < n; c0 += chunk) {
            const int cn = std::min(chunk, n - c0);
            materialize(cn, T + c0, addend ? addend + c0 : nullptr, out + c0);
        }
        return;
    }
    // tensor to the coefficient domain (out of place: the pending value stays valid)
    u64* Tc = alloc((size_t)n * 3 * D * N);
    NttJobs tj = jobs_contig(Tc, n * 3 * D, 0, D);
    for (u32 k = 0; k < nB; ++k) tj.prime[L + k] = (unsigned char)(L + K + k);
    tj.unscaled = kLazyOut;  // k_scale_round: Shoup by dhat_inv_n; B limbs reduced, times T_n
    if (ntt_fusable_size(hp_.dev)) {
        std::vector<const u64*> src((size_t)n * 3 * D);
        for (int i = 0; i < n; ++i)
            for (u32 w = 0; w < 3 * D; ++w) src[(size_t)i * 3 * D + w] = T[i] + (size_t)w * N;
        tj.src = upload(src);
    } else {
        std::vector<const u64*> src(T, T + n);
        std::vector<u64*> dst(n);
        for (int i = 0; i < n; ++i) dst[i] = Tc + (size_t)i * 3 * D * N;
        k_copy<<<grid_of(N, n), kThreads, 0, stream_>>>(n, (size_t)3 * D * N, upload(src), upload(dst)); ++launches_;
    }
    ntt(false, tj);
    scale_relin(n, Tc, out);
    if (addend) add(n, out, addend, out);
    HGM_CUDA(cudaGetLastError());
}

}  // namespace hgm
