// ntt.cu -- see ntt.cuh for the design.
#include "ntt.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <mutex>
#include <utility>
#include <cstdlib>
#include <stdexcept>

// code-generation variant of the register-round butterflies (common.cuh shoup_rem)
#ifndef HGM_SHOUP_FWD
#define HGM_SHOUP_FWD HGM_SHOUP_V
#endif
#ifndef HGM_SHOUP_INV
#define HGM_SHOUP_INV HGM_SHOUP_V
#endif

namespace hgm {

namespace {

__constant__ DevParams c_dp[kParamSets];

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }
// 32-bit shared::cluster addresses (mapa): four quarters cost four registers
__device__ __forceinline__ u32 dsmem_base(const u64* local, u32 rank) {
    u32 r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((u32)__cvta_generic_to_shared(local)), "r"(rank));
    return r;
}
__device__ __forceinline__ void dsmem_st(u32 base, int i, u64 v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(base + 8u * (u32)i), "l"(v) : "memory");
}
__device__ __forceinline__ u64 dsmem_ld(u32 base, int i) {
    u64 v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(base + 8u * (u32)i) : "memory");
    return v;
}

// Runs f once per (call site, device): the dynamic shared-memory opt-in is a
// per-device function attribute.
template <typename F>
void once_per_device(std::once_flag (&flags)[64], F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::call_once(flags[dev & 63], std::forward<F>(f));
}
// pad() of a compile-time offset.  For base = (block << b) + o with b >= 4 and an
// offset k * 2^s whose bits lie above o's (o < 2^s), pad(base + off) =
// pad(base) + padc(off): one runtime pad per group, immediates for the rest.
constexpr int padc(int i) { return i + (i >> 4); }

template <int LB>
constexpr int smem_words() {
    return (1 << LB) + (1 << (LB - 4));
}

// Twiddles: the stages whose twiddles are shared by many threads (forward
// local stages 0..8, inverse local stages with t >= 16) read them from a
// per-CTA shared-memory cache of 511 Shoup pairs; the deep stages (distinct
// twiddles per thread) prefetch the 15 pairs of their group into registers
// before the butterflies, so no global load sits on the critical path.
constexpr int kTwCache = 511;
#ifndef HGM_TWFILL_ROLLED
#define HGM_TWFILL_ROLLED 1
#endif
// residues per thread: NB / kElems threads per CTA
constexpr int kElems = 16;
// 3-CTA/SM variant: 256 threads x 32 residues, 255 cached twiddle pairs
constexpr int kElems3 = 32, kTwCache3 = 255;
// Twiddle tables hold (w, w') Shoup pairs interleaved, one 16-byte load per
// twiddle: per prime [forward pairs: N][inverse pairs: N] (params.cpp).
__device__ __forceinline__ const ulonglong2* pairs(const u64* t) { return reinterpret_cast<const ulonglong2*>(t); }

// Forward value bounds, in units of q, before global stage s (inputs canonical).
// A stage maps inputs < b q to outputs < (b + 4) q (U + V with V < 3q, and
// U - V + 4q); values must stay below 16q <= 2^64 (q < 2^60), so U is reduced
// by 8q only where b > 12: about every other stage instead of every stage.
// b0: the bound of the transform's inputs (1 = canonical; 8 for the block stages of the
// N = 2^15 cluster transform, whose outer stages hand over sums below 7q -- starting
// at 8 moves the reductions to the even stages without adding one).
constexpr int fwd_bound(int s, int b0 = 1) {
    int b = b0;
    for (int i = 0; i < s; ++i) b = (b > 12 ? 8 : b) + 4;
    return b;
}
constexpr bool fwd_reduce(int s, int b0 = 1) { return fwd_bound(s, b0) > 12; }
// N = 2^15 forward cluster transform: HGM_C4_LAZY=1 runs its outer stages lazily (no
// reductions, block stages from the bound 8); exact, measured -1% on the forward
// transform (the phase is bound by its loads and remote stores, and the last stage
// then needs one more reduction), so the canonical form stays the default.  The
// inverse's outer stages are lazy (+7.6%: they sit behind remote loads).
#ifndef HGM_C4_LAZY
#define HGM_C4_LAZY 0
#endif
constexpr int kC4B0 = HGM_C4_LAZY ? 8 : 1;

// Cooley-Tukey stage r (global stage SG + r) of an R-stage register round
// (compile-time bounds so the round unrolls and x[] stays in registers).
// tw(r, c) yields (w, w') for the c-th twiddle of stage r within this group.
template <int R, int r, int SG, int B0, typename Tw>
__device__ __forceinline__ void fwd_stage(u64 (&x)[1 << R], u64 q, u64 q4, u64 q8, const Tw& tw) {
    constexpr int h = 1 << (R - 1 - r);
    constexpr bool kReduce = fwd_reduce(SG + r, B0);
#pragma unroll
    for (int c = 0; c < (1 << r); ++c) {
        u64 w, ws;
        tw(r, c, w, ws);
#pragma unroll
        for (int u = 0; u < h; ++u) {
            // lazy butterfly: U < 12q, V = w x mod q in [0, 3q) (shoup_lazy3)
            const int k = c * 2 * h + u;
            const u64 U = kReduce ? reduce_once(x[k], q8) : x[k];
            const u64 V = shoup_lazy3<HGM_SHOUP_FWD>(x[k + h], w, ws, q);
            x[k] = U + V;
            x[k + h] = U - V + q4;
        }
    }
    if constexpr (r + 1 < R) fwd_stage<R, r + 1, SG, B0>(x, q, q4, q8, tw);
}

// Gentleman-Sande rounds track a compile-time bound (units of q) per register
// element: a butterfly's sum output is the sum of its input bounds and its
// difference output is shoup_lazy3's 3q.  Values stay below 16q <= 2^64, a
// sum is reduced (one conditional subtraction of a power-of-two multiple of q)
// only above kGsT, and the round ends with every element below kGsIn, the
// bound its inputs were assumed to have -- about 5 reductions per 8 butterflies
// instead of 8.
constexpr int kGsIn = 4, kGsT = 8;
constexpr int p2ceil(int x) {
    int m = 1;
    while (m < x) m *= 2;
    return m;
}
constexpr int red_to(int v) { return p2ceil(v) / 2; }  // reduce_once by m = p2ceil(v)/2: < m
struct GsAct {
    int mU, mV, off, mS;  // pre-reductions of U and V, U - V offset, sum reduction (0: none)
};
template <int R>
struct GsPlan {
    GsAct act[R][1 << R];  // [stage][top index k]
    int fin[1 << R][2];    // round-end reductions of element k
};
template <int R>
constexpr GsPlan<R> make_gs_plan() {
    GsPlan<R> p{};
    int b[1 << R] = {};
    for (int k = 0; k < (1 << R); ++k) b[k] = kGsIn;
    for (int r = 0; r < R; ++r) {
        const int h = 1 << r;
        int nb[1 << R] = {};
        for (int k = 0; k < (1 << R); ++k) nb[k] = b[k];
        for (int k = 0; k < (1 << R); ++k) {
            if (k & h) continue;
            GsAct a{0, 0, 0, 0};
            int U = b[k], V = b[k + h];
            if (U + p2ceil(V) > 16 || U + V > 16) {
                if (U >= V) a.mU = U = red_to(U); else a.mV = V = red_to(V);
            }
            if (U + p2ceil(V) > 16 || U + V > 16) {
                if (!a.mU && U > 1) a.mU = U = red_to(U);
                else if (!a.mV && V > 1) a.mV = V = red_to(V);
            }
            a.off = p2ceil(V);
            int S = U + V;
            if (S > kGsT) a.mS = S = red_to(S);
            nb[k] = S;
            nb[k + h] = 3;
            p.act[r][k] = a;
        }
        for (int k = 0; k < (1 << R); ++k) b[k] = nb[k];
    }
    for (int k = 0; k < (1 << R); ++k) {
        for (int st = 0; st < 2; ++st) {
            p.fin[k][st] = 0;
            if (b[k] > kGsIn) p.fin[k][st] = b[k] = red_to(b[k]);
        }
    }
    return p;
}
template <int R>
constexpr bool gs_plan_ok() {
    constexpr GsPlan<R> p = make_gs_plan<R>();
    int b[1 << R] = {};
    for (int k = 0; k < (1 << R); ++k) b[k] = kGsIn;
    for (int r = 0; r < R; ++r)
        for (int k = 0; k < (1 << R); ++k) {
            if (k & (1 << r)) continue;
            const GsAct a = p.act[r][k];
            int U = b[k], V = b[k + (1 << r)];
            if (a.mU) { if (U > 2 * a.mU) return false; U = a.mU; }
            if (a.mV) { if (V > 2 * a.mV) return false; V = a.mV; }
            if (U + V > 16 || U + a.off > 16 || a.off < V) return false;
            int S = U + V;
            if (a.mS) { if (S > 2 * a.mS) return false; S = a.mS; }
            b[k] = S;
            b[k + (1 << r)] = 3;
        }
    for (int k = 0; k < (1 << R); ++k) {
        int v = b[k];
        for (int st = 0; st < 2; ++st)
            if (p.fin[k][st]) { if (v > 2 * p.fin[k][st]) return false; v = p.fin[k][st]; }
        if (v > kGsIn) return false;
    }
    return true;
}
template <int R>
struct GsPlanOf {
    static_assert(gs_plan_ok<R>(), "Gentleman-Sande bound plan exceeds 16q");
    static constexpr GsPlan<R> v = make_gs_plan<R>();
};
constexpr int ilog2c(int m) { return m <= 1 ? 0 : 1 + ilog2c(m / 2); }
template <int M>
__device__ __forceinline__ u64 red_by(u64 x, u64 q) {
    if constexpr (M == 0) return x;
    else return reduce_once(x, q << ilog2c(M));
}

template <int R, int r, int c, int u, typename Tw>
__device__ __forceinline__ void inv_bf(u64 (&x)[1 << R], u64 q, u64 w, u64 ws) {
    constexpr int h = 1 << r, k = c * 2 * h + u;
    constexpr GsAct a = GsPlanOf<R>::v.act[r][k];
    const u64 U = red_by<a.mU>(x[k], q), V = red_by<a.mV>(x[k + h], q);
    x[k] = red_by<a.mS>(U + V, q);
    x[k + h] = shoup_lazy3<HGM_SHOUP_INV>(U - V + (q << ilog2c(a.off)), w, ws, q);
    if constexpr (u + 1 < h) inv_bf<R, r, c, u + 1, Tw>(x, q, w, ws);
}
template <int R, int r, int c, typename Tw>
__device__ __forceinline__ void inv_group(u64 (&x)[1 << R], u64 q, const Tw& tw) {
    u64 w, ws;
    tw(r, c, w, ws);
    inv_bf<R, r, c, 0, Tw>(x, q, w, ws);
    if constexpr (c + 1 < (1 << (R - 1 - r))) inv_group<R, r, c + 1>(x, q, tw);
}
template <int R, int k>
__device__ __forceinline__ void inv_finish(u64 (&x)[1 << R], u64 q) {
    x[k] = red_by<GsPlanOf<R>::v.fin[k][1]>(red_by<GsPlanOf<R>::v.fin[k][0]>(x[k], q), q);
    if constexpr (k + 1 < (1 << R)) inv_finish<R, k + 1>(x, q);
}
// Gentleman-Sande stage r (half-size 2^(LT_LO + r)) of an R-stage round;
// inputs and round outputs in [0, kGsIn q).
template <int R, int r, typename Tw>
__device__ __forceinline__ void inv_stage(u64 (&x)[1 << R], u64 q, u64 /*q4*/, const Tw& tw) {
    inv_group<R, r, 0>(x, q, tw);
    if constexpr (r + 1 < R)
        inv_stage<R, r + 1>(x, q, 0, tw);
    else
        inv_finish<R, 0>(x, q);
}

// Forward local stages [S0, S0+R): stage s = S0 + r, twiddle
//   2^(pre+s) + (blk << s) + (block << r) + c   (global table index)
//   (1 << s) - 1 + (block << r) + c             (CTA cache index, s < 9)
struct NoLoad {
    __device__ u64 operator()(int) const { return 0; }
};

template <int LB, int S0, int R, bool kCached, bool kFromGlobal = false, typename Ld = NoLoad, int E = kElems,
          int B0 = 1>
__device__ __forceinline__ void fwd_round(u64* sm, const u64* __restrict__ tw_cache,
                                          const ulonglong2* __restrict__ tw_tab,
                                          u64 q, int pre, int blk, const Ld& ld = Ld(),
                                          const u64* x0 = nullptr) {
    constexpr int NB = 1 << LB, T = NB / E, G = (NB >> R) / T;
    constexpr int LT_FIRST = LB - 1 - S0, LT_MIN = LT_FIRST - (R - 1);
    const u64 q4 = q << 2, q8 = q << 3;  // lazy bounds (fwd_stage)
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
        const int gi = threadIdx.x + gg * T;
        const int o = gi & ((1 << LT_MIN) - 1);
        const int block = gi >> LT_MIN;
        const int base = (block << (LT_FIRST + 1)) + o;
        constexpr bool kFold = !kFromGlobal;  // measured: folding in the global-load round costs registers
        const int pb = pad(base);
        auto at = [&](int k) { return kFold ? pb + padc(k << LT_MIN) : pad(base + (k << LT_MIN)); };
        u64 x[1 << R];
        if constexpr (kCached) {
            if constexpr (kFromGlobal) {
#pragma unroll
                for (int k = 0; k < (1 << R); ++k) x[k] = (x0 && gg == 0) ? x0[k] : ld(base + (k << LT_MIN));
            } else {
#pragma unroll
                for (int k = 0; k < (1 << R); ++k) x[k] = sm[at(k)];
            }
            auto tw = [&](int r, int c, u64& w, u64& ws) {
                const int i = (1 << (S0 + r)) - 1 + (block << r) + c;
                w = tw_cache[2 * i];
                ws = tw_cache[2 * i + 1];
            };
            fwd_stage<R, 0, S0, B0>(x, q, q4, q8, tw);
        } else {
            u64 pw[(1 << R) - 1], pws[(1 << R) - 1];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < (1 << r); ++c) {
                    const int g = (1 << (pre + S0 + r)) + (blk << (S0 + r)) + (block << r) + c;
                    const ulonglong2 t = __ldg(tw_tab + g);
                    pw[(1 << r) - 1 + c] = t.x;
                    pws[(1 << r) - 1 + c] = t.y;
                }
#pragma unroll
            for (int k = 0; k < (1 << R); ++k) x[k] = sm[at(k)];
            auto tw = [&](int r, int c, u64& w, u64& ws) {
                w = pw[(1 << r) - 1 + c];
                ws = pws[(1 << r) - 1 + c];
            };
            fwd_stage<R, 0, S0, B0>(x, q, q4, q8, tw);
        }
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) sm[at(k)] = x[k];
    }
}

// Inverse local stages with half-sizes 2^(LT_LO + r), r < R; twiddle
//   2^(logN-lt-1) + (blk << (LB-lt-1)) + (block << (R-r-1)) + c,  lt = LT_LO + r
//   cache index (1 << (LB-lt-1)) - 1 + (block << (R-r-1)) + c     (LB-lt-1 < 9)
template <int LB, int LT_LO, int R, bool kCached, int E = kElems>
__device__ __forceinline__ void inv_round(u64* sm, const u64* __restrict__ tw_cache,
                                          const ulonglong2* __restrict__ tw_tab,
                                          u64 q, int logN, int blk) {
    constexpr int NB = 1 << LB, T = NB / E, G = (NB >> R) / T;
    const u64 q4 = q << 2;  // lazy bound 4q (inv_stage)
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
        const int gi = threadIdx.x + gg * T;
        const int o = gi & ((1 << LT_LO) - 1);
        const int block = gi >> LT_LO;
        const int base = (block << (LT_LO + R)) + o;
        const int pb = pad(base);
        u64 x[1 << R];
        if constexpr (kCached) {
#pragma unroll
            for (int k = 0; k < (1 << R); ++k) x[k] = sm[pb + padc(k << LT_LO)];
            auto tw = [&](int r, int c, u64& w, u64& ws) {
                const int i = (1 << (LB - LT_LO - r - 1)) - 1 + (block << (R - r - 1)) + c;
                w = tw_cache[2 * i];
                ws = tw_cache[2 * i + 1];
            };
            inv_stage<R, 0>(x, q, q4, tw);
        } else {
            u64 pw[(1 << R) - 1], pws[(1 << R) - 1];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < (1 << (R - 1 - r)); ++c) {
                    const int lt = LT_LO + r;
                    const int g = (1 << (logN - lt - 1)) + (blk << (LB - lt - 1)) + (block << (R - r - 1)) + c;
                    const int slot = (1 << R) - (1 << (R - r)) + c;  // stage r occupies 2^(R-1-r) slots
                    const ulonglong2 t = __ldg(tw_tab + g);
                    pw[slot] = t.x;
                    pws[slot] = t.y;
                }
#pragma unroll
            for (int k = 0; k < (1 << R); ++k) x[k] = sm[pb + padc(k << LT_LO)];
            auto tw = [&](int r, int c, u64& w, u64& ws) {
                const int slot = (1 << R) - (1 << (R - r)) + c;
                w = pw[slot];
                ws = pws[slot];
            };
            inv_stage<R, 0>(x, q, q4, tw);
        }
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) sm[pb + padc(k << LT_LO)] = x[k];
    }
}

// Fill the CTA twiddle cache: entry (1 << s) - 1 + c, c < 2^s, s < 9, holds the
// global index base(s) + c with base(s) = 2^(outer+s) + (blk << s) (forward:
// outer = pre; inverse: base(s) = 2^(logN-LB+s) + (blk << s) for the stage
// with m-offset 2^s inside the block).
__device__ __forceinline__ void fill_tw_cache(u64* cache, const ulonglong2* __restrict__ tw_tab, int outer, int blk,
                                              int count = kTwCache) {
    // (not unrolled: an unrolled strided loop derives its trip count by an integer
    // division in every thread, for what is a single pass at count <= blockDim)
#if HGM_TWFILL_ROLLED
#pragma unroll 1
#endif
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        const int s = 31 - __clz(i + 1);  // i + 1 in [2^s, 2^(s+1))
        const int c = i + 1 - (1 << s);
        const int g = (1 << (outer + s)) + (blk << s) + c;
        const ulonglong2 t = __ldg(tw_tab + g);
        cache[2 * i] = t.x;
        cache[2 * i + 1] = t.y;
    }
}

// The same fill through cp.async (16-byte copies that bypass the registers): the
// issuing thread does not wait for the twiddles, so the block's own loads go
// out behind them.  Visible to the CTA after cp_async_wait_all + barrier.
__device__ __forceinline__ void fill_tw_cache_async(u64* cache, const ulonglong2* __restrict__ tw_tab, int outer,
                                                    int blk, int count) {
#if HGM_TWFILL_ROLLED
#pragma unroll 1
#endif
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        const int s = 31 - __clz(i + 1);
        const int c = i + 1 - (1 << s);
        const int g = (1 << (outer + s)) + (blk << s) + c;
        const unsigned d = (unsigned)__cvta_generic_to_shared(cache + 2 * i);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(tw_tab + g));
    }
    asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

struct JobView {
    u64* ptr;
    int prime;
};

__device__ __forceinline__ JobView job_of(const NttJobs& jobs, u32 j, u32 N) {
    JobView v;
    v.ptr = jobs.ptrs ? jobs.ptrs[j] : jobs.base + (size_t)j * N;
    // select chain over the packed pattern (no dynamic indexing of the
    // by-value parameter, which would spill it to local memory)
    const u32 idx = j % jobs.period;
    const u32 word = idx >> 3;
    u64 pw = jobs.packed[0];
    pw = word == 1 ? jobs.packed[1] : pw;
    pw = word == 2 ? jobs.packed[2] : pw;
    pw = word == 3 ? jobs.packed[3] : pw;
    v.prime = (int)((pw >> (8 * (idx & 7))) & 0xff);
    return v;
}

// io kernels: 2 (default) prefetches the transform input only, 1 also the store
// epilogue's streams (measured -1%: 85 MB of prefetches in flight thrash L2), 0 none
__constant__ int pf_mode = 2;
// cp.async.bulk L2 prefetch of [p, p + bytes), 16 KB per thread of the calling warp
__device__ __forceinline__ void pf_l2(const void* p, u32 bytes) {
    for (u32 o = (threadIdx.x & 31) * 16384u; o < bytes; o += 32 * 16384u) {
        const u32 n = bytes - o < 16384u ? bytes - o : 16384u;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const char*)p + o), "r"(n) : "memory");
    }
}

// One wave ahead: the CTA of job x asks the copy engine (cp.async.bulk
// prefetch, no registers or issue slots) to stage job x + ahead's block in L2,
// so that the CTA taking this slot next finds its loads there instead of in HBM.
template <int LB>
__device__ __forceinline__ void l2_prefetch_ahead(const NttJobs& jobs, u32 N) {
    constexpr u32 kParts = 4, kBytes = (8u << LB) / kParts;
    if (threadIdx.x < kParts && jobs.ahead) {
        const u32 nx = blockIdx.x + jobs.ahead;
        if (nx < jobs.count) {
            const u64* p = jobs.src ? jobs.src[nx] : job_of(jobs, nx, N).ptr;
            p += ((size_t)blockIdx.y << LB) + (size_t)threadIdx.x * (kBytes / 8);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(kBytes) : "memory");
        }
    }
}

// Forward: the last Cooley-Tukey stage (t = 1, m = N/2) pairs adjacent
// residues, i.e. exactly the 16-byte vector each thread stores, so it is
// fused into the coalesced store together with the reduction to [0, q).
template <int LB, int E = kElems>
__device__ __forceinline__ void store_last_stage(const u64* sm, u64* g, const ulonglong2* __restrict__ tw_tab, u64 q, int logN, int blk) {
    constexpr int NB = 1 << LB, T = NB / E;
    ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
    const int tw0 = (1 << (logN - 1)) + (blk << (LB - 1));
#ifndef HGM_LAST_UNROLL
#define HGM_LAST_UNROLL 8
#endif
    constexpr int kLastUnroll = HGM_LAST_UNROLL;
#pragma unroll kLastUnroll
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        const ulonglong2 t = __ldg(tw_tab + tw0 + i);
        const u64 w = t.x, ws = t.y;
        const u64 q2 = q << 1, q4 = q << 2;
        const u64 U = reduce_once(reduce_once(reduce_once(sm[pad(2 * i)], q4 << 1), q4), q2);  // [0, 16q) -> [0, 2q)
        const u64 V = shoup_lazy(sm[pad(2 * i + 1)], w, ws, q);
        ulonglong2 v;
        v.x = reduce_once(reduce_once(U + V, q2), q);
        v.y = reduce_once(reduce_once(U - V + q2, q2), q);
        g2[i] = v;
    }
}

// x < 16q -> [0, q) in one table step and one conditional subtraction: every
// prime lies so close below 2^s (16 (2^s - q) < q, checked in params.cpp) that
// x - floor(x / 2^s) q falls in [0, 2q).  tab[i] = i q, 16 entries in shared
// memory (no multiply: the transforms are bound by the integer multiply pipe).
// HGM_LAST_TAB: 1 table (default), 2 the product by IMAD instead, 0 the chain of
// conditional subtractions (previous form).
#ifndef HGM_LAST_TAB
#define HGM_LAST_TAB 1
#endif
struct Canon {
    const u64* tab;
    u32 sh32;  // s - 32
    u64 q;
    __device__ __forceinline__ u64 operator()(u64 x) const {
        const u32 k = (u32)(x >> 32) >> sh32;
#if HGM_LAST_TAB == 2
        return reduce_once(x - mul_lo_q((u64)k, q), q);
#else
        return reduce_once(x - tab[k], q);
#endif
    }
};
__device__ __forceinline__ Canon make_canon(u64* tab, const Prime& P) {
    if (threadIdx.x < 16) tab[threadIdx.x] = (u64)threadIdx.x * P.q;  // visible after the next barrier
    return Canon{tab, P.s - 32, P.q};
}

// Last stage with the table reduction: U < kU q (reduced by 8q once where the
// round bounds allow more), V = w x in [0, 3q), outputs U + V and U - V + 3q
// below (kU + 3) q canonicalised by `cn`.
template <int LB, int E = kElems, int B0 = 1>
__device__ __forceinline__ void store_last_stage_tab(const u64* sm, u64* g, const ulonglong2* __restrict__ tw_tab, u64 q,
                                                     int logN, int blk, const Canon& cn) {
    constexpr int NB = 1 << LB, T = NB / E;
    constexpr bool kRedU = fwd_bound(LB - 1, B0) > 12;  // U + V must stay below 16q
    ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
    const int tw0 = (1 << (logN - 1)) + (blk << (LB - 1));
    const u64 q3 = q + (q << 1), q8 = q << 3;
#pragma unroll 8
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        const ulonglong2 t = __ldg(tw_tab + tw0 + i);
        const u64 u = sm[pad(2 * i)];
        const u64 U = kRedU ? reduce_once(u, q8) : u;
        const u64 V = shoup_lazy3(sm[pad(2 * i + 1)], t.x, t.y, q);
        ulonglong2 v;
        v.x = cn(U + V);
        v.y = cn(U - V + q3);
        g2[i] = v;
    }
}
// The same handing (U + V, U - V + 3q), both below 11q, to `st`: the consumer may
// add up to 4q more before canonicalising with the same table.
template <int LB, typename St, int E = kElems, int B0 = 1>
__device__ __forceinline__ void store_last_stage_io_tab(const u64* sm, const St& st, const ulonglong2* __restrict__ tw_tab,
                                                        u64 q, int logN, int blk) {
    constexpr int NB = 1 << LB, T = NB / E;
    constexpr bool kRedU = fwd_bound(LB - 1, B0) > 8;
    const int tw0 = (1 << (logN - 1)) + (blk << (LB - 1));
    const u64 q3 = q + (q << 1), q8 = q << 3;
#pragma unroll 4
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        const ulonglong2 t = __ldg(tw_tab + tw0 + i);
        const u64 u = sm[pad(2 * i)];
        const u64 U = kRedU ? reduce_once(u, q8) : u;
        const u64 V = shoup_lazy3(sm[pad(2 * i + 1)], t.x, t.y, q);
        st(i, U + V, U - V + q3);
    }
}

// Same, handing each finished pair (elements 2i, 2i+1, in [0, 4q)) to `st`.
template <int LB, typename St, int E = kElems>
__device__ __forceinline__ void store_last_stage_io(const u64* sm, const St& st, const ulonglong2* __restrict__ tw_tab, u64 q, int logN, int blk) {
    constexpr int NB = 1 << LB, T = NB / E;
    const int tw0 = (1 << (logN - 1)) + (blk << (LB - 1));
    const u64 q2 = q << 1, q4 = q << 2;
#pragma unroll 4
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        const ulonglong2 t = __ldg(tw_tab + tw0 + i);
        const u64 w = t.x, ws = t.y;
        const u64 U = reduce_once(reduce_once(reduce_once(sm[pad(2 * i)], q4 << 1), q4), q2);  // [0, 16q) -> [0, 2q)
        const u64 V = shoup_lazy(sm[pad(2 * i + 1)], w, ws, q);
        st(i, U + V, U - V + q2);  // lazy, in [0, 4q): the consumer reduces
    }
}

template <int LB, int E, typename Ld2, int kLoadBatch = 8>
__device__ __forceinline__ void load_first_stage_fn(u64* sm, const Ld2& ld2, const ulonglong2* __restrict__ tw_tab,
                                                    u64 q, int logN, int blk) {
    constexpr int NB = 1 << LB, T = NB / E;
    const int tw0 = (1 << (logN - 1)) + (blk << (LB - 1));
    // batches of kB pairs: all loads of a batch in flight before any use
    constexpr int kIt = NB / 2 / T, kB = kIt < kLoadBatch ? kIt : kLoadBatch;
#pragma unroll 1
    for (int i0 = 0; i0 < kIt; i0 += kB) {
        ulonglong2 v[kB];
        u64 w[kB], ws[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            const int i = threadIdx.x + (i0 + b) * T;
            v[b] = ld2(i);
            const ulonglong2 t = __ldg(tw_tab + tw0 + i);
            w[b] = t.x;
            ws[b] = t.y;
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            const int p = pad(2 * (int)threadIdx.x) + padc(2 * (i0 + b) * T);
            sm[p] = reduce_once(v[b].x + v[b].y, q << 1);
            sm[p + 1] = shoup_lazy3(v[b].x - v[b].y + (q << 1), w[b], ws[b], q);
        }
    }
}

// Inverse: the first Gentleman-Sande stage (t = 1) fused into the coalesced load
// (inputs canonical, or below 2q).
template <int LB, int E = kElems, int kLoadBatch = 8>
__device__ __forceinline__ void load_first_stage(u64* sm, const u64* g, const ulonglong2* __restrict__ tw_tab, u64 q,
                                                 int logN, int blk) {
    const ulonglong2* g2 = reinterpret_cast<const ulonglong2*>(g);
    auto ld = [g2](int i) { return __ldcs(g2 + i); };
    load_first_stage_fn<LB, E, decltype(ld), kLoadBatch>(sm, ld, tw_tab, q, logN, blk);
}

template <int LB, int E = kElems>
__device__ __forceinline__ void load_block(u64* sm, const u64* g) {
    constexpr int NB = 1 << LB, T = NB / E;
    const ulonglong2* g2 = reinterpret_cast<const ulonglong2*>(g);
    const int p0 = pad(2 * (int)threadIdx.x);
#pragma unroll 4
    for (int j = 0; j < NB / 2 / T; ++j) {
        const ulonglong2 v = g2[threadIdx.x + j * T];
        sm[p0 + padc(2 * j * T)] = v.x;
        sm[p0 + padc(2 * j * T) + 1] = v.y;
    }
}

// stores the smem values as they are (in [0, 4q): NttJobs::kLazyOut)
template <int LB, int E = kElems>
__device__ __forceinline__ void store_block_raw(const u64* sm, u64* g) {
    constexpr int NB = 1 << LB, T = NB / E;
    ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
    const int p0 = pad(2 * (int)threadIdx.x);
#pragma unroll 4
    for (int j = 0; j < NB / 2 / T; ++j) {
        const int p = p0 + padc(2 * j * T);
        ulonglong2 v;
        v.x = sm[p];
        v.y = sm[p + 1];
        __stcs(g2 + threadIdx.x + j * T, v);
    }
}

// stores canonical residues from smem values in [0, 4q), optionally scaled
template <int LB, bool kScale, int E = kElems>
__device__ __forceinline__ void store_block(const u64* sm, u64* g, u64 q, u64 s, u64 ssh) {
    constexpr int NB = 1 << LB, T = NB / E;
    ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
    const int p0 = pad(2 * (int)threadIdx.x);
#pragma unroll 4
    for (int j = 0; j < NB / 2 / T; ++j) {
        const int p = p0 + padc(2 * j * T);
        ulonglong2 v;
        if constexpr (kScale) {
            v.x = shoup_mul(sm[p], s, ssh, q);
            v.y = shoup_mul(sm[p + 1], s, ssh, q);
        } else {
            v.x = reduce_once(reduce_once(sm[p], q << 1), q);
            v.y = reduce_once(reduce_once(sm[p + 1], q << 1), q);
        }
        g2[threadIdx.x + j * T] = v;
    }
}

// ---------------------------------------------------------------- persistent kernels
// One CTA per SM loops over (limb, block) work items; the next item's residues
// stream into the second shared-memory buffer with cp.async (8-byte granules,
// the padded layout) while the current one is transformed, so HBM latency is
// hidden behind the butterflies even at one CTA per SM.
__device__ __forceinline__ void cp_async8(u64* smem_dst, const u64* gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

template <int LB, int E = kElems>
__device__ __forceinline__ void prefetch_block(u64* buf, const u64* g) {
    constexpr int NB = 1 << LB, T = NB / E;
#pragma unroll 4
    for (int i = threadIdx.x; i < NB; i += T) cp_async8(buf + pad(i), g + i);
}

struct WorkItem {
    u64* g;        // destination block
    const u64* s;  // source block (== g unless out of place)
    int prime, blk;
};
__device__ __forceinline__ WorkItem work_item(const NttJobs& jobs, u32 v, int sub, u32 N, int LB) {
    const JobView jv = job_of(jobs, v / sub, N);
    WorkItem w;
    w.blk = (int)(v % sub);
    w.prime = jv.prime;
    w.g = jv.ptr + ((size_t)w.blk << LB);
    w.s = jobs.src ? jobs.src[v / sub] + ((size_t)w.blk << LB) : w.g;
    return w;
}

// Forward block transform: rounds of 4 register stages (local stages 0..LB-2,
// the first eight with CTA-cached twiddles), the last stage fused into the store.
template <int LB>
__global__ void __launch_bounds__((1 << LB) / kElems, 1)
    k_ntt_fwd(DevCtx cx, NttJobs jobs, int sub) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    extern __shared__ u64 sm[];
    u64* buf0 = sm;
    u64* buf1 = sm + smem_words<LB>();
    u64* cache = sm + 2 * smem_words<LB>();
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const int pre = logN - LB;
    const u32 total = jobs.count * (u32)sub;
    u32 v = blockIdx.x;
    if (v >= total) return;
    WorkItem cur = work_item(jobs, v, sub, N, LB);
    prefetch_block<LB>(buf0, cur.s);
    cp_async_commit();
    int cached_prime = -1, cached_blk = -1;
    for (int slot = 0; v < total; v += gridDim.x, slot ^= 1) {
        u64* b = slot ? buf1 : buf0;
        const u32 vn = v + gridDim.x;
        WorkItem nxt{nullptr, nullptr, 0, 0};
        if (vn < total) {
            nxt = work_item(jobs, vn, sub, N, LB);
            prefetch_block<LB>(slot ? buf0 : buf1, nxt.s);
        }
        cp_async_commit();
        const u64 q = dp->pr[cur.prime].q;
        const u64* w = cx.tw + (size_t)cur.prime * 4 * N;
        if (cur.prime != cached_prime || cur.blk != cached_blk) {
            fill_tw_cache(cache, pairs(w), pre, cur.blk);
            cached_prime = cur.prime;
            cached_blk = cur.blk;
        }
        cp_async_wait1();
        __syncthreads();
        fwd_round<LB, 0, 4, true>(b, cache, pairs(w), q, pre, cur.blk);
        __syncthreads();
        fwd_round<LB, 4, 4, true>(b, cache, pairs(w), q, pre, cur.blk);
        __syncthreads();
        fwd_round<LB, 8, LB - 9, false>(b, cache, pairs(w), q, pre, cur.blk);
        __syncthreads();
        store_last_stage<LB>(b, cur.g, pairs(w), q, logN, cur.blk);
        __syncthreads();
        cur = nxt;
    }
}

// Forward transform of a limb whose input is COMPUTED by io.load(job, j) and
// whose canonical NTT-domain output is CONSUMED by io.store(job, i, v0, v1)
// (elements 2i, 2i+1): base-conversion passes fused around the NTT.
template <int LB, typename IO>
__global__ void __launch_bounds__((1 << LB) / kElems3, 3) k_ntt_fwd_io(DevCtx cx, IO io, u32 ahead) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    extern __shared__ u64 sm[];
    u64* cache = sm + smem_words<LB>();
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const u32 job = blockIdx.x;
    if (ahead && threadIdx.x < 32 && job + ahead < gridDim.x) io.prefetch(job + ahead);
    const int prime = io.prime(job);
    const u64 q = dp->pr[prime].q;
    const u64* w = cx.tw + (size_t)prime * 4 * N;
#if HGM_LAST_TAB
    __shared__ u64 qtab[16];
    const Canon cn = make_canon(qtab, dp->pr[prime]);
#endif
    fill_tw_cache(cache, pairs(w), 0, 0, kTwCache3);
    __syncthreads();
    auto ld = [&](int j) { return io.load(dp, job, (u32)j); };
    fwd_round<LB, 0, 4, true, true, decltype(ld), kElems3>(sm, cache, pairs(w), q, 0, 0, ld);
    __syncthreads();
    fwd_round<LB, 4, 4, true, false, NoLoad, kElems3>(sm, cache, pairs(w), q, 0, 0);
    __syncthreads();
    fwd_round<LB, 8, LB - 9, false, false, NoLoad, kElems3>(sm, cache, pairs(w), q, 0, 0);
    __syncthreads();
#if HGM_LAST_TAB
    auto st = [&](int i, u64 v0, u64 v1) { io.store_lazy(dp, job, (u32)i, v0, v1, cn); };
    store_last_stage_io_tab<LB, decltype(st), kElems3>(sm, st, pairs(w), q, logN, 0);
#else
    auto st = [&](int i, u64 v0, u64 v1) { io.store(dp, job, (u32)i, v0, v1); };
    store_last_stage_io<LB, decltype(st), kElems3>(sm, st, pairs(w), q, logN, 0);
#endif
}

// y < src < 2*dst (one bit length per prime set): centred y mod dst
__device__ __forceinline__ u64 centred_lift_n(u64 y, u64 src, u64 dst) {
    if (y > (src - 1) / 2) {
        u64 m = src - y;
        if (m >= dst) m -= dst;
        return m ? dst - m : 0;
    }
    return y >= dst ? y - dst : y;
}

// ModUp fused into the forward NTT: job = (item, digit dg, target limb r).
struct ModUpIO {
    const u64* C;      // [item] c_stride words: L coefficient-domain limbs
    size_t c_stride;
    u64* D;            // [item][dnum][R][N]
    u32 R, dnum, L, A, N;
    __device__ int prime(u32 job) const { return (int)(job % R); }
    __device__ void prefetch(u32) const {}
    __device__ u64 load(const DevParams* dp, u32 job, u32 j) const {
        const u32 item = job / (dnum * R), dg = (job / R) % dnum, r = job % R;
        const u64* c = C + item * c_stride;
        if (r < L && r / A == dg) return c[(size_t)r * N + j];
        const u64 qr = dp->pr[r].q;
        u64 v = 0;
        for (u32 a = 0; a < A; ++a) {
            const u32 i = dg * A + a;
            const u64 y = shoup_mul(c[(size_t)i * N + j], dp->dg_hat_inv[i], dp->dg_hat_inv_sh[i], dp->pr[i].q);
            v = add_mod(v, shoup_mul(centred_lift_n(y, dp->pr[i].q, qr), dp->dg_hat[i][r], dp->dg_hat_sh[i][r], qr), qr);
        }
        return v;
    }
    __device__ void store(const DevParams* dp, u32 job, u32 i, u64 v0, u64 v1) const {
        const u64 q = dp->pr[job % R].q;
        ulonglong2 v;
        v.x = reduce_once(reduce_once(v0, q << 1), q);
        v.y = reduce_once(reduce_once(v1, q << 1), q);
        reinterpret_cast<ulonglong2*>(D + (size_t)job * N)[i] = v;
    }
    // v0, v1 < 11q (store_last_stage_io_tab)
    __device__ void store_lazy(const DevParams*, u32 job, u32 i, u64 v0, u64 v1, const Canon& cn) const {
        ulonglong2 v;
        v.x = cn(v0);
        v.y = cn(v1);
        reinterpret_cast<ulonglong2*>(D + (size_t)job * N)[i] = v;
    }
};

// ModDown fused into the forward NTT: job = (item, component c, limb i).
//   out_c,i = NTT(addc_c,i - P^-1 conv_c,i) + P^-1 acc_c,i + [c = 0] addn_i[galois_src]
// which equals the oracle's (acc - NTT(conv)) P^-1 (+ NTT(addc)) (+ phi(c0)) by
// linearity of the NTT mod q_i -- exact.
// kPre: acc's Q limbs already hold P^-1 acc (k_ks_plan over masked keys scaled by
// P^-1, Context::masked_key): the store adds them as they are.
template <bool kPre>
struct ModDownIOT {
    u64* const* acc;         // per item [2][R][N]; P limbs already inverse-transformed
    const u64* const* addc;  // per item [2][L][N] coefficient-domain addend, or null
    const u64* const* addn;  // per item [L][N] NTT-domain addend for c = 0, or null
    const u32* g;            // per item Galois element for addn
    u64* const* out;         // per item [2][L][N]
    u32 L, K, R, N, logN;
    __device__ int prime(u32 job) const { return (int)(job % L); }
    // the store's streams: acc's limb i and (c = 0) the addend's limb i
    __device__ void prefetch_store(u32 job) const {
        const u32 item = job / (2 * L), c = (job / L) & 1, i = job % L;
        pf_l2(acc[item] + ((size_t)c * R + i) * N, N * 8);
        if (c == 0 && addn) pf_l2(addn[item] + (size_t)i * N, N * 8);
    }
    __device__ void prefetch(u32 job) const { if (pf_mode == 1) prefetch_store(job); }
    __device__ u64 load(const DevParams* dp, u32 job, u32 j) const {
        const u32 item = job / (2 * L), c = (job / L) & 1, i = job % L;
        const u64* a = acc[item] + (size_t)c * R * N;
        const u64 q = dp->pr[i].q;
        u64 v = 0;
        for (u32 k = 0; k < K; ++k) {
            const u64 p = dp->pr[L + k].q;
            const u64 z = shoup_mul(a[(size_t)(L + k) * N + j], dp->phat_inv_n[k], dp->phat_inv_n_sh[k], p);
            v = add_mod(v, shoup_mul(centred_lift_n(z, p, q), dp->phat_mod_q[k][i], dp->phat_mod_q_sh[k][i], q), q);
        }
        const u64 base = addc ? addc[item][((size_t)c * L + i) * N + j] : 0;
        return sub_mod(base, shoup_mul(v, dp->P_inv_q[i], dp->P_inv_q_sh[i], q), q);
    }
    __device__ void store(const DevParams* dp, u32 job, u32 i2, u64 v0, u64 v1) const {
        const u32 item = job / (2 * L), c = (job / L) & 1, i = job % L;
        const u64 q = dp->pr[i].q, pi = dp->P_inv_q[i], pis = dp->P_inv_q_sh[i];
        const ulonglong2 av = __ldcs(reinterpret_cast<const ulonglong2*>(acc[item] + ((size_t)c * R + i) * N) + i2);
        // lazy sums (v < 4q, Shoup < 3q, addend < q), one reduction chain from [0, 8q)
        u64 r0 = v0 + (kPre ? av.x : shoup_lazy3(av.x, pi, pis, q));
        u64 r1 = v1 + (kPre ? av.y : shoup_lazy3(av.y, pi, pis, q));
        if (c == 0 && addn) {
            const u64* x = addn[item] + (size_t)i * N;
            const u32 ge = g[item];
            r0 += x[ge == 1 ? 2 * i2 : galois_src(2 * i2, ge, logN)];
            r1 += x[ge == 1 ? 2 * i2 + 1 : galois_src(2 * i2 + 1, ge, logN)];
        }
        const u64 q2 = q << 1, q4 = q << 2;
        ulonglong2 v;
        v.x = reduce_once(reduce_once(reduce_once(r0, q4), q2), q);
        v.y = reduce_once(reduce_once(reduce_once(r1, q4), q2), q);
        reinterpret_cast<ulonglong2*>(out[item] + ((size_t)c * L + i) * N)[i2] = v;
    }
    // v0, v1 < 11q (store_last_stage_io_tab): + Shoup < 3q + addend < q stays below 15q,
    // canonicalised by the table step
    __device__ void store_lazy(const DevParams* dp, u32 job, u32 i2, u64 v0, u64 v1, const Canon& cn) const {
        const u32 item = job / (2 * L), c = (job / L) & 1, i = job % L;
        const u64 q = dp->pr[i].q, pi = dp->P_inv_q[i], pis = dp->P_inv_q_sh[i];
        const ulonglong2 av = __ldcs(reinterpret_cast<const ulonglong2*>(acc[item] + ((size_t)c * R + i) * N) + i2);
        u64 r0 = v0 + (kPre ? av.x : shoup_lazy3(av.x, pi, pis, q));
        u64 r1 = v1 + (kPre ? av.y : shoup_lazy3(av.y, pi, pis, q));
        if (c == 0 && addn) {
            const u64* x = addn[item] + (size_t)i * N;
            const u32 ge = g[item];
            r0 += x[ge == 1 ? 2 * i2 : galois_src(2 * i2, ge, logN)];
            r1 += x[ge == 1 ? 2 * i2 + 1 : galois_src(2 * i2 + 1, ge, logN)];
        }
        ulonglong2 v;
        v.x = cn(r0);
        v.y = cn(r1);
        reinterpret_cast<ulonglong2*>(out[item] + ((size_t)c * L + i) * N)[i2] = v;
    }
};

// ModDown's forward NTT with the finishing pass fused into its store: input is
// V = ecoef - P^-1 conv (k_moddown_conv), job = (item, component c, limb i) over
// the contiguous [n][2][L][N] buffer; the store is ModDownIO's.
using ModDownIO = ModDownIOT<false>;
template <bool kPre>
struct FinishIOT : ModDownIOT<kPre> {
    const u64* V;
    __device__ void prefetch(u32 job) const {
        pf_l2(V + (size_t)job * this->N, this->N * 8);
        if (pf_mode == 1) this->prefetch_store(job);
    }
    __device__ u64 load(const DevParams*, u32 job, u32 j) const { return __ldcs(V + (size_t)job * this->N + j); }
};
using FinishIO = FinishIOT<false>;

bool ntt_l2_prefetch();
int sm_count();
// resident CTAs of the 3-CTA/SM kernels: the one-wave-ahead distance
u32 io_ahead() {
    static const bool on = [] {
        const char* v = std::getenv("HGM_NTT_PFIO");
        return !(v && v[0] == '0');
    }();
    static std::once_flag once[64];
    once_per_device(once, [] {
        const char* v = std::getenv("HGM_NTT_PFIO");
        const int m = v ? std::atoi(v) : 2;
        cudaMemcpyToSymbol(pf_mode, &m, sizeof(int));
    });
    return on && ntt_l2_prefetch() ? (u32)(3 * sm_count()) : 0u;
}

// k_ntt_fwd_c4 with its input read through io.load and its output handed to
// io.store (pair index over the whole 2^15 limb): N = 32768's fused epilogues
// (ModDown's finishing pass) in the one-HBM-pass cluster transform.
template <int LB, typename IO>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__((1 << LB) / kElems3, 3)
    k_ntt_fwd_c4_io(DevCtx cx, IO io) {
    namespace cg = cooperative_groups;
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    extern __shared__ u64 sm[];
    u64* cache = sm + smem_words<LB>();
    constexpr int NB = 1 << LB, T = NB / kElems3, COLS = NB / 4;
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const int blk = (int)(blockIdx.x & 3);
    const u32 job = blockIdx.x >> 2;
    const int prime = io.prime(job);
    const u64 q = dp->pr[prime].q;
    const u64* w = cx.tw + (size_t)prime * 4 * N;
#if HGM_LAST_TAB
    __shared__ u64 qtab[16];
    const Canon cn = make_canon(qtab, dp->pr[prime]);
#endif
    fill_tw_cache_async(cache, pairs(w), 2, blk, kTwCache3);
    const ulonglong2* t = pairs(w);
    const u64 w1 = t[1].x, w1s = t[1].y, w2 = t[2].x, w2s = t[2].y, w3 = t[3].x, w3s = t[3].y;
    u32 quarter[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) quarter[r] = dsmem_base(sm, r);
    constexpr int kBatch = 4;
#pragma unroll 1
    for (int c0 = 0; c0 < COLS / T; c0 += kBatch) {
        u64 x[kBatch][4];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int j = blk * COLS + (c0 + b) * T + (int)threadIdx.x;
#pragma unroll
            for (int k = 0; k < 4; ++k) x[b][k] = io.load(dp, job, (u32)(j + k * NB));
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int j = blk * COLS + (c0 + b) * T + (int)threadIdx.x;
            const int p = pad(j);
#if HGM_C4_LAZY
            // lazy: Shoup products in [0, 3q), differences offset by 3q, no reduction --
            // the quarters receive values below 7q and the block stages start from the
            // bound 8 (kC4B0), which costs them no extra reduction
            const u64 q3 = q + (q << 1);
            u64 V = shoup_lazy3(x[b][2], w1, w1s, q);
            const u64 y0 = x[b][0] + V, y2 = x[b][0] - V + q3;  // < 4q
            V = shoup_lazy3(x[b][3], w1, w1s, q);
            const u64 y1 = x[b][1] + V, y3 = x[b][1] - V + q3;  // < 4q
            V = shoup_lazy3(y1, w2, w2s, q);
            dsmem_st(quarter[0], p, y0 + V);                    // < 7q
            dsmem_st(quarter[1], p, y0 - V + q3);
            V = shoup_lazy3(y3, w3, w3s, q);
            dsmem_st(quarter[2], p, y2 + V);
            dsmem_st(quarter[3], p, y2 - V + q3);
#else
            u64 V = shoup_mul(x[b][2], w1, w1s, q);
            const u64 y0 = add_mod(x[b][0], V, q), y2 = sub_mod(x[b][0], V, q);
            V = shoup_mul(x[b][3], w1, w1s, q);
            const u64 y1 = add_mod(x[b][1], V, q), y3 = sub_mod(x[b][1], V, q);
            V = shoup_mul(y1, w2, w2s, q);
            dsmem_st(quarter[0], p, add_mod(y0, V, q));
            dsmem_st(quarter[1], p, sub_mod(y0, V, q));
            V = shoup_mul(y3, w3, w3s, q);
            dsmem_st(quarter[2], p, add_mod(y2, V, q));
            dsmem_st(quarter[3], p, sub_mod(y2, V, q));
#endif
        }
    }
    cp_async_wait_all();
    cg::this_cluster().sync();
    fwd_round<LB, 0, 4, true, false, NoLoad, kElems3, kC4B0>(sm, cache, pairs(w), q, 2, blk);
    __syncthreads();
    fwd_round<LB, 4, 4, true, false, NoLoad, kElems3, kC4B0>(sm, cache, pairs(w), q, 2, blk);
    __syncthreads();
    fwd_round<LB, 8, LB - 9, false, false, NoLoad, kElems3, kC4B0>(sm, cache, pairs(w), q, 2, blk);
    __syncthreads();
    const u32 pair0 = (u32)blk << (LB - 1);
#if HGM_LAST_TAB
    auto st = [&](int i, u64 v0, u64 v1) { io.store_lazy(dp, job, pair0 + (u32)i, v0, v1, cn); };
    store_last_stage_io_tab<LB, decltype(st), kElems3, kC4B0>(sm, st, pairs(w), q, logN, blk);
#else
    auto st = [&](int i, u64 v0, u64 v1) { io.store(dp, job, pair0 + (u32)i, v0, v1); };
    store_last_stage_io<LB, decltype(st), kElems3>(sm, st, pairs(w), q, logN, blk);
#endif
}

template <typename IO>
void launch_fwd_io(const DevCtx& cx, const DevParams& hp, const IO& io, u32 jobs, cudaStream_t s) {
    if (jobs == 0) return;
    if (hp.logN == 15) {
        const size_t smem = (smem_words<13>() + 2 * kTwCache3) * sizeof(u64);
        static std::once_flag once15[64];
        once_per_device(once15, [&] {
            cudaFuncSetAttribute(k_ntt_fwd_c4_io<13, IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        });
        k_ntt_fwd_c4_io<13, IO><<<jobs * 4, (1 << 13) / kElems3, smem, s>>>(cx, io);
        return;
    }
    if (hp.logN == 13) {
        const size_t smem = (smem_words<13>() + 2 * kTwCache3) * sizeof(u64);
        static std::once_flag once13[64];
        once_per_device(once13, [&] {
            cudaFuncSetAttribute(k_ntt_fwd_io<13, IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        });
        k_ntt_fwd_io<13, IO><<<jobs, (1 << 13) / kElems3, smem, s>>>(cx, io, io_ahead());
    } else {
        const size_t smem = (smem_words<12>() + 2 * kTwCache3) * sizeof(u64);
        static std::once_flag once12[64];
        once_per_device(once12, [&] {
            cudaFuncSetAttribute(k_ntt_fwd_io<12, IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        });
        k_ntt_fwd_io<12, IO><<<jobs, (1 << 12) / kElems3, smem, s>>>(cx, io, io_ahead());
    }
}

// Inverse block transform: prefetched block, first stage as an smem pass, then
// rounds of 4 (the last eight local stages with CTA-cached twiddles); N^-1
// folded into the store when the block is the whole limb.
template <int LB>
__global__ void __launch_bounds__((1 << LB) / kElems, 1)
    k_ntt_inv(DevCtx cx, NttJobs jobs, int sub) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    extern __shared__ u64 sm[];
    constexpr int NB = 1 << LB, T = NB / kElems;
    u64* buf0 = sm;
    u64* buf1 = sm + smem_words<LB>();
    u64* cache = sm + 2 * smem_words<LB>();
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const u32 total = jobs.count * (u32)sub;
    u32 v = blockIdx.x;
    if (v >= total) return;
    WorkItem cur = work_item(jobs, v, sub, N, LB);
    prefetch_block<LB>(buf0, cur.s);
    cp_async_commit();
    int cached_prime = -1, cached_blk = -1;
    for (int slot = 0; v < total; v += gridDim.x, slot ^= 1) {
        u64* b = slot ? buf1 : buf0;
        const u32 vn = v + gridDim.x;
        WorkItem nxt{nullptr, nullptr, 0, 0};
        if (vn < total) {
            nxt = work_item(jobs, vn, sub, N, LB);
            prefetch_block<LB>(slot ? buf0 : buf1, nxt.s);
        }
        cp_async_commit();
        const Prime& P = dp->pr[cur.prime];
        const u64 q = P.q;
        const u64* w = cx.tw + (size_t)cur.prime * 4 * N;
        if (cur.prime != cached_prime || cur.blk != cached_blk) {
            fill_tw_cache(cache, pairs(w + 2 * N), logN - LB, cur.blk);
            cached_prime = cur.prime;
            cached_blk = cur.blk;
        }
        cp_async_wait1();
        __syncthreads();
        {  // first Gentleman-Sande stage (t = 1) on adjacent pairs
            const int tw0 = (1 << (logN - 1)) + (cur.blk << (LB - 1));
            const ulonglong2* wt = pairs(w + 2 * N);
#pragma unroll 4
            for (int i = threadIdx.x; i < NB / 2; i += T) {
                const u64 x0 = b[pad(2 * i)], x1 = b[pad(2 * i + 1)];
                const ulonglong2 t = __ldg(wt + tw0 + i);
                const u64 tw = t.x, tws = t.y;
                b[pad(2 * i)] = reduce_once(x0 + x1, q << 1);
                b[pad(2 * i + 1)] = shoup_lazy(x0 - x1 + (q << 1), tw, tws, q);
            }
        }
        __syncthreads();
        inv_round<LB, 1, LB - 9, false>(b, cache, pairs(w + 2 * N), q, logN, cur.blk);
        __syncthreads();
        inv_round<LB, LB - 8, 4, true>(b, cache, pairs(w + 2 * N), q, logN, cur.blk);
        __syncthreads();
        inv_round<LB, LB - 4, 4, true>(b, cache, pairs(w + 2 * N), q, logN, cur.blk);
        __syncthreads();
        if (logN == LB && !jobs.unscaled)
            store_block<LB, true>(b, cur.g, q, P.ninv, P.ninv_sh);
        else
            store_block<LB, false>(b, cur.g, q, 0, 0);
        __syncthreads();
        cur = nxt;
    }
}

// Two outermost forward stages for N = 4 * 2^LB: element j, j+N/4, j+N/2, j+3N/4.
__global__ void k_ntt_fwd_outer2(DevCtx cx, NttJobs jobs) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, Q4 = N / 4;
    const JobView jv = job_of(jobs, blockIdx.y, N);
    const u64 q = dp->pr[jv.prime].q;
    const ulonglong2* t = pairs(cx.tw + (size_t)jv.prime * 4 * N);
    const u64 w1 = t[1].x, w1s = t[1].y, w2 = t[2].x, w2s = t[2].y, w3 = t[3].x, w3s = t[3].y;
    for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < Q4; j += gridDim.x * blockDim.x) {
        u64* a = jv.ptr;
        u64 x0 = a[j], x1 = a[j + Q4], x2 = a[j + 2 * Q4], x3 = a[j + 3 * Q4];
        u64 V = shoup_mul(x2, w1, w1s, q);
        u64 y0 = add_mod(x0, V, q), y2 = sub_mod(x0, V, q);
        V = shoup_mul(x3, w1, w1s, q);
        u64 y1 = add_mod(x1, V, q), y3 = sub_mod(x1, V, q);
        V = shoup_mul(y1, w2, w2s, q);
        a[j] = add_mod(y0, V, q);
        a[j + Q4] = sub_mod(y0, V, q);
        V = shoup_mul(y3, w3, w3s, q);
        a[j + 2 * Q4] = add_mod(y2, V, q);
        a[j + 3 * Q4] = sub_mod(y2, V, q);
    }
}

// Two outermost inverse stages (t = N/4, N/2) plus the N^-1 scaling.
__global__ void k_ntt_inv_outer2(DevCtx cx, NttJobs jobs) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    const u32 N = dp->N, Q4 = N / 4;
    const JobView jv = job_of(jobs, blockIdx.y, N);
    const Prime& P = dp->pr[jv.prime];
    const u64 q = P.q;
    const ulonglong2* t = pairs(cx.tw + (size_t)jv.prime * 4 * N + 2 * N);
    const u64 w2 = t[2].x, w2s = t[2].y, w3 = t[3].x, w3s = t[3].y, w1 = t[1].x, w1s = t[1].y;
    for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < Q4; j += gridDim.x * blockDim.x) {
        u64* a = jv.ptr;
        u64 x0 = a[j], x1 = a[j + Q4], x2 = a[j + 2 * Q4], x3 = a[j + 3 * Q4];
        // t = N/4: pairs (0,1) with m=2 -> w[2], (2,3) with w[3]
        u64 y0 = add_mod(x0, x1, q), y1 = shoup_mul(sub_mod(x0, x1, q), w2, w2s, q);
        u64 y2 = add_mod(x2, x3, q), y3 = shoup_mul(sub_mod(x2, x3, q), w3, w3s, q);
        // t = N/2: pairs (0,2), (1,3) with m=1 -> w[1]
        u64 z0 = add_mod(y0, y2, q), z2 = shoup_mul(sub_mod(y0, y2, q), w1, w1s, q);
        u64 z1 = add_mod(y1, y3, q), z3 = shoup_mul(sub_mod(y1, y3, q), w1, w1s, q);
        if (jobs.unscaled) {
            a[j] = z0;
            a[j + Q4] = z1;
            a[j + 2 * Q4] = z2;
            a[j + 3 * Q4] = z3;
        } else {
            a[j] = shoup_mul(z0, P.ninv, P.ninv_sh, q);
            a[j + Q4] = shoup_mul(z1, P.ninv, P.ninv_sh, q);
            a[j + 2 * Q4] = shoup_mul(z2, P.ninv, P.ninv_sh, q);
            a[j + 3 * Q4] = shoup_mul(z3, P.ninv, P.ninv_sh, q);
        }
    }
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <int LB>
void launch_block(bool fwd, const DevCtx& cx, const NttJobs& jobs, int sub, cudaStream_t s) {
    const size_t smem = (2 * smem_words<LB>() + 2 * kTwCache) * sizeof(u64);
    static std::once_flag once[64];
    once_per_device(once, [&] {
        cudaFuncSetAttribute(k_ntt_fwd<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_ntt_inv<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    const u32 items = jobs.count * (u32)sub;
    const u32 grid = std::min<u32>(items, (u32)sm_count());
    if (fwd)
        k_ntt_fwd<LB><<<grid, (1 << LB) / kElems, smem, s>>>(cx, jobs, sub);
    else
        k_ntt_inv<LB><<<grid, (1 << LB) / kElems, smem, s>>>(cx, jobs, sub);
}


// ---------------------------------------------------------------- 3-CTA variant
// 256 threads x 32 residues, radix-16 rounds over two groups per thread,
// 255 cached twiddle pairs (stages < 8), no double buffer: 72 KB of shared
// memory and <= 85 registers, so three CTAs (24 warps) share an SM.

template <int LB, int E = kElems3, int MINB = 3>
__global__ void __launch_bounds__((1 << LB) / E, MINB) k_ntt_fwd3(DevCtx cx, NttJobs jobs) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    extern __shared__ u64 sm[];
    u64* cache = sm + smem_words<LB>();
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const int pre = logN - LB;
    const int blk = blockIdx.y;
    const JobView jv = job_of(jobs, blockIdx.x, N);
    const u64 q = dp->pr[jv.prime].q;
    const u64* w = cx.tw + (size_t)jv.prime * 4 * N;
    u64* g = jv.ptr + ((size_t)blk << LB);
    const u64* src = jobs.src ? jobs.src[blockIdx.x] + ((size_t)blk << LB) : g;
#if HGM_LAST_TAB
    __shared__ u64 qtab[16];
    const Canon cn = make_canon(qtab, dp->pr[jv.prime]);
#endif
    l2_prefetch_ahead<LB>(jobs, N);
    auto ld = [src](int j) { return __ldcs(src + j); };
    // group 0 of the first round is loaded while the twiddle cache fills
    static_assert((1 << LB) / E <= (1 << (LB - 4)), "first-round group 0 is base = threadIdx.x");
    u64 x0[16];
    fill_tw_cache_async(cache, pairs(w), pre, blk, kTwCache3);
#pragma unroll
    for (int k = 0; k < 16; ++k) x0[k] = ld((int)threadIdx.x + (k << (LB - 4)));
    cp_async_wait_all();
    __syncthreads();
    fwd_round<LB, 0, 4, true, true, decltype(ld), E>(sm, cache, pairs(w), q, pre, blk, ld, x0);
    __syncthreads();
    fwd_round<LB, 4, 4, true, false, NoLoad, E>(sm, cache, pairs(w), q, pre, blk);
    __syncthreads();
    fwd_round<LB, 8, LB - 9, false, false, NoLoad, E>(sm, cache, pairs(w), q, pre, blk);
    __syncthreads();
#if HGM_LAST_TAB
    store_last_stage_tab<LB, E>(sm, g, pairs(w), q, logN, blk, cn);
#else
    store_last_stage<LB, E>(sm, g, pairs(w), q, logN, blk);
#endif
}

template <int LB, int E = kElems3, int MINB = 3>
__global__ void __launch_bounds__((1 << LB) / E, MINB) k_ntt_inv3(DevCtx cx, NttJobs jobs) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    extern __shared__ u64 sm[];
    u64* cache = sm + smem_words<LB>();
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const int blk = blockIdx.y;
    const JobView jv = job_of(jobs, blockIdx.x, N);
    const Prime& P = dp->pr[jv.prime];
    const u64 q = P.q;
    const u64* w = cx.tw + (size_t)jv.prime * 4 * N;
    u64* g = jv.ptr + ((size_t)blk << LB);
    const u64* src = jobs.src ? jobs.src[blockIdx.x] + ((size_t)blk << LB) : g;
    l2_prefetch_ahead<LB>(jobs, N);
    fill_tw_cache_async(cache, pairs(w + 2 * N), logN - LB, blk, kTwCache3);
    if (jobs.first_done)
        load_block<LB, E>(sm, src);
    else
        load_first_stage<LB, E, (MINB < 3 ? 16 : 8)>(sm, src, pairs(w + 2 * N), q, logN, blk);
    cp_async_wait_all();
    __syncthreads();
    inv_round<LB, 1, LB - 9, false, E>(sm, cache, pairs(w + 2 * N), q, logN, blk);
    __syncthreads();
    inv_round<LB, LB - 8, 4, true, E>(sm, cache, pairs(w + 2 * N), q, logN, blk);
    __syncthreads();
    inv_round<LB, LB - 4, 4, true, E>(sm, cache, pairs(w + 2 * N), q, logN, blk);
    __syncthreads();
    if (logN == LB && !jobs.unscaled)
        store_block<LB, true, E>(sm, g, q, P.ninv, P.ninv_sh);
    else if (logN == LB && jobs.unscaled == kLazyOut)
        store_block_raw<LB, E>(sm, g);
    else
        store_block<LB, false, E>(sm, g, q, 0, 0);
}

// Inverse transform of a whole limb read as pairs from io.load2(job, i) (values
// below 2q) whose UNSCALED
// (N * INTT) output, in [0, 4q), is consumed by io.store(job, i, v0, v1)
// (elements 2i, 2i+1): a base conversion fused behind the INTT.
template <int LB, typename IO>
__global__ void __launch_bounds__((1 << LB) / kElems3, 3) k_ntt_inv_io(DevCtx cx, IO io, u32 ahead) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    extern __shared__ u64 sm[];
    u64* cache = sm + smem_words<LB>();
    constexpr int NB = 1 << LB, T = NB / kElems3;
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const u32 job = blockIdx.x;
    if (ahead && threadIdx.x < 32 && job + ahead < gridDim.x) io.prefetch(job + ahead);
    const int prime = io.prime(job);
    const u64 q = dp->pr[prime].q;
    const u64* w = cx.tw + (size_t)prime * 4 * N;
    fill_tw_cache_async(cache, pairs(w + 2 * N), 0, 0, kTwCache3);
    load_first_stage_fn<LB, kElems3>(sm, [&](int i) { return io.load2(dp, job, (u32)i); }, pairs(w + 2 * N), q, logN, 0);
    cp_async_wait_all();
    __syncthreads();
    inv_round<LB, 1, LB - 9, false, kElems3>(sm, cache, pairs(w + 2 * N), q, logN, 0);
    __syncthreads();
    inv_round<LB, LB - 8, 4, true, kElems3>(sm, cache, pairs(w + 2 * N), q, logN, 0);
    __syncthreads();
    inv_round<LB, LB - 4, 4, true, kElems3>(sm, cache, pairs(w + 2 * N), q, logN, 0);
    __syncthreads();
    const int p0 = pad(2 * (int)threadIdx.x);
#pragma unroll 4
    for (int j = 0; j < NB / 2 / T; ++j) {  // values in [0, 4q): io.store takes any 64-bit input
        const int p = p0 + padc(2 * j * T);
        io.store(dp, job, (u32)(threadIdx.x + j * T), sm[p], sm[p + 1]);
    }
}

// ModDown conversion fused behind the INTT of acc's P limb (K = 1, so P/p = 1):
// job = (item, component c);  V[item][c][i] = ecoef[c][i] - P^-1 centred(N^-1 * INTT_p)
// -- k_moddown_conv's output, from the unscaled INTT (N^-1 folded into phat_inv_n).
template <u32 kL>  // the Q limb count, compile-time so the conversion loop unrolls
struct MdConvIO {
    static constexpr u32 L = kL;
    u64* const* acc;           // per item [2][R][N]; the P limb in the NTT domain
    const u64* const* ecoef;   // per item [2][L][N] coefficient-domain addend, or null
    u64* V;                    // [n][2][L][N]
    u32 R, N;
    __device__ int prime(u32) const { return (int)L; }
    __device__ void prefetch(u32 job) const {
        pf_l2(acc[job >> 1] + ((size_t)(job & 1) * R + L) * N, N * 8);
        if (ecoef && pf_mode == 1) pf_l2(ecoef[job >> 1] + (size_t)(job & 1) * L * N, L * N * 8);
    }
    __device__ ulonglong2 load2(const DevParams*, u32 job, u32 i) const {
        return __ldcs(reinterpret_cast<const ulonglong2*>(acc[job >> 1] + ((size_t)(job & 1) * R + L) * N) + i);
    }
    __device__ void store(const DevParams* dp, u32 job, u32 i2, u64 v0, u64 v1) const {
        const u32 item = job >> 1, c = job & 1;
        const u64 p = dp->pr[L].q;
        const u64 z0 = shoup_mul(v0, dp->phat_inv_n[0], dp->phat_inv_n_sh[0], p);
        const u64 z1 = shoup_mul(v1, dp->phat_inv_n[0], dp->phat_inv_n_sh[0], p);
        const u64* ec = ecoef ? ecoef[item] + (size_t)c * L * N : nullptr;
        u64* out = V + ((size_t)item * 2 + c) * L * N;
        // K = 1, so P = p: P^-1 centred(z) = P^-1 z - [z > (p-1)/2] (mod q_i), and
        // V = e - P^-1 centred(z) = e + 3q - lazy(P^-1 z) + [z > (p-1)/2], which lies
        // in [0, 4q) (the lazy product is never 0 for 0 < z < q_i) -- the same
        // canonical residue as reducing the centred lift first.
        const u64 h0 = z0 > (p - 1) / 2, h1 = z1 > (p - 1) / 2;
#pragma unroll
        for (u32 i = 0; i < L; ++i) {
            const u64 q = dp->pr[i].q, pi = dp->P_inv_q[i], pis = dp->P_inv_q_sh[i];
            const u64 q2 = q << 1, q3 = 3 * q;
            ulonglong2 b{0, 0};
            if (ec) b = __ldcs(reinterpret_cast<const ulonglong2*>(ec + (size_t)i * N) + i2);
            ulonglong2 v;
            v.x = reduce_once(reduce_once(b.x + h0 + q3 - shoup_lazy3(z0, pi, pis, q), q2), q);
            v.y = reduce_once(reduce_once(b.y + h1 + q3 - shoup_lazy3(z1, pi, pis, q), q2), q);
            reinterpret_cast<ulonglong2*>(out + (size_t)i * N)[i2] = v;
        }
    }
};

// The BFV tensor product fused into the INTT that brings it back to the
// coefficient domain: job = (item, component p, limb d of Q ++ B); the INTT
// input pair is computed from the NTT-domain operands (Q limbs of a, b; B limbs
// of their extension XB) and the output, N * INTT in [0, 4q), is stored to
// T[item][p][d] (k_scale_round's input, kLazyOut).
template <int S>
struct TensorIO {
    const u64* const* A;
    const u64* const* B;
    const u64* XB;  // [n][4][nB][N]: a.c0, a.c1, b.c0, b.c1 over B
    u64* T;         // [n][3][D][N]
    u32 L, K, nB, D, N;
    __device__ void prefetch(u32) const {}
    __device__ int prime(u32 job) const {
        const u32 d = job % D;
        return (int)(d < L ? d : L + K + (d - L));
    }
    __device__ ulonglong2 load2(const DevParams* dp, u32 job, u32 i) const {
        const u32 item = job / (3 * D), p = (job / D) % 3, d = job % D;
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
        const Prime& P = dp->pr[d < L ? d : L + K + (d - L)];
        Cols s0, s1;
        if (p == 0) {
            const ulonglong2 x = a0[i], y = b0[i];
            s0.mac(split<S>(x.x), split<S>(y.x));
            s1.mac(split<S>(x.y), split<S>(y.y));
        } else if (p == 2) {
            const ulonglong2 x = a1[i], y = b1[i];
            s0.mac(split<S>(x.x), split<S>(y.x));
            s1.mac(split<S>(x.y), split<S>(y.y));
        } else {
            const ulonglong2 x0 = a0[i], x1 = a1[i], y0 = b0[i], y1 = b1[i];
            s0.mac(split<S>(x0.x), split<S>(y1.x));
            s0.mac(split<S>(x1.x), split<S>(y0.x));
            s1.mac(split<S>(x0.y), split<S>(y1.y));
            s1.mac(split<S>(x1.y), split<S>(y0.y));
        }
        return make_ulonglong2(reduce_acc(s0.fold<S>(), P), reduce_acc(s1.fold<S>(), P));
    }
    __device__ void store(const DevParams*, u32 job, u32 i, u64 v0, u64 v1) const {
        __stcs(reinterpret_cast<ulonglong2*>(T + (size_t)job * N) + i, make_ulonglong2(v0, v1));
    }
};

template <typename IO>
void launch_inv_io(const DevCtx& cx, const DevParams& hp, const IO& io, u32 jobs, cudaStream_t s) {
    if (jobs == 0) return;
    if (hp.logN == 13) {
        const size_t smem = (smem_words<13>() + 2 * kTwCache3) * sizeof(u64);
        static std::once_flag once13[64];
        once_per_device(once13, [&] {
            cudaFuncSetAttribute(k_ntt_inv_io<13, IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        });
        k_ntt_inv_io<13, IO><<<jobs, (1 << 13) / kElems3, smem, s>>>(cx, io, io_ahead());
    } else {
        const size_t smem = (smem_words<12>() + 2 * kTwCache3) * sizeof(u64);
        static std::once_flag once12[64];
        once_per_device(once12, [&] {
            cudaFuncSetAttribute(k_ntt_inv_io<12, IO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        });
        k_ntt_inv_io<12, IO><<<jobs, (1 << 12) / kElems3, smem, s>>>(cx, io, io_ahead());
    }
}

bool ntt_inv2() {
    static const bool on = [] {
        const char* v = std::getenv("HGM_NTT_INV2");
        return v && v[0] == '1';
    }();
    return on;
}

int ntt_elems() {
    static const int e = [] {
        const char* v = std::getenv("HGM_NTT_E");
        const int x = v ? std::atoi(v) : 32;
        return x == 16 || x == 322 ? x : 32;
    }();
    return e;
}

// L2 prefetch one wave ahead in the block kernels (HGM_NTT_PF=0 disables)
bool ntt_l2_prefetch() {
    static const bool on = [] {
        const char* v = std::getenv("HGM_NTT_PF");
        return !(v && v[0] == '0');
    }();
    return on;
}

template <int LB, int E, int MINB>
void launch_block_e(bool fwd, const DevCtx& cx, const NttJobs& jobs, int sub, cudaStream_t s) {
    const size_t smem = (smem_words<LB>() + 2 * kTwCache3) * sizeof(u64);
    static std::once_flag once[64];
    once_per_device(once, [&] {
        cudaFuncSetAttribute(k_ntt_fwd3<LB, E, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_ntt_inv3<LB, E, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    const dim3 grid(jobs.count, sub);
    NttJobs j = jobs;
    if (ntt_l2_prefetch()) j.ahead = (u32)(sm_count() * MINB);
    if (fwd)
        k_ntt_fwd3<LB, E, MINB><<<grid, (1 << LB) / E, smem, s>>>(cx, j);
    else
        k_ntt_inv3<LB, E, MINB><<<grid, (1 << LB) / E, smem, s>>>(cx, j);
}

// ---------------------------------------------------------------- N = 2^15: 4-CTA clusters
// One limb of 2^15 residues (256 KiB) crosses HBM once: a cluster of four CTAs
// holds it in their shared memories (one 2^13 quarter each, the same 72 KB image
// as k_ntt_fwd3), and the two outermost stages, which pair elements j, j + N/4,
// j + N/2, j + 3N/4 of different quarters, exchange them through distributed
// shared memory instead of an extra HBM pass.
//
// Forward: CTA r loads columns j in [r N/16, (r+1) N/16) of all four quarters
// straight from HBM (coalesced), applies the two outer stages in registers and
// stores each result into the owning quarter's shared memory (three of the four
// remotely); after a cluster barrier every CTA runs the 13 block stages of its
// quarter (twiddle offset pre = 2, blk = r) and stores it.
// Inverse: every CTA runs the 13 block stages of its quarter (first stage fused
// into its load), then after a cluster barrier CTA r reads its columns of the
// four quarters (three remotely), applies the two outer stages (+ N^-1) and
// writes them to HBM; a final barrier keeps the shared memories alive until
// every remote read is done.
template <int LB>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__((1 << LB) / kElems3, 3)
    k_ntt_fwd_c4(DevCtx cx, NttJobs jobs) {
    namespace cg = cooperative_groups;
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    extern __shared__ u64 sm[];
    u64* cache = sm + smem_words<LB>();
    constexpr int NB = 1 << LB, T = NB / kElems3, COLS = NB / 4;
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const int blk = (int)(blockIdx.x & 3);
    const JobView jv = job_of(jobs, blockIdx.x >> 2, N);
    const u64 q = dp->pr[jv.prime].q;
    const u64* w = cx.tw + (size_t)jv.prime * 4 * N;
#if HGM_LAST_TAB
    __shared__ u64 qtab[16];
    const Canon cn = make_canon(qtab, dp->pr[jv.prime]);
#endif
    fill_tw_cache_async(cache, pairs(w), 2, blk, kTwCache3);
    const ulonglong2* t = pairs(w);
    const u64 w1 = t[1].x, w1s = t[1].y, w2 = t[2].x, w2s = t[2].y, w3 = t[3].x, w3s = t[3].y;
    u32 quarter[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) quarter[r] = dsmem_base(sm, r);
    const u64* a = jobs.src ? jobs.src[blockIdx.x >> 2] : jv.ptr;  // out-of-place: read the source limb
    constexpr int kBatch = 4;  // columns per batch: 16 loads in flight per thread
#pragma unroll 1
    for (int c0 = 0; c0 < COLS / T; c0 += kBatch) {
        u64 x[kBatch][4];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int j = blk * COLS + (c0 + b) * T + (int)threadIdx.x;
#pragma unroll
            for (int k = 0; k < 4; ++k) x[b][k] = __ldcs(a + j + k * NB);
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int j = blk * COLS + (c0 + b) * T + (int)threadIdx.x;
            const int p = pad(j);
#if HGM_C4_LAZY
            // lazy: Shoup products in [0, 3q), differences offset by 3q, no reduction --
            // the quarters receive values below 7q and the block stages start from the
            // bound 8 (kC4B0), which costs them no extra reduction
            const u64 q3 = q + (q << 1);
            u64 V = shoup_lazy3(x[b][2], w1, w1s, q);
            const u64 y0 = x[b][0] + V, y2 = x[b][0] - V + q3;  // < 4q
            V = shoup_lazy3(x[b][3], w1, w1s, q);
            const u64 y1 = x[b][1] + V, y3 = x[b][1] - V + q3;  // < 4q
            V = shoup_lazy3(y1, w2, w2s, q);
            dsmem_st(quarter[0], p, y0 + V);                    // < 7q
            dsmem_st(quarter[1], p, y0 - V + q3);
            V = shoup_lazy3(y3, w3, w3s, q);
            dsmem_st(quarter[2], p, y2 + V);
            dsmem_st(quarter[3], p, y2 - V + q3);
#else
            u64 V = shoup_mul(x[b][2], w1, w1s, q);
            const u64 y0 = add_mod(x[b][0], V, q), y2 = sub_mod(x[b][0], V, q);
            V = shoup_mul(x[b][3], w1, w1s, q);
            const u64 y1 = add_mod(x[b][1], V, q), y3 = sub_mod(x[b][1], V, q);
            V = shoup_mul(y1, w2, w2s, q);
            dsmem_st(quarter[0], p, add_mod(y0, V, q));
            dsmem_st(quarter[1], p, sub_mod(y0, V, q));
            V = shoup_mul(y3, w3, w3s, q);
            dsmem_st(quarter[2], p, add_mod(y2, V, q));
            dsmem_st(quarter[3], p, sub_mod(y2, V, q));
#endif
        }
    }
    cp_async_wait_all();
    cg::this_cluster().sync();  // every quarter complete (and the twiddle caches)
    fwd_round<LB, 0, 4, true, false, NoLoad, kElems3, kC4B0>(sm, cache, pairs(w), q, 2, blk);
    __syncthreads();
    fwd_round<LB, 4, 4, true, false, NoLoad, kElems3, kC4B0>(sm, cache, pairs(w), q, 2, blk);
    __syncthreads();
    fwd_round<LB, 8, LB - 9, false, false, NoLoad, kElems3, kC4B0>(sm, cache, pairs(w), q, 2, blk);
    __syncthreads();
#if HGM_LAST_TAB
    store_last_stage_tab<LB, kElems3, kC4B0>(sm, jv.ptr + ((size_t)blk << LB), pairs(w), q, logN, blk, cn);
#else
    store_last_stage<LB, kElems3>(sm, jv.ptr + ((size_t)blk << LB), pairs(w), q, logN, blk);
#endif
}

template <int LB>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__((1 << LB) / kElems3, 3)
    k_ntt_inv_c4(DevCtx cx, NttJobs jobs) {
    namespace cg = cooperative_groups;
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    extern __shared__ u64 sm[];
    u64* cache = sm + smem_words<LB>();
    constexpr int NB = 1 << LB, T = NB / kElems3, COLS = NB / 4;
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const int blk = (int)(blockIdx.x & 3);
    const JobView jv = job_of(jobs, blockIdx.x >> 2, N);
    const Prime& P = dp->pr[jv.prime];
    const u64 q = P.q;
    const u64* w = cx.tw + (size_t)jv.prime * 4 * N;
    fill_tw_cache_async(cache, pairs(w + 2 * N), logN - LB, blk, kTwCache3);
    const u64* src = jobs.src ? jobs.src[blockIdx.x >> 2] : jv.ptr;  // every read precedes the first write
    load_first_stage<LB, kElems3, 8>(sm, src + ((size_t)blk << LB), pairs(w + 2 * N), q, logN, blk);
    cp_async_wait_all();
    __syncthreads();
    inv_round<LB, 1, LB - 9, false, kElems3>(sm, cache, pairs(w + 2 * N), q, logN, blk);
    __syncthreads();
    inv_round<LB, LB - 8, 4, true, kElems3>(sm, cache, pairs(w + 2 * N), q, logN, blk);
    __syncthreads();
    inv_round<LB, LB - 4, 4, true, kElems3>(sm, cache, pairs(w + 2 * N), q, logN, blk);
    cg::this_cluster().sync();  // all four quarters transformed
    const ulonglong2* t = pairs(w + 2 * N);
    const u64 w1 = t[1].x, w1s = t[1].y, w2 = t[2].x, w2s = t[2].y, w3 = t[3].x, w3s = t[3].y;
    const u32 mode = jobs.unscaled;  // 0: scaled by N^-1, 1: canonical, kLazyOut: [0, 4q)
    u32 quarter[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) quarter[r] = dsmem_base(sm, r);
    u64* a = jv.ptr;
    const u64 q2 = q << 1, q3 = q2 + q, q4 = q << 2, q8 = q << 3;
#ifndef HGM_C4_INV_BATCH
#define HGM_C4_INV_BATCH 2
#endif
    constexpr int kBatch = HGM_C4_INV_BATCH;  // columns (4 remote loads each) in flight per thread
#pragma unroll 1
    for (int c0 = 0; c0 < COLS / T; c0 += kBatch) {
        u64 x[kBatch][4];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int p = pad(blk * COLS + (c0 + b) * T + (int)threadIdx.x);
#pragma unroll
            for (int k = 0; k < 4; ++k) x[b][k] = dsmem_ld(quarter[k], p);  // [0, 4q) (the rounds' bound kGsIn)
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int j = blk * COLS + (c0 + b) * T + (int)threadIdx.x;
            // t = N/4: pairs (0,1) with w[2], (2,3) with w[3]; t = N/2: (0,2), (1,3) with w[1].
            // Lazy: sums grow to 8q and 16q < 2^64, differences are offset by the
            // subtrahend's bound and go straight into the Shoup product ([0, 3q), any
            // 64-bit input); one reduction chain at the end, as short as the output allows.
            const u64 y0 = x[b][0] + x[b][1], y1 = shoup_lazy3(x[b][0] - x[b][1] + q4, w2, w2s, q);
            const u64 y2 = x[b][2] + x[b][3], y3 = shoup_lazy3(x[b][2] - x[b][3] + q4, w3, w3s, q);
            u64 z[4];
            z[0] = y0 + y2;                                    // < 16q
            z[2] = shoup_lazy3(y0 - y2 + q8, w1, w1s, q);      // < 3q
            z[1] = y1 + y3;                                    // < 6q
            z[3] = shoup_lazy3(y1 - y3 + q3, w1, w1s, q);      // < 3q
            if (mode == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) z[k] = shoup_mul(z[k], P.ninv, P.ninv_sh, q);
            } else {
                z[0] = reduce_once(reduce_once(z[0], q8), q4);
                z[1] = reduce_once(z[1], q4);
                if (mode != kLazyOut) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) z[k] = reduce_once(reduce_once(z[k], q2), q);
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) __stcs(a + j + k * NB, z[k]);
        }
    }
    cg::this_cluster().sync();  // keep this CTA's shared memory until every remote read is done
}

bool ntt_cluster4() {
    static const bool on = [] {
        const char* e = std::getenv("HGM_NTT_CLUSTER");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <int LB>
void launch_c4(bool fwd, const DevCtx& cx, const NttJobs& jobs, cudaStream_t s) {
    const size_t smem = (smem_words<LB>() + 2 * kTwCache3) * sizeof(u64);
    static std::once_flag once[64];
    once_per_device(once, [&] {
        cudaFuncSetAttribute(k_ntt_fwd_c4<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_ntt_inv_c4<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    const dim3 grid(jobs.count * 4);
    if (fwd)
        k_ntt_fwd_c4<LB><<<grid, (1 << LB) / kElems3, smem, s>>>(cx, jobs);
    else
        k_ntt_inv_c4<LB><<<grid, (1 << LB) / kElems3, smem, s>>>(cx, jobs);
}

// shared-memory resident block kernels: 256 threads x 32 residues, 3 CTAs/SM
// (default), 512 x 16 at 2 CTAs/SM (HGM_NTT_E=16: spills, -8%), or 256 x 32 at
// 2 CTAs/SM (HGM_NTT_E=322: no spills, forward -4%, inverse +2%)
template <int LB>
void launch_block3(bool fwd, const DevCtx& cx, const NttJobs& jobs, int sub, cudaStream_t s) {
    if (ntt_elems() == 16)
        launch_block_e<LB, 16, 2>(fwd, cx, jobs, sub, s);
    else if (ntt_elems() == 322 || (!fwd && ntt_inv2()))  // 2 CTAs/SM, 128 registers
        launch_block_e<LB, kElems3, 2>(fwd, cx, jobs, sub, s);
    else
        launch_block_e<LB, kElems3, 3>(fwd, cx, jobs, sub, s);
}

bool use_ntt3() {
    static const bool on = [] {
        const char* e = std::getenv("HGM_NTT3");
        return !(e && e[0] == '0');
    }();
    return on;
}

}  // namespace

// The fused variants are exact but measured slower on B200 while the NTT is
// integer-pipe bound (the conversions then compete with the butterflies at
// one CTA per SM); they are opt-in via HGM_FUSED_KS=1 for experiments.
bool ntt_fusable(const DevParams& hp, int which) {
    // HGM_FUSED_KS: "1" both, "u" ModUp only, "d" ModDown only
    static const int mask = [] {
        const char* e = std::getenv("HGM_FUSED_KS");
        if (!e) return 0;
        return e[0] == '1' ? 3 : e[0] == 'u' ? 1 : e[0] == 'd' ? 2 : 0;
    }();
    return (mask & which) && hp.logN <= 13;
}

void ntt_modup_fused(const DevCtx& cx, const DevParams& hp, int n, const u64* C, size_t c_stride, u64* D,
                     cudaStream_t s) {
    ModUpIO io{C, c_stride, D, hp.R, hp.dnum, hp.L, hp.alpha, hp.N};
    launch_fwd_io(cx, hp, io, (u32)n * hp.dnum * hp.R, s);
}

void ntt_moddown_fused(const DevCtx& cx, const DevParams& hp, int n, u64* const* acc, const u64* const* addc,
                       const u64* const* addn, const u32* g, u64* const* out, cudaStream_t s) {
    ModDownIO io{acc, addc, addn, g, out, hp.L, hp.K, hp.R, hp.N, hp.logN};
    launch_fwd_io(cx, hp, io, (u32)n * 2 * hp.L, s);
}

bool ntt_finish_fusable(const DevParams& hp) {
    static const bool on = [] {
        const char* e = std::getenv("HGM_FUSED_FINISH");
        return !e || e[0] != '0';
    }();
    return on && (hp.logN <= 13 || (hp.logN == 15 && ntt_cluster4()));
}

void ntt_finish_fused(const DevCtx& cx, const DevParams& hp, int n, const u64* V, u64* const* acc,
                      const u64* const* addn, const u32* g, u64* const* out, cudaStream_t s, bool prescaled) {
    if (prescaled) {
        FinishIOT<true> io;
        static_cast<ModDownIOT<true>&>(io) = ModDownIOT<true>{acc, nullptr, addn, g, out, hp.L, hp.K, hp.R, hp.N, hp.logN};
        io.V = V;
        launch_fwd_io(cx, hp, io, (u32)n * 2 * hp.L, s);
        return;
    }
    FinishIO io;
    static_cast<ModDownIO&>(io) = ModDownIO{acc, nullptr, addn, g, out, hp.L, hp.K, hp.R, hp.N, hp.logN};
    io.V = V;
    launch_fwd_io(cx, hp, io, (u32)n * 2 * hp.L, s);
}

bool ntt_conv_fusable(const DevParams& hp) {
    static const bool on = [] {
        const char* e = std::getenv("HGM_FUSED_CONV");
        return !e || e[0] != '0';
    }();
    return on && hp.logN <= 13 && hp.K == 1 && hp.L == 3;
}

void ntt_moddown_conv_fused(const DevCtx& cx, const DevParams& hp, int n, u64* const* acc, const u64* const* ecoef,
                            u64* V, cudaStream_t s) {
    if (hp.L != 3) throw std::logic_error("the fused ModDown conversion is built for 3 ciphertext primes");
    MdConvIO<3> io{acc, ecoef, V, hp.R, hp.N};
    launch_inv_io(cx, hp, io, (u32)n * 2, s);
}

bool ntt_tensor_fusable(const DevParams& hp) {
    static const bool on = [] {
        const char* e = std::getenv("HGM_FUSED_TENSOR");
        return e && e[0] == '1';  // opt-in: measured 1% slower than k_tensor + INTT
    }();
    return on && hp.logN <= 13;
}

void ntt_tensor_fused(const DevCtx& cx, const DevParams& hp, int n, const u64* const* A, const u64* const* B,
                      const u64* XB, u64* T, cudaStream_t s) {
    const u32 D = hp.L + hp.nB;
    if (hp.logN == 13 || hp.logN == 12) {
        if (hp.L == 3) {
            TensorIO<30> io{A, B, XB, T, hp.L, hp.K, hp.nB, D, hp.N};
            launch_inv_io(cx, hp, io, (u32)n * 3 * D, s);
        } else {
            TensorIO<28> io{A, B, XB, T, hp.L, hp.K, hp.nB, D, hp.N};
            launch_inv_io(cx, hp, io, (u32)n * 3 * D, s);
        }
    }
}

bool ntt_inverse_takes_first_stage(const DevParams& hp) { return hp.logN == 13 && use_ntt3(); }

bool ntt_out_of_place_ok(const DevParams& hp) { return hp.logN <= 13 || (hp.logN == 15 && ntt_cluster4()); }

void ntt_upload_params(int pid, const DevParams& p) {
    cudaMemcpyToSymbol(c_dp, &p, sizeof(DevParams), (size_t)pid * sizeof(DevParams));
}

namespace {
// Transforms mod the plaintext modulus t = 65537 (encode's INTT and decode's
// NTT: a few polynomials per product, client path).  t is not of the form
// c 2^32 + 1 that the ciphertext kernels' reductions assume (common.cuh
// mul_lo_q), so it has this plain kernel: one CTA per polynomial, residues as
// u32 in shared memory, one radix-2 stage per barrier, products below 2^34
// reduced by the compiler's constant-divisor sequence.  Same definition as the
// ciphertext transforms (natural in / bit-reversed out, inverse scaled by N^-1),
// canonical inputs and outputs.
template <bool kFwd>
__global__ void __launch_bounds__(1024) k_ntt_t(DevCtx cx, NttJobs jobs) {
    const DevParams* __restrict__ dp = &c_dp[cx.pid];
    extern __shared__ u32 st[];
    const u32 N = dp->N, H = N / 2;
    u64* g = jobs.ptrs ? jobs.ptrs[blockIdx.x] : jobs.base + (size_t)blockIdx.x * N;
    const ulonglong2* tw = pairs(cx.tw + (size_t)kTIndex * 4 * N) + (kFwd ? 0 : N);
    for (u32 i = threadIdx.x; i < N; i += blockDim.x) st[i] = (u32)g[i];
    __syncthreads();
    if constexpr (kFwd) {
        for (u32 m = 1, lt = dp->logN - 1; m < N; m <<= 1, --lt) {
            for (u32 b = threadIdx.x; b < H; b += blockDim.x) {
                const u32 i = b >> lt, j = (i << (lt + 1)) + (b & ((1u << lt) - 1)), t = 1u << lt;
                const u32 w = (u32)tw[m + i].x;
                const u32 U = st[j], V = (u32)((u64)st[j + t] * w % kT);
                st[j] = U + V >= (u32)kT ? U + V - (u32)kT : U + V;
                st[j + t] = U >= V ? U - V : U + (u32)kT - V;
            }
            __syncthreads();
        }
    } else {
        for (u32 m = H, lt = 0; m >= 1; m >>= 1, ++lt) {
            for (u32 b = threadIdx.x; b < H; b += blockDim.x) {
                const u32 i = b >> lt, j = (i << (lt + 1)) + (b & ((1u << lt) - 1)), t = 1u << lt;
                const u32 w = (u32)tw[m + i].x;
                const u32 U = st[j], V = st[j + t];
                st[j] = U + V >= (u32)kT ? U + V - (u32)kT : U + V;
                st[j + t] = (u32)((u64)(U >= V ? U - V : U + (u32)kT - V) * w % kT);
            }
            __syncthreads();
        }
    }
    const u64 sc = kFwd ? 1 : dp->pr[kTIndex].ninv;
    for (u32 i = threadIdx.x; i < N; i += blockDim.x) g[i] = kFwd ? st[i] : st[i] * sc % kT;
}
std::once_flag g_ntt_t_attr[2][64];
// true if the batch is a transform mod t (all its jobs: t is never mixed with ciphertext primes)
bool launch_t(bool fwd, const DevCtx& cx, const DevParams& hp, const NttJobs& jobs, cudaStream_t s) {
    bool any = false, all = true;
    for (u32 i = 0; i < jobs.period && i < 32; ++i) {
        const bool t = jobs.prime[i] == kTIndex;
        any |= t;
        all &= t;
    }
    if (!any) return false;
    if (!all || jobs.src || jobs.unscaled || jobs.first_done)
        throw std::logic_error("a transform mod t must be a plain, in-place batch of t jobs only");
    const int smem = (int)(hp.N * sizeof(u32));
    auto k = fwd ? k_ntt_t<true> : k_ntt_t<false>;
    once_per_device(g_ntt_t_attr[fwd], [&] {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4);
    });
    k<<<jobs.count, 1024, smem, s>>>(cx, jobs);
    return true;
}
}  // namespace

void ntt_forward(const DevCtx& cx, const DevParams& hp, const NttJobs& jobs_in, cudaStream_t s) {
    if (jobs_in.count == 0) return;
    if (jobs_in.src && !ntt_out_of_place_ok(hp)) throw std::logic_error("out-of-place NTT needs whole-limb blocks");
    NttJobs jobs = jobs_in;
    jobs.pack();
    if (launch_t(true, cx, hp, jobs, s)) return;
    if (hp.logN == 13 && use_ntt3()) {
        launch_block3<13>(true, cx, jobs, 1, s);
    } else if (hp.logN == 13) {
        launch_block<13>(true, cx, jobs, 1, s);
    } else if (hp.logN == 12) {
        launch_block<12>(true, cx, jobs, 1, s);
    } else if (hp.logN == 15 && ntt_cluster4()) {  // one HBM pass: 4-CTA cluster per limb
        launch_c4<13>(true, cx, jobs, s);
    } else {  // 2^15: two outer stages, then four 2^13 blocks
        k_ntt_fwd_outer2<<<dim3(16, jobs.count), 512, 0, s>>>(cx, jobs);
        if (use_ntt3())
            launch_block3<13>(true, cx, jobs, 4, s);
        else
            launch_block<13>(true, cx, jobs, 4, s);
    }
}

void ntt_inverse(const DevCtx& cx, const DevParams& hp, const NttJobs& jobs_in, cudaStream_t s) {
    if (jobs_in.count == 0) return;
    if (jobs_in.src && !ntt_out_of_place_ok(hp)) throw std::logic_error("out-of-place NTT needs whole-limb blocks");
    NttJobs jobs = jobs_in;
    jobs.pack();
    if (launch_t(false, cx, hp, jobs, s)) return;
    if (hp.logN == 13 && use_ntt3()) {
        launch_block3<13>(false, cx, jobs, 1, s);
    } else if (hp.logN == 13) {
        launch_block<13>(false, cx, jobs, 1, s);
    } else if (hp.logN == 12) {
        launch_block<12>(false, cx, jobs, 1, s);
    } else if (hp.logN == 15 && ntt_cluster4()) {
        launch_c4<13>(false, cx, jobs, s);
    } else {
        if (use_ntt3())
            launch_block3<13>(false, cx, jobs, 4, s);
        else
            launch_block<13>(false, cx, jobs, 4, s);
        k_ntt_inv_outer2<<<dim3(16, jobs.count), 512, 0, s>>>(cx, jobs);
    }
}

}  // namespace hgm
