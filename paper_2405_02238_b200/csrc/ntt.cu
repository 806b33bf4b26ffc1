// ntt.cu -- see ntt.cuh for the design.
#include "ntt.cuh"

namespace hgm {

namespace {

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }

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
// residues per thread: NB / kElems threads per CTA
constexpr int kElems = 16;

// Cooley-Tukey stage r of an R-stage register round (compile-time bounds so the
// round unrolls and x[] stays in registers).  tw(r, c) yields (w, w') for the
// c-th twiddle of stage r within this group.
template <int R, int r, typename Tw>
__device__ __forceinline__ void fwd_stage(u64 (&x)[1 << R], u64 q, u64 q3, u64 q4, const Tw& tw) {
    constexpr int h = 1 << (R - 1 - r);
#pragma unroll
    for (int c = 0; c < (1 << r); ++c) {
        u64 w, ws;
        tw(r, c, w, ws);
#pragma unroll
        for (int u = 0; u < h; ++u) {
            // Harvey butterfly: values in [0, 4q), U in [0, 2q), V in [0, 2q)
            const int k = c * 2 * h + u;
            const u64 U = reduce_once(x[k], q3);
            const u64 V = shoup_lazy(x[k + h], w, ws, q);
            x[k] = U + V;
            x[k + h] = U - V + q3;
        }
    }
    if constexpr (r + 1 < R) fwd_stage<R, r + 1>(x, q, q3, q4, tw);
}

// Gentleman-Sande stage r (half-size 2^(LT_LO + r)) of an R-stage round.
template <int R, int r, typename Tw>
__device__ __forceinline__ void inv_stage(u64 (&x)[1 << R], u64 q, u64 q4, const Tw& tw) {
    constexpr int h = 1 << r;
#pragma unroll
    for (int c = 0; c < (1 << (R - 1 - r)); ++c) {
        u64 w, ws;
        tw(r, c, w, ws);
#pragma unroll
        for (int u = 0; u < h; ++u) {
            // Harvey butterfly: inputs and outputs in [0, 2q)
            const int k = c * 2 * h + u;
            const u64 U = x[k], V = x[k + h];
            x[k] = reduce_once(U + V, q4);
            x[k + h] = shoup_lazy(U - V + q4, w, ws, q);
        }
    }
    if constexpr (r + 1 < R) inv_stage<R, r + 1>(x, q, q4, tw);
}

// Forward local stages [S0, S0+R): stage s = S0 + r, twiddle
//   2^(pre+s) + (blk << s) + (block << r) + c   (global table index)
//   (1 << s) - 1 + (block << r) + c             (CTA cache index, s < 9)
template <int LB, int S0, int R, bool kCached, bool kFromGlobal = false>
__device__ __forceinline__ void fwd_round(u64* sm, const u64* __restrict__ tw_cache,
                                          const u64* __restrict__ w_tab, const u64* __restrict__ ws_tab,
                                          u64 q, int pre, int blk, const u64* __restrict__ gsrc = nullptr) {
    constexpr int NB = 1 << LB, T = NB / kElems, G = (NB >> R) / T;
    constexpr int LT_FIRST = LB - 1 - S0, LT_MIN = LT_FIRST - (R - 1);
    const u64 q3 = q << 1, q4 = q << 1;  // 2q (Harvey bounds)
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
        const int gi = threadIdx.x + gg * T;
        const int o = gi & ((1 << LT_MIN) - 1);
        const int block = gi >> LT_MIN;
        const int base = (block << (LT_FIRST + 1)) + o;
        u64 x[1 << R];
        if constexpr (kCached) {
            if constexpr (kFromGlobal) {
#pragma unroll
                for (int k = 0; k < (1 << R); ++k) x[k] = __ldcs(gsrc + base + (k << LT_MIN));
            } else {
#pragma unroll
                for (int k = 0; k < (1 << R); ++k) x[k] = sm[pad(base + (k << LT_MIN))];
            }
            auto tw = [&](int r, int c, u64& w, u64& ws) {
                const int i = (1 << (S0 + r)) - 1 + (block << r) + c;
                w = tw_cache[2 * i];
                ws = tw_cache[2 * i + 1];
            };
            fwd_stage<R, 0>(x, q, q3, q4, tw);
        } else {
            u64 pw[(1 << R) - 1], pws[(1 << R) - 1];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int c = 0; c < (1 << r); ++c) {
                    const int g = (1 << (pre + S0 + r)) + (blk << (S0 + r)) + (block << r) + c;
                    pw[(1 << r) - 1 + c] = __ldg(w_tab + g);
                    pws[(1 << r) - 1 + c] = __ldg(ws_tab + g);
                }
#pragma unroll
            for (int k = 0; k < (1 << R); ++k) x[k] = sm[pad(base + (k << LT_MIN))];
            auto tw = [&](int r, int c, u64& w, u64& ws) {
                w = pw[(1 << r) - 1 + c];
                ws = pws[(1 << r) - 1 + c];
            };
            fwd_stage<R, 0>(x, q, q3, q4, tw);
        }
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) sm[pad(base + (k << LT_MIN))] = x[k];
    }
}

// Inverse local stages with half-sizes 2^(LT_LO + r), r < R; twiddle
//   2^(logN-lt-1) + (blk << (LB-lt-1)) + (block << (R-r-1)) + c,  lt = LT_LO + r
//   cache index (1 << (LB-lt-1)) - 1 + (block << (R-r-1)) + c     (LB-lt-1 < 9)
template <int LB, int LT_LO, int R, bool kCached>
__device__ __forceinline__ void inv_round(u64* sm, const u64* __restrict__ tw_cache,
                                          const u64* __restrict__ w_tab, const u64* __restrict__ ws_tab,
                                          u64 q, int logN, int blk) {
    constexpr int NB = 1 << LB, T = NB / kElems, G = (NB >> R) / T;
    const u64 q4 = q << 1;  // 2q (Harvey bounds)
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
        const int gi = threadIdx.x + gg * T;
        const int o = gi & ((1 << LT_LO) - 1);
        const int block = gi >> LT_LO;
        const int base = (block << (LT_LO + R)) + o;
        u64 x[1 << R];
        if constexpr (kCached) {
#pragma unroll
            for (int k = 0; k < (1 << R); ++k) x[k] = sm[pad(base + (k << LT_LO))];
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
                    pw[slot] = __ldg(w_tab + g);
                    pws[slot] = __ldg(ws_tab + g);
                }
#pragma unroll
            for (int k = 0; k < (1 << R); ++k) x[k] = sm[pad(base + (k << LT_LO))];
            auto tw = [&](int r, int c, u64& w, u64& ws) {
                const int slot = (1 << R) - (1 << (R - r)) + c;
                w = pw[slot];
                ws = pws[slot];
            };
            inv_stage<R, 0>(x, q, q4, tw);
        }
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) sm[pad(base + (k << LT_LO))] = x[k];
    }
}

// Fill the CTA twiddle cache: entry (1 << s) - 1 + c, c < 2^s, s < 9, holds the
// global index base(s) + c with base(s) = 2^(outer+s) + (blk << s) (forward:
// outer = pre; inverse: base(s) = 2^(logN-LB+s) + (blk << s) for the stage
// with m-offset 2^s inside the block).
__device__ __forceinline__ void fill_tw_cache(u64* cache, const u64* __restrict__ w_tab,
                                              const u64* __restrict__ ws_tab, int outer, int blk) {
    for (int i = threadIdx.x; i < kTwCache; i += blockDim.x) {
        const int s = 31 - __clz(i + 1);  // i + 1 in [2^s, 2^(s+1))
        const int c = i + 1 - (1 << s);
        const int g = (1 << (outer + s)) + (blk << s) + c;
        cache[2 * i] = __ldg(w_tab + g);
        cache[2 * i + 1] = __ldg(ws_tab + g);
    }
}

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

// Forward: the last Cooley-Tukey stage (t = 1, m = N/2) pairs adjacent
// residues, i.e. exactly the 16-byte vector each thread stores, so it is
// fused into the coalesced store together with the reduction to [0, q).
template <int LB>
__device__ __forceinline__ void store_last_stage(const u64* sm, u64* g, const u64* __restrict__ w_tab,
                                                 const u64* __restrict__ ws_tab, u64 q, int logN, int blk) {
    constexpr int NB = 1 << LB, T = NB / kElems;
    ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
    const int tw0 = (1 << (logN - 1)) + (blk << (LB - 1));
#pragma unroll 4
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        const u64 w = __ldg(w_tab + tw0 + i), ws = __ldg(ws_tab + tw0 + i);
        const u64 q2 = q << 1;
        const u64 U = reduce_once(sm[pad(2 * i)], q2);
        const u64 V = shoup_lazy(sm[pad(2 * i + 1)], w, ws, q);
        ulonglong2 v;
        v.x = reduce_once(reduce_once(U + V, q2), q);
        v.y = reduce_once(reduce_once(U - V + q2, q2), q);
        g2[i] = v;
    }
}

// Inverse: the first Gentleman-Sande stage (t = 1) fused into the coalesced load.
template <int LB>
__device__ __forceinline__ void load_first_stage(u64* sm, const u64* g, const u64* __restrict__ w_tab,
                                                 const u64* __restrict__ ws_tab, u64 q, int logN, int blk) {
    constexpr int NB = 1 << LB, T = NB / kElems;
    const ulonglong2* g2 = reinterpret_cast<const ulonglong2*>(g);
    const int tw0 = (1 << (logN - 1)) + (blk << (LB - 1));
#pragma unroll 4
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        const ulonglong2 v = g2[i];
        const u64 w = __ldg(w_tab + tw0 + i), ws = __ldg(ws_tab + tw0 + i);
        sm[pad(2 * i)] = reduce_once(v.x + v.y, q << 1);
        sm[pad(2 * i + 1)] = shoup_lazy(v.x - v.y + (q << 1), w, ws, q);
    }
}

template <int LB>
__device__ __forceinline__ void load_block(u64* sm, const u64* g) {
    constexpr int NB = 1 << LB, T = NB / kElems;
    const ulonglong2* g2 = reinterpret_cast<const ulonglong2*>(g);
#pragma unroll 4
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        const ulonglong2 v = g2[i];
        sm[pad(2 * i)] = v.x;
        sm[pad(2 * i + 1)] = v.y;
    }
}

// stores canonical residues from smem values in [0, 2q), optionally scaled
template <int LB, bool kScale>
__device__ __forceinline__ void store_block(const u64* sm, u64* g, u64 q, u64 s, u64 ssh) {
    constexpr int NB = 1 << LB, T = NB / kElems;
    ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
#pragma unroll 4
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        ulonglong2 v;
        if constexpr (kScale) {
            v.x = shoup_mul(sm[pad(2 * i)], s, ssh, q);
            v.y = shoup_mul(sm[pad(2 * i + 1)], s, ssh, q);
        } else {
            v.x = reduce_once(sm[pad(2 * i)], q);
            v.y = reduce_once(sm[pad(2 * i + 1)], q);
        }
        g2[i] = v;
    }
}

// Forward block transform: rounds of 4 register stages (local stages 0..LB-2,
// the first eight with CTA-cached twiddles), the last stage fused into the store.
template <int LB>
__global__ void __launch_bounds__((1 << LB) / kElems, 1)
    k_ntt_fwd(const DevParams* __restrict__ dp, NttJobs jobs) {
    extern __shared__ u64 sm[];
    u64* cache = sm + smem_words<LB>();
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const int pre = logN - LB;
    const int blk = blockIdx.y;
    const JobView jv = job_of(jobs, blockIdx.x, N);
    const u64 q = dp->pr[jv.prime].q;
    const u64* w = dp->tw + (size_t)jv.prime * 4 * N;
    u64* g = jv.ptr + ((size_t)blk << LB);
    fill_tw_cache(cache, w, w + N, pre, blk);
    __syncthreads();
    fwd_round<LB, 0, 4, true, true>(sm, cache, w, w + N, q, pre, blk, g);
    __syncthreads();
    fwd_round<LB, 4, 4, true>(sm, cache, w, w + N, q, pre, blk);
    __syncthreads();
    fwd_round<LB, 8, LB - 9, false>(sm, cache, w, w + N, q, pre, blk);
    __syncthreads();
    store_last_stage<LB>(sm, g, w, w + N, q, logN, blk);
}

// Inverse block transform: first stage fused into the load, then rounds of 4
// (the last eight local stages with CTA-cached twiddles); N^-1 folded into the
// store when the block is the whole limb.
template <int LB>
__global__ void __launch_bounds__((1 << LB) / kElems, 1)
    k_ntt_inv(const DevParams* __restrict__ dp, NttJobs jobs) {
    extern __shared__ u64 sm[];
    u64* cache = sm + smem_words<LB>();
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const int blk = blockIdx.y;
    const JobView jv = job_of(jobs, blockIdx.x, N);
    const Prime& P = dp->pr[jv.prime];
    const u64 q = P.q;
    const u64* w = dp->tw + (size_t)jv.prime * 4 * N;
    u64* g = jv.ptr + ((size_t)blk << LB);
    fill_tw_cache(cache, w + 2 * N, w + 3 * N, logN - LB, blk);
    load_first_stage<LB>(sm, g, w + 2 * N, w + 3 * N, q, logN, blk);
    __syncthreads();
    inv_round<LB, 1, LB - 9, false>(sm, cache, w + 2 * N, w + 3 * N, q, logN, blk);
    __syncthreads();
    inv_round<LB, LB - 8, 4, true>(sm, cache, w + 2 * N, w + 3 * N, q, logN, blk);
    __syncthreads();
    inv_round<LB, LB - 4, 4, true>(sm, cache, w + 2 * N, w + 3 * N, q, logN, blk);
    __syncthreads();
    if (logN == LB)
        store_block<LB, true>(sm, g, q, P.ninv, P.ninv_sh);
    else
        store_block<LB, false>(sm, g, q, 0, 0);
}

// Two outermost forward stages for N = 4 * 2^LB: element j, j+N/4, j+N/2, j+3N/4.
__global__ void k_ntt_fwd_outer2(const DevParams* __restrict__ dp, NttJobs jobs) {
    const u32 N = dp->N, Q4 = N / 4;
    const JobView jv = job_of(jobs, blockIdx.y, N);
    const u64 q = dp->pr[jv.prime].q;
    const u64* w = dp->tw + (size_t)jv.prime * 4 * N;
    const u64 w1 = w[1], w1s = w[N + 1], w2 = w[2], w2s = w[N + 2], w3 = w[3], w3s = w[N + 3];
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
__global__ void k_ntt_inv_outer2(const DevParams* __restrict__ dp, NttJobs jobs) {
    const u32 N = dp->N, Q4 = N / 4;
    const JobView jv = job_of(jobs, blockIdx.y, N);
    const Prime& P = dp->pr[jv.prime];
    const u64 q = P.q;
    const u64* w = dp->tw + (size_t)jv.prime * 4 * N + 2 * N;
    const u64* ws = w + N;
    const u64 w2 = w[2], w2s = ws[2], w3 = w[3], w3s = ws[3], w1 = w[1], w1s = ws[1];
    for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < Q4; j += gridDim.x * blockDim.x) {
        u64* a = jv.ptr;
        u64 x0 = a[j], x1 = a[j + Q4], x2 = a[j + 2 * Q4], x3 = a[j + 3 * Q4];
        // t = N/4: pairs (0,1) with m=2 -> w[2], (2,3) with w[3]
        u64 y0 = add_mod(x0, x1, q), y1 = shoup_mul(sub_mod(x0, x1, q), w2, w2s, q);
        u64 y2 = add_mod(x2, x3, q), y3 = shoup_mul(sub_mod(x2, x3, q), w3, w3s, q);
        // t = N/2: pairs (0,2), (1,3) with m=1 -> w[1]
        u64 z0 = add_mod(y0, y2, q), z2 = shoup_mul(sub_mod(y0, y2, q), w1, w1s, q);
        u64 z1 = add_mod(y1, y3, q), z3 = shoup_mul(sub_mod(y1, y3, q), w1, w1s, q);
        a[j] = shoup_mul(z0, P.ninv, P.ninv_sh, q);
        a[j + Q4] = shoup_mul(z1, P.ninv, P.ninv_sh, q);
        a[j + 2 * Q4] = shoup_mul(z2, P.ninv, P.ninv_sh, q);
        a[j + 3 * Q4] = shoup_mul(z3, P.ninv, P.ninv_sh, q);
    }
}

template <int LB>
void launch_block(bool fwd, const DevParams* dp, const NttJobs& jobs, int sub, cudaStream_t s) {
    const size_t smem = (smem_words<LB>() + 2 * kTwCache) * sizeof(u64);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_ntt_fwd<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_ntt_inv<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    dim3 grid(jobs.count, sub);
    if (fwd)
        k_ntt_fwd<LB><<<grid, (1 << LB) / kElems, smem, s>>>(dp, jobs);
    else
        k_ntt_inv<LB><<<grid, (1 << LB) / kElems, smem, s>>>(dp, jobs);
}

}  // namespace

void ntt_forward(const DevParams* dp, const DevParams& hp, const NttJobs& jobs_in, cudaStream_t s) {
    if (jobs_in.count == 0) return;
    NttJobs jobs = jobs_in;
    jobs.pack();
    if (hp.logN == 13) {
        launch_block<13>(true, dp, jobs, 1, s);
    } else if (hp.logN == 12) {
        launch_block<12>(true, dp, jobs, 1, s);
    } else {  // 2^15: two outer stages, then four 2^13 blocks
        k_ntt_fwd_outer2<<<dim3(16, jobs.count), 512, 0, s>>>(dp, jobs);
        launch_block<13>(true, dp, jobs, 4, s);
    }
}

void ntt_inverse(const DevParams* dp, const DevParams& hp, const NttJobs& jobs_in, cudaStream_t s) {
    if (jobs_in.count == 0) return;
    NttJobs jobs = jobs_in;
    jobs.pack();
    if (hp.logN == 13) {
        launch_block<13>(false, dp, jobs, 1, s);
    } else if (hp.logN == 12) {
        launch_block<12>(false, dp, jobs, 1, s);
    } else {
        launch_block<13>(false, dp, jobs, 4, s);
        k_ntt_inv_outer2<<<dim3(16, jobs.count), 512, 0, s>>>(dp, jobs);
    }
}

}  // namespace hgm
