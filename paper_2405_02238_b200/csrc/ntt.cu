// ntt.cu -- see ntt.cuh for the design.
#include "ntt.cuh"

namespace hgm {

namespace {

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }

template <int LB>
constexpr int smem_words() {
    return (1 << LB) + (1 << (LB - 4));
}

// Cooley-Tukey stages [S0, S0+R) of a block of 2^LB residues.  `pre` outer
// stages were already applied (N = 2^(LB+pre)); `blk` is the block's index.
template <int LB, int S0, int R>
__device__ __forceinline__ void fwd_round(u64* sm, const u64* __restrict__ w_tab,
                                          const u64* __restrict__ ws_tab, u64 q, int pre,
                                          int blk) {
    constexpr int NB = 1 << LB, T = NB / 32, G = (NB >> R) / T;
    constexpr int LT_FIRST = LB - 1 - S0, LT_MIN = LT_FIRST - (R - 1);
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
        const int gi = threadIdx.x + gg * T;
        const int o = gi & ((1 << LT_MIN) - 1);
        const int block = gi >> LT_MIN;
        const int base = (block << (LT_FIRST + 1)) + o;
        u64 x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) x[k] = sm[pad(base + (k << LT_MIN))];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int h = 1 << (R - 1 - r);
            const int tw0 = (1 << (pre + S0 + r)) + (blk << (S0 + r)) + (block << r);
#pragma unroll
            for (int c = 0; c < (1 << r); ++c) {
                const u64 w = __ldg(w_tab + tw0 + c), ws = __ldg(ws_tab + tw0 + c);
#pragma unroll
                for (int u = 0; u < h; ++u) {
                    const int k = c * 2 * h + u;
                    const u64 U = x[k];
                    const u64 V = shoup_mul(x[k + h], w, ws, q);
                    x[k] = add_mod(U, V, q);
                    x[k + h] = sub_mod(U, V, q);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) sm[pad(base + (k << LT_MIN))] = x[k];
    }
}

// Gentleman-Sande stages with half-sizes t = 2^LT_LO .. 2^(LT_LO+R-1).
template <int LB, int LT_LO, int R>
__device__ __forceinline__ void inv_round(u64* sm, const u64* __restrict__ w_tab,
                                          const u64* __restrict__ ws_tab, u64 q, int logN,
                                          int blk) {
    constexpr int NB = 1 << LB, T = NB / 32, G = (NB >> R) / T;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
        const int gi = threadIdx.x + gg * T;
        const int o = gi & ((1 << LT_LO) - 1);
        const int block = gi >> LT_LO;
        const int base = (block << (LT_LO + R)) + o;
        u64 x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) x[k] = sm[pad(base + (k << LT_LO))];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int lt = LT_LO + r;
            const int h = 1 << r;
            const int tw0 = (1 << (logN - lt - 1)) + (blk << (LB - lt - 1)) + (block << (R - r - 1));
#pragma unroll
            for (int c = 0; c < (1 << (R - 1 - r)); ++c) {
                const u64 w = __ldg(w_tab + tw0 + c), ws = __ldg(ws_tab + tw0 + c);
#pragma unroll
                for (int u = 0; u < h; ++u) {
                    const int k = c * 2 * h + u;
                    const u64 U = x[k], V = x[k + h];
                    x[k] = add_mod(U, V, q);
                    x[k + h] = shoup_mul(sub_mod(U, V, q), w, ws, q);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << R); ++k) sm[pad(base + (k << LT_LO))] = x[k];
    }
}

struct JobView {
    u64* ptr;
    int prime;
};

__device__ __forceinline__ JobView job_of(const NttJobs& jobs, u32 j, u32 N) {
    JobView v;
    v.ptr = jobs.ptrs ? jobs.ptrs[j] : jobs.base + (size_t)j * N;
    v.prime = jobs.prime[j % jobs.period];
    return v;
}

template <int LB>
__device__ __forceinline__ void load_block(u64* sm, const u64* g) {
    constexpr int NB = 1 << LB, T = NB / 32;
    const ulonglong2* g2 = reinterpret_cast<const ulonglong2*>(g);
#pragma unroll 4
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        const ulonglong2 v = g2[i];
        sm[pad(2 * i)] = v.x;
        sm[pad(2 * i + 1)] = v.y;
    }
}

template <int LB>
__device__ __forceinline__ void store_block(const u64* sm, u64* g) {
    constexpr int NB = 1 << LB, T = NB / 32;
    ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
#pragma unroll 4
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        ulonglong2 v;
        v.x = sm[pad(2 * i)];
        v.y = sm[pad(2 * i + 1)];
        g2[i] = v;
    }
}

template <int LB>
__device__ __forceinline__ void store_block_scaled(const u64* sm, u64* g, u64 s, u64 ssh, u64 q) {
    constexpr int NB = 1 << LB, T = NB / 32;
    ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
#pragma unroll 4
    for (int i = threadIdx.x; i < NB / 2; i += T) {
        ulonglong2 v;
        v.x = shoup_mul(sm[pad(2 * i)], s, ssh, q);
        v.y = shoup_mul(sm[pad(2 * i + 1)], s, ssh, q);
        g2[i] = v;
    }
}

template <int LB>
__global__ void __launch_bounds__((1 << LB) / 32)
    k_ntt_fwd(const DevParams* __restrict__ dp, NttJobs jobs) {
    extern __shared__ u64 sm[];
    const u32 N = dp->N;
    const int pre = (int)dp->logN - LB;
    const int blk = blockIdx.y;
    const JobView jv = job_of(jobs, blockIdx.x, N);
    const u64 q = dp->pr[jv.prime].q;
    const u64* w = dp->tw + (size_t)jv.prime * 4 * N;
    u64* g = jv.ptr + ((size_t)blk << LB);
    load_block<LB>(sm, g);
    __syncthreads();
    fwd_round<LB, 0, 5>(sm, w, w + N, q, pre, blk);
    __syncthreads();
    fwd_round<LB, 5, 4>(sm, w, w + N, q, pre, blk);
    __syncthreads();
    fwd_round<LB, 9, LB - 9>(sm, w, w + N, q, pre, blk);
    __syncthreads();
    store_block<LB>(sm, g);
}

template <int LB>
__global__ void __launch_bounds__((1 << LB) / 32)
    k_ntt_inv(const DevParams* __restrict__ dp, NttJobs jobs) {
    extern __shared__ u64 sm[];
    const u32 N = dp->N;
    const int logN = (int)dp->logN;
    const int blk = blockIdx.y;
    const JobView jv = job_of(jobs, blockIdx.x, N);
    const Prime& P = dp->pr[jv.prime];
    const u64 q = P.q;
    const u64* w = dp->tw + (size_t)jv.prime * 4 * N;
    u64* g = jv.ptr + ((size_t)blk << LB);
    load_block<LB>(sm, g);
    __syncthreads();
    inv_round<LB, 0, LB - 9>(sm, w + 2 * N, w + 3 * N, q, logN, blk);
    __syncthreads();
    inv_round<LB, LB - 9, 4>(sm, w + 2 * N, w + 3 * N, q, logN, blk);
    __syncthreads();
    inv_round<LB, LB - 5, 5>(sm, w + 2 * N, w + 3 * N, q, logN, blk);
    __syncthreads();
    if (logN == LB)
        store_block_scaled<LB>(sm, g, P.ninv, P.ninv_sh, q);
    else
        store_block<LB>(sm, g);
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
    const size_t smem = smem_words<LB>() * sizeof(u64);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_ntt_fwd<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_ntt_inv<LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    dim3 grid(jobs.count, sub);
    if (fwd)
        k_ntt_fwd<LB><<<grid, (1 << LB) / 32, smem, s>>>(dp, jobs);
    else
        k_ntt_inv<LB><<<grid, (1 << LB) / 32, smem, s>>>(dp, jobs);
}

}  // namespace

void ntt_forward(const DevParams* dp, const DevParams& hp, const NttJobs& jobs, cudaStream_t s) {
    if (jobs.count == 0) return;
    if (hp.logN == 13) {
        launch_block<13>(true, dp, jobs, 1, s);
    } else if (hp.logN == 12) {
        launch_block<12>(true, dp, jobs, 1, s);
    } else {  // 2^15: two outer stages, then four 2^13 blocks
        k_ntt_fwd_outer2<<<dim3(16, jobs.count), 512, 0, s>>>(dp, jobs);
        launch_block<13>(true, dp, jobs, 4, s);
    }
}

void ntt_inverse(const DevParams* dp, const DevParams& hp, const NttJobs& jobs, cudaStream_t s) {
    if (jobs.count == 0) return;
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
