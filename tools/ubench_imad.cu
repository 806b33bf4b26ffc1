// Throughput of the integer multiply forms on one SM (cycles per warp
// instruction per SMSP), to cost the modular-arithmetic kernels:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ubench_imad.cu -o /tmp/ub && /tmp/ub
#include <cstdio>
#include <cstdint>

template <int KIND>
__global__ void k(uint32_t* out, uint32_t seed, long long* cyc) {
    uint32_t x[8], y = seed | 1;
    uint64_t acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = seed + i * 7 + threadIdx.x;
        acc[i] = x[i];
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < 4096; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(y));
            if (KIND == 1) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(y));
            if (KIND == 2) {
                uint64_t w = ((uint64_t)x[i] << 32) | x[i];
                asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w) : "r"((uint32_t)(w >> 7)), "r"(y));
                x[i] = (uint32_t)(w >> 32);
            }
            if (KIND == 3) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(y));
            if (KIND == 4) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"((uint32_t)acc[i]), "r"(y));
            if (KIND == 5) asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(x[i]) : "r"(x[i]), "r"(y));
            if (KIND == 6) asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(x[i]) : "r"(x[i]), "r"(y));
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= x[i] ^ (uint32_t)acc[i] ^ (uint32_t)(acc[i] >> 32);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char* name) {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * 4);
    cudaMalloc(&cyc, 8);
    k<KIND><<<1, 1024>>>(out, 12345, cyc);  // 32 warps = 8 per SMSP
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double warp_instr_per_smsp = 4096.0 * 8 * 8;
    printf("%-12s %.2f cycles per warp-instruction per SMSP\n", name, c / warp_instr_per_smsp);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<0>("mul.lo.u32");
    run<1>("mul.hi.u32");
    run<2>("mul.wide.u32");
    run<3>("add.u32");
    run<4>("mad.wide.u32 (acc)");
    run<5>("mad.lo.u32");
    run<6>("mad.hi.u32");
    return 0;
}
