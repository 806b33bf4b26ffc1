// params.hpp -- BFV parameter sets and their precomputed constants (host side).
#pragma once
#include <string>
#include <vector>

#include "common.cuh"

namespace hgm {

// Parameter sets (BASELINE.json configs):
//   0: N 8192,  Q = 3 x 60-bit, P = 1 x 60-bit, dnum 3, B = 4 x 60-bit  (configs 1-4)
//   1: N 32768, Q = 8 x 55-bit, P = 4 x 55-bit, dnum 2, B = 9 x 55-bit  (config 5)
//   2: N 4096,  as set 0 (a small set for quick parity tests only)
struct ParamSpec {
    unsigned logN, qbits, L, K, dnum, nB;
};
const ParamSpec& param_spec(int id);

struct HostParams {
    ParamSpec spec{};
    int id = 0;
    unsigned N = 0, logN = 0, L = 0, K = 0, nB = 0, dnum = 0, alpha = 0, R = 0;
    u64 seed = 0;
    std::vector<u64> primes;          // Q ++ P ++ B
    std::vector<u64> psi;             // primitive 2N-th roots, same order, then t's
    std::vector<u64> tw;              // [(kMaxPrimes+1)][fwd, inv][N][w, w'] interleaved Shoup pairs
    std::vector<u32> slot_ntt;        // N
    DevParams dev{};                  // scalar part (pointers filled on upload)
};

// Builds the full constant set; throws std::invalid_argument on a bad id.
HostParams make_params(int id, u64 seed);

extern const u64 kGaussCdt[20];

}  // namespace hgm
