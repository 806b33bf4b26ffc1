#!/bin/bash
# A/B experiment driver (under gpurun): NTT GB/s and bench device value per variant library
bash tools/ntt_variants.sh > gpurun_out/ntt_variants.txt 2>&1
bash tools/bench_variants.sh > gpurun_out/bench_variants.txt 2>&1
cat gpurun_out/ntt_variants.txt gpurun_out/bench_variants.txt
