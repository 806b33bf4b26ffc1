#!/bin/bash
# host timeline of the end-to-end path (HGM_TRACE=1) for the bench workload
HGM_TRACE=1 python tools/e2e_breakdown.py 4096 2>&1 | tail -30
nproc; lscpu | grep -E "Model name|^CPU\(s\)|MHz" | head -4
