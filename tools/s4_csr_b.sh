#!/bin/bash
# staged CSR sweep, one stage per CTA, 256-row tiles: CTAs per SM (shared memory vs L1 for the gathers), interleaved A/B on config 2
cd "$(dirname "$0")/.."
bash tools/ab_lib.sh "--workload 2 --steps 3 --warmup 3" 2 libpgb200_csrB8.so libpgb200_csrB7.so libpgb200_csrB6.so libpgb200_csrR224B9.so > gpurun_out/s4_csr_b.txt 2>&1
cat gpurun_out/s4_csr_b.txt
