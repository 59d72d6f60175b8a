#!/bin/bash
# staged CSR sweep, one stage per CTA: smaller tiles, more CTAs per SM, interleaved A/B on config 2
cd "$(dirname "$0")/.."
bash tools/ab_lib.sh "--workload 2 --steps 3 --warmup 3" 2 libpgb200_csrRef.so libpgb200_csrS1R256B8.so libpgb200_csrS1R128B16.so libpgb200_csrS1R192B10.so libpgb200_csrS1R128B14.so > gpurun_out/s4_csr_s1c.txt 2>&1
cat gpurun_out/s4_csr_s1c.txt
