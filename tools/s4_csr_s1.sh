#!/bin/bash
# staged CSR sweep: one stage per CTA with 3-4 CTAs per SM (the other CTAs cover a CTA's load; branch values read from the stage after the gathers, 64 registers) vs the default two-stage ring, interleaved A/B on config 2
cd "$(dirname "$0")/.."
bash tools/ab_lib.sh "--workload 2 --steps 3 --warmup 3" 2 libpgb200_csrRef.so libpgb200_csrWl.so libpgb200_csrS1B4.so libpgb200_csrS1B3.so > gpurun_out/s4_csr_s1.txt 2>&1
cat gpurun_out/s4_csr_s1.txt
