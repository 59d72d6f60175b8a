#!/bin/bash
# staged CSR sweep: stage count S (S - 1 tiles in flight ahead of the compute) x tile geometry, interleaved A/B on config 2
cd "$(dirname "$0")/.."
bash tools/ab_lib.sh "--workload 2 --steps 3 --warmup 3" 2 libpgb200_csrS2.so libpgb200_csrR256T256B2S4.so libpgb200_csrR128T128B4S4.so libpgb200_csrR256T128B2S4.so libpgb200_csrR256T256B2S3.so > gpurun_out/s4_csr_stages.txt 2>&1
cat gpurun_out/s4_csr_stages.txt
