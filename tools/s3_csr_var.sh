#!/bin/bash
# staged CSR sweep geometry variants (rows per tile R, threads T, CTAs per SM B), interleaved
cd "$(dirname "$0")/.."
bash tools/ab_lib.sh "--workload 2 --steps 3 --warmup 3" 2 libpgb200_csrR512T256B2.so libpgb200_csrR256T128B4.so libpgb200_csrR512T512B2.so libpgb200_csrR256T256B4.so > gpurun_out/s3_csr_var.txt 2>&1
cat gpurun_out/s3_csr_var.txt
