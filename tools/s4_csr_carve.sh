#!/bin/bash
# staged CSR sweep (default geometry): preferred shared-memory carveout set to the maximum vs left to the driver
cd "$(dirname "$0")/.."
bash tools/ab_lib.sh "--workload 2 --steps 3 --warmup 3" 3 libpgb200_csrCarve.so libpgb200_csrNoCarve.so > gpurun_out/s4_csr_carve.txt 2>&1
cat gpurun_out/s4_csr_carve.txt
