#!/bin/bash
# staged CSR sweep: the rows' own voltages requested together with the gathers (Vh) vs after them, interleaved A/B on config 2
cd "$(dirname "$0")/.."
bash tools/ab_lib.sh "--workload 2 --steps 3 --warmup 3" 3 libpgb200_csrS2.so libpgb200_csrVh.so libpgb200_csrVhR256T128B4S2.so > gpurun_out/s4_csr_vh.txt 2>&1
cat gpurun_out/s4_csr_vh.txt
