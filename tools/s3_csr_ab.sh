#!/bin/bash
# CSR staged sweep: row-pointer bounds of the refill tile loaded one tile ahead (B) vs base (A)
cd "$(dirname "$0")/.."
cp paper_1409_7166_b200/lib/libpgb200_csrB.so paper_1409_7166_b200/lib/libpgb200.so
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "csr or config2 or c2 or fullsize" > gpurun_out/s3_csr_tests.log 2>&1; tail -n 2 gpurun_out/s3_csr_tests.log
bash tools/ab_lib.sh "--workload 2 --steps 3 --warmup 3" 3 libpgb200_csrA.so libpgb200_csrB.so > gpurun_out/s3_csr_ab.txt 2>&1
cat gpurun_out/s3_csr_ab.txt
