#!/bin/bash
# fuzzers on HEAD with fresh seeds
cd "$(dirname "$0")/.."
timeout 1500 python tools/fuzz_csr_builder.py 300 4242 > gpurun_out/s4_fuzz_csr_builder.log 2>&1; tail -n 1 gpurun_out/s4_fuzz_csr_builder.log
timeout 1500 python tools/fuzz_sweep.py 300 4242 > gpurun_out/s4_fuzz_sweep.log 2>&1; tail -n 1 gpurun_out/s4_fuzz_sweep.log
