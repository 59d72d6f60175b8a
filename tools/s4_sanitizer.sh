#!/bin/bash
# compute-sanitizer over the small GPU parity tests (memcheck on the sweep /
# CSR / RHS / builder kernels, then racecheck and synccheck on the two
# staged-pipeline kernels).  Each leg has its own timeout; the summary lines
# go to gpurun_out/s4_sanitizer.txt.
cd "$(dirname "$0")/.."
O=gpurun_out
S=$O/s4_sanitizer.txt
: > $S
leg() {  # name tool timeout pytest-args...
  local name=$1 tool=$2 to=$3; shift 3
  local log=$O/s4_san_${name}.log
  timeout $to compute-sanitizer --tool $tool --error-exitcode 86 --print-limit 20 \
    python -m pytest -m gpu -x -q -p no:cacheprovider "$@" > $log 2>&1
  local rc=$?
  echo "== $name ($tool) rc=$rc: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -n 1) | $(grep -E 'passed|failed|error' $log | tail -n 1)" >> $S
}
leg mem_pipe   memcheck 900 tests/test_gpu_pipe.py
leg mem_store  memcheck 900 tests/test_gpu_store.py
leg mem_parity memcheck 900 tests/test_gpu_parity.py -k "rb_sweep_iterates or fused_sweep or jacobi or rlc or csr_grid or zero_current or device_inputs or errors"
leg mem_tall   memcheck 600 tests/test_gpu_tall.py
leg mem_misc   memcheck 600 tests/test_gpu_continue.py tests/test_gpu_dc_omega.py
leg race_pipe  racecheck 600 tests/test_gpu_pipe.py -k "pipe_equals_fused_and_oracle"
leg race_store racecheck 600 tests/test_gpu_store.py -k "staged_csr or rhs_tiles"
leg sync_pipe  synccheck 600 tests/test_gpu_pipe.py -k "pipe_equals_fused_and_oracle"
leg sync_resident synccheck 600 tests/test_gpu_parity.py -k "rb_sweep_iterates"
cat $S
