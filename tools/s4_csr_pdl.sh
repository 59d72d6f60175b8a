#!/bin/bash
# staged CSR sweep with programmatic dependent launch (option pdl=1) vs without: tests, then interleaved A/B on config 2
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_store.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "csr" > $O/s4_csr_pdl_tests.log 2>&1
tail -n 3 $O/s4_csr_pdl_tests.log
{
for rep in 1 2 3; do
  for o in "--opt pdl=0" "--opt pdl=1"; do
    echo -n "config2 [$o] rep $rep: "; timeout 600 python bench.py --workload 2 --steps 3 --warmup 3 --no-e2e --no-cpu $o 2>/dev/null | python tools/summ.py
  done
done
} > $O/s4_csr_pdl.txt 2>&1
cat $O/s4_csr_pdl.txt
