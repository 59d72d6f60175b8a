#!/bin/bash
# default staged CSR geometry (one stage per CTA, 256-row tiles, 8 CTAs per SM, carveout left to the driver): full GPU suite, golden printouts, config-2 bench line, ncu capture of one colour launch
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/s4c_pytest_gpu.log 2>&1
tail -n 2 $O/s4c_pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_golden.py -m gpu -x -q -s -p no:cacheprovider -k "c2" > $O/s4c_golden_c2.log 2>&1
grep "c2" $O/s4c_golden_c2.log | cut -c 1-400
timeout 900 python bench.py --workload 2 --steps 3 --warmup 3 > $O/s4c_bench_config2.json 2> $O/s4c_bench_config2.err
python tools/summ.py < $O/s4c_bench_config2.json
CMD2="python bench.py --workload 2 --tsteps 1 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD2 > $O/s4c_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_sweep -s 40 -c 1 -f -o $O/s4c_csr_staged_config2 $CMD2 > $O/s4c_ncu_f2.log 2>&1
tail -n 2 $O/s4c_ncu_f2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/s4c_smoke.log 2>&1; tail -n 2 $O/s4c_smoke.log
