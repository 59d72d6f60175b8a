#!/bin/bash
# new default staged CSR geometry (one stage per CTA, 256-row tiles, 8 CTAs per SM): full GPU suite, CSR fuzz, config-2 bench line, ncu capture of one colour launch
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/s4b_pytest_gpu.log 2>&1
tail -n 2 $O/s4b_pytest_gpu.log
timeout 600 python tools/fuzz_csr_builder.py 300 777 > $O/s4b_fuzz_csr_builder.log 2>&1; tail -n 1 $O/s4b_fuzz_csr_builder.log
timeout 900 python bench.py --workload 2 --steps 3 --warmup 3 > $O/s4b_bench_config2.json 2> $O/s4b_bench_config2.err
python tools/summ.py < $O/s4b_bench_config2.json
CMD2="python bench.py --workload 2 --tsteps 1 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD2 > $O/s4b_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_sweep -s 40 -c 1 -f -o $O/s4b_csr_staged_config2 $CMD2 > $O/s4b_ncu_f2.log 2>&1
tail -n 2 $O/s4b_ncu_f2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/s4b_smoke.log 2>&1; tail -n 2 $O/s4b_smoke.log
