#!/bin/bash
# last check of HEAD: smoke, store / CSR tests, default bench (config 4)
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/s4d_smoke.log 2>&1; tail -n 2 $O/s4d_smoke.log
timeout 600 python -m pytest tests/test_gpu_store.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $O/s4d_tests.log 2>&1; tail -n 1 $O/s4d_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/s4d_bench_config4.json 2> $O/s4d_bench_config4.err
python tools/summ.py < $O/s4d_bench_config4.json
