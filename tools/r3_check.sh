#!/bin/bash
# session check on the checkpointed build: GPU suite + smoke + default bench line
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s3_pytest_gpu.log 2>&1
tail -n 2 gpurun_out/s3_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; tail -n 3 gpurun_out/s3_smoke.log
timeout 600 python bench.py --workload 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/s3_bench_config1.json 2> gpurun_out/s3_bench_config1.err
python tools/summ.py < gpurun_out/s3_bench_config1.json
