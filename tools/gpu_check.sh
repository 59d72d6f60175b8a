python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1; tail -3 gpurun_out/pytest_gpu2.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; python tools/summ.py < gpurun_out/bench2.json
python -c "import json;d=json.loads(open('gpurun_out/bench2.json').read().strip().splitlines()[-1]);print(d['e2e'], d['detail'])"
