# uploads overlapped with candidate runs in pf_eval_batch: GPU tests + bench e2e
set -x
timeout 1200 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'e2e', d['e2e']); print(d['per_kernel']['ATAX'])"
