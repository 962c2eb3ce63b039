# final state check: GPU tests, smoke, bench
set -x
timeout 1200 python -m pytest tests/ -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'roofline', d['roofline']['frac'], 'clocks', d['clocks'])"
