# Full validation pass on one B200: GPU tests, smoke, default bench, per-variant report
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -12
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 900 python tools/variant_report.py --out gpurun_out/variant_report.json 2>&1 | tail -30
