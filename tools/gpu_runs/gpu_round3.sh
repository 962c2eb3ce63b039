set -x
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
python tools/variant_report.py --out gpurun_out/variant_report.json 2>&1 | tail -17
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
bash tools/gpu_profile.sh > gpurun_out/profile.log 2>&1; tail -5 gpurun_out/profile.log
