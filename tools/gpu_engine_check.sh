mkdir -p gpurun_out/c19
timeout 900 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_e2e.py tests/test_gpu_dropin.py tests/test_gpu_campaign_dist.py -m gpu -q > gpurun_out/c19/tests.log 2>&1; echo "rc=$?" >> gpurun_out/c19/tests.log
bash tools/gpu_bench_only.sh gpurun_out/c19
