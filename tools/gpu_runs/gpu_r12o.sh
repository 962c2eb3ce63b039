set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GRAMSCHM" 2>&1 | tail -3
echo "GRAMSCHM v5 $(timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 5 2>&1 | tail -1)"
