# GRAMSCHM mbarrier-suspended factorisation; config-scale tensor-core parity
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GRAMSCHM or config_paths or FDTD" 2>&1 | tail -4
echo "GRAMSCHM v3b $(timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 5 2>&1 | tail -1)"
