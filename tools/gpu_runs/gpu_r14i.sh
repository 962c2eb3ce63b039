set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "CORR or COVAR or tensor_core or config_paths or SYRK" 2>&1 | tail -1
for b in CORR COVAR SYRK; do echo "$b $(timeout 120 python tools/profile_kernels.py $b 2048,2048 stage=2 10 2>&1 | tail -1)"; done
