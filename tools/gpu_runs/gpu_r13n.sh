# 3DCONV L2 prefetch distance sweep; chained-lo parity cases
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config_paths or 3DCONV or stencil" 2>&1 | tail -2
for d in 0 1 2 3 4 6; do echo "3DCONV l2=$d $(PF_C3_L2=$d timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 15 2>&1 | tail -1)"; done
