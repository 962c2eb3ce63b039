# 3DCONV TMA plane streaming with folded taps vs the direct form
set -x
PF_C3=t timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "3DCONV or stencil" 2>&1 | tail -1
for m in t 0; do echo "3DCONV mode=$m $(PF_C3=$m timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 15 2>&1 | tail -1)"; done
