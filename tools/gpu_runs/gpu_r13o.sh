# 3DCONV occupancy (min blocks per SM 6/7/8 via launch bounds)
set -x
for m in 0 6 7 8; do
  PF_C3=$m timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "3DCONV" 2>&1 | tail -1
  echo "3DCONV mode=$m $(PF_C3=$m timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 15 2>&1 | tail -1)"
done
