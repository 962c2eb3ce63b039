set -x
for m in 0 1 2 3 4; do
  PF_C2=$m timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "2DCONV" 2>&1 | tail -1
  echo "2DCONV mode=$m $(PF_C2=$m timeout 120 python tools/profile_kernels.py 2DCONV 4096,4096 stage=2 15 2>&1 | tail -1)"
done
