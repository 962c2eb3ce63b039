# GRAMSCHM panel-wide q staging, 3DCONV chunk sweep, tcgen05 mainloop diagnostics
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GRAMSCHM or 3DCONV or CORR or COVAR" 2>&1 | tail -3
echo "GRAMSCHM v2 $(timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 5 2>&1 | tail -1)"
for m in 0 1 2 3 4 5 6 7; do
  echo "3DCONV mode=$m $(PF_C3=$m timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 10 2>&1 | tail -1)"
done
for d in 0 1 2 4 8 3 5 6; do
  echo "2MM diag=$d $(PF_TC_DIAG=$d timeout 120 python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 10 2>&1 | tail -1)"
done
for b in CORR COVAR; do echo "$b $(timeout 120 python tools/profile_kernels.py $b 2048,2048 stage=2 10 2>&1 | tail -1)"; done
