# direct 3DCONV v2 (compute-then-refill), DSMEM-batched cluster reduce, CORR/COVAR TMA path
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GEMM or CORR or COVAR or tensor_core" 2>&1 | tail -5
PF_TC_CREDUCE=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GEMM or CORR or COVAR" 2>&1 | tail -2
for m in 0 1 2 3 4 5; do
  echo "3DCONV mode=$m $(PF_C3=$m timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 10 2>&1 | tail -1)"
  PF_C3=$m timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "3DCONV" 2>&1 | tail -1
done
for c in 1 0; do
  echo "GEMM creduce=$c $(PF_TC_CREDUCE=$c timeout 120 python tools/profile_kernels.py GEMM 512,512,512 stage=2 10 2>&1 | tail -1)"
done
for b in CORR COVAR; do echo "$b $(timeout 120 python tools/profile_kernels.py $b 2048,2048 stage=2 10 2>&1 | tail -1)"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py CORR 2048,2048 stage=2 2 2>/dev/null | grep -E "^\"[0-9]" | cut -d, -f5,15 | tail -9
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py GEMM 512,512,512 stage=2 2 2>/dev/null | grep -E "^\"[0-9]" | cut -d, -f5,15 | tail -4
