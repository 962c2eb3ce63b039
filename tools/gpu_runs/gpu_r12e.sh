# 3DCONV direct fix, GEMM split default, GRAMSCHM register panels: parity + timings + launch lists
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "3DCONV or GEMM or GRAMSCHM or stencil or tensor_core" 2>&1 | tail -5
for m in 0 1 5; do
  echo "3DCONV mode=$m $(PF_C3=$m timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 10 2>&1 | tail -1)"
  PF_C3=$m timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "3DCONV" 2>&1 | tail -3
done
echo "GEMM $(timeout 120 python tools/profile_kernels.py GEMM 512,512,512 stage=2 10 2>&1 | tail -1)"
echo "GRAMSCHM v2 $(timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 5 2>&1 | tail -1)"
echo "GRAMSCHM v1 $(PF_GS_PANEL=1 timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 3 2>&1 | tail -1)"
for spec in "CORR 2048,2048" "GEMM 512,512,512" "SYRK 2048,2048"; do
  set -- $spec
  echo "== launch list $1"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py $1 $2 stage=2 2 2>/dev/null | python tools/ncu_list.py | tail -12
done
