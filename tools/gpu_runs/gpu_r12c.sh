# direct-form 3DCONV configurations + split-K cluster reduction (GEMM 512): parity and A/B timings
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GEMM or 2MM or 3MM or SYRK or SYR2K or tensor_core" 2>&1 | tail -5
for m in 0 1 2 3 4 5; do
  echo "3DCONV mode=$m $(PF_C3=$m timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 10 2>&1 | tail -1)"
  PF_C3=$m timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "3DCONV" 2>&1 | tail -1
done
for c in 1 0; do for pair in 1 0; do
  echo "GEMM creduce=$c pair=$pair $(PF_TC_CREDUCE=$c PF_TC_PAIR=$pair timeout 120 python tools/profile_kernels.py GEMM 512,512,512 stage=2 10 2>&1 | tail -1)"
done; done
echo "GEMM 1024 $(timeout 120 python tools/profile_kernels.py GEMM 1024,1024,1024 stage=2 10 2>&1 | tail -1)"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py GEMM 512,512,512 stage=2 3 2>/dev/null | grep -E "tc_|prescale" | cut -d, -f5,9,15 | tail -4
for m in 0 2; do
timeout 300 env PF_C3=$m ncu --set full --clock-control none --import-source on -k regex:conv3d_s2d -s 1 -c 1 \
   -o gpurun_out/prof_3DCONV_s2d_m$m python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 3 > /dev/null 2>&1
done
