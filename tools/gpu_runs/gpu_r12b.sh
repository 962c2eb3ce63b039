# TMA epilogue (tcgen05 contractions) + direct-form 3DCONV stage 2: parity, then A/B timings
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "3DCONV or GEMM or 2MM or 3MM or SYRK or SYR2K or tensor_core or stencil" 2>&1 | tail -15
for m in 0 1 2 3 4; do
  echo "3DCONV mode=$m $(PF_C3=$m timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 10 2>&1 | tail -1)"
  PF_C3=$m timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "3DCONV" 2>&1 | tail -1
done
echo "3DCONV tma $(PF_C3=t timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 10 2>&1 | tail -1)"
for b in "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048" "GEMM 512,512,512"; do
  set -- $b
  for d in 0 32 8; do
    echo "$1 diag=$d $(PF_TC_DIAG=$d timeout 120 python tools/profile_kernels.py $1 $2 stage=2 10 2>&1 | tail -1)"
  done
done
for pair in 1 0; do echo "GEMM pair=$pair $(PF_TC_PAIR=$pair timeout 120 python tools/profile_kernels.py GEMM 512,512,512 stage=2 10 2>&1 | tail -1)"; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv3d_s2d -s 1 -c 1 \
   -o gpurun_out/prof_3DCONV_s2d python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 3 > gpurun_out/prof_3DCONV_s2d.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py GEMM 512,512,512 stage=2 3 2>/dev/null | grep -E "tc_|prescale" | cut -d, -f5,9,15 | tail -4
