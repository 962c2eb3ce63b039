# A/B: tcgen05 epilogue (coalesced rows32 vs lane-row, PF_TC_DIAG=16), pair vs single;
# ncu --set full of the pair kernel (2MM) and of 3DCONV stage 2.
set -x
mkdir -p gpurun_out
for b in "2MM 2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048"; do
  set -- $b
  for pair in 1 0; do for d in 0 16 8; do
    echo "$1 pair=$pair diag=$d $(PF_TC_PAIR=$pair PF_TC_DIAG=$d timeout 120 python tools/profile_kernels.py $1 $2 stage=2 10 2>&1 | tail -1)"
  done; done
done
echo "3DCONV s2 $(timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 10 2>&1 | tail -1)"
echo "3DCONV s1 $(timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=1 10 2>&1 | tail -1)"
echo "2DCONV s2 $(timeout 120 python tools/profile_kernels.py 2DCONV 4096,4096 stage=2 10 2>&1 | tail -1)"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_tma2 -s 1 -c 1 \
   -o gpurun_out/prof_2MM_pair python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 3 > gpurun_out/prof_2MM_pair.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv3d_s2 -s 1 -c 1 \
   -o gpurun_out/prof_3DCONV_s2 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 3 > gpurun_out/prof_3DCONV_s2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv2d_s2 -s 1 -c 1 \
   -o gpurun_out/prof_2DCONV_s2 python tools/profile_kernels.py 2DCONV 4096,4096 stage=2 3 > gpurun_out/prof_2DCONV_s2.log 2>&1
ls -la gpurun_out
