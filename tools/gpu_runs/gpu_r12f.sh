# 3DCONV direct configurations, GRAMSCHM register panels v2b, CORR/COVAR pair split-2: parity + timings
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GRAMSCHM or CORR or COVAR or tensor_core" 2>&1 | tail -3
for m in 0 1 2 3 4 5 6; do
  echo "3DCONV mode=$m $(PF_C3=$m timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 10 2>&1 | tail -1)"
done
echo "GRAMSCHM v2 $(timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 5 2>&1 | tail -1)"
for b in CORR COVAR; do echo "$b $(timeout 120 python tools/profile_kernels.py $b 2048,2048 stage=2 10 2>&1 | tail -1)"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py CORR 2048,2048 stage=2 2 2>/dev/null | python tools/ncu_list.py | tail -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gs_panel2 -c 1 \
   -o gpurun_out/prof_GRAMSCHM_panel2 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 1 > /dev/null 2>&1
timeout 300 env PF_C3=0 ncu --set full --clock-control none --import-source on -k regex:conv3d_s2d -s 1 -c 1 \
   -o gpurun_out/prof_3DCONV_s2d_v3 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 3 > /dev/null 2>&1
