set -x
PF_FDTD_TB=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:step_tb -s 2 -c 1 \
   -o gpurun_out/prof_FDTD_tb python tools/profile_kernels.py FDTD-2D 2048,2048,20 stage=2 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gs_panel2 -c 1 \
   -o gpurun_out/prof_GRAMSCHM_v2 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 1 > /dev/null 2>&1
ls gpurun_out
