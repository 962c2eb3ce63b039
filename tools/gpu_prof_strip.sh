mkdir -p gpurun_out/c12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:f16_split -s 3 -c 1 \
      -o gpurun_out/c12/prof_strip python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 2 > gpurun_out/c12/log.txt 2>&1
