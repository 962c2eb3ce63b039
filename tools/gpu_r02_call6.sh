bash tools/gpu_dense_check.sh gpurun_out/c6
mkdir -p gpurun_out/c6/prof
for spec in "CORR 2048,2048 colpart" "CORR 2048,2048 centre_split" "2MM 2048,2048,2048,2048 f16_split" "2MM 2048,2048,2048,2048 f16_tsplit"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o gpurun_out/c6/prof/prof_$1_$3 python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
