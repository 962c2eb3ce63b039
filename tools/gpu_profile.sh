# ncu evidence for profiles/ (never a bench number: ncu serialises and replays)
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --cpu-evals 0 --num-sequences 200 > gpurun_out/bench_under_ncu.log 2>&1
for spec in "ATAX 16384,16384 stage=2 s2_fused" "BICG 16384,16384 stage=2 s2_fused" \
            "GESUMMV 16384 stage=2 gesummv_s2" "2MM 2048,2048,2048,2048 stage=2 tc_gemm_kernel" \
            "3DCONV 256,256,256 stage=1 conv3d_s1" "FDTD-2D 2048,2048,20 stage=1 step_fused"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 \
      -o gpurun_out/prof_$1_$4 python tools/profile_kernels.py $1 $2 $3 3 > gpurun_out/prof_$1_$4.log 2>&1
done
ls -la gpurun_out
