set -x
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
python tools/variant_report.py --out gpurun_out/variant_report.json --benches 2DCONV 3DCONV 2MM 3MM ATAX BICG CORR COVAR FDTD-2D GEMM GESUMMV MVT SYR2K SYRK 2>&1 | tail -16
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 2500 gpurun_out/bench.json
for spec in "ATAX 16384,16384 stage=2 s2_fused" "MVT 16384 stage=2 s2_fused" "2MM 2048,2048,2048,2048 stage=2 tc_gemm_kernel" \
            "FDTD-2D 2048,2048,20 stage=1 step_fused4" "3DCONV 256,256,256 stage=2 conv3d_s2" "2DCONV 4096,4096 stage=2 conv2d_s2"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 \
      -o gpurun_out/prof_$1_$4 python tools/profile_kernels.py $1 $2 $3 3 > gpurun_out/prof_$1_$4.log 2>&1
done
ls gpurun_out
