# Round-2 evidence pass (one GPU): racecheck detail for GRAMSCHM, ncu --set full
# captures of the chosen variants' dominant kernels (incl. the round-1 gaps
# BICG / MVT / 3MM / COVAR / SYR2K), per-variant launch lists of the dense set,
# and the all-variant report at config sizes.
set -x
O=gpurun_out/ev
mkdir -p $O/prof
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 40 \
    python tools/sanitize_variants.py GRAMSCHM > $O/racecheck_GRAMSCHM.log 2>&1
for spec in "BICG 16384,16384 stage=2 s2_fused 1" "MVT 16384 stage=2 s2_fused 1" \
            "3MM 2048,2048,2048,2048,2048 stage=2 tc_tma2_kernel 3" "COVAR 2048,2048 stage=2 tc_tma2_kernel 1" \
            "SYR2K 2048,2048 stage=2 tc_tma2_kernel 1" "CORR 2048,2048 stage=2 tc_tma2_kernel 1" \
            "2MM 2048,2048,2048,2048 stage=2 tc_tma2_kernel 2" "GEMM 512,512,512 stage=2 tc_tma_kernel 1" \
            "ATAX 16384,16384 stage=2 s2_fused 1" "3DCONV 256,256,256 stage=2 conv3d_s2d 1" "2DCONV 4096,4096 stage=2 conv2d_s2 1"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$4 -s $5 -c $5 \
      -o $O/prof/prof_$1_$4 python tools/profile_kernels.py $1 $2 $3 3 > $O/prof/prof_$1.log 2>&1
done
for spec in "CORR 2048,2048" "COVAR 2048,2048" "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" \
            "SYRK 2048,2048" "SYR2K 2048,2048" "GEMM 512,512,512"; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$1.csv \
      python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
timeout 1500 python tools/variant_report.py --out $O/variant_report.json > $O/variant_report.md 2> $O/variant_report.err
ls -la $O $O/prof
