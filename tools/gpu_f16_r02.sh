# Round-2 pass: 3xFP16 contractions + fused CORR/COVAR statistics (parity,
# A/B timings against 3xTF32 / the two-launch statistics path, launch lists),
# and the stencils at sizes whose output exceeds L2.  Outputs: gpurun_out/f16/
O=gpurun_out/f16
mkdir -p $O
export PF_PARITY_LOG=$O/parity.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_parity.py tests/test_gpu_tc_modes.py -m gpu -q \
    -k "2MM or 3MM or SYRK or SYR2K or CORR or COVAR or GEMM or compare or wide or tf32" > $O/parity.log 2>&1
echo "rc=$?" >> $O/parity.log
for spec in "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048" \
            "CORR 2048,2048" "COVAR 2048,2048" "2MM 4096,4096,4096,4096" "SYRK 4096,4096"; do
  set -- $spec
  for f in 1 0; do PF_TC_F16=$f timeout 300 python tools/ab_time.py $1 $2 stage=2 20 >> $O/ab.log 2>&1; done
done
for spec in "CORR 2048,2048" "COVAR 2048,2048"; do
  set -- $spec
  PF_CC_FUSED=0 PF_TC_F16=0 timeout 300 python tools/ab_time.py $1 $2 stage=2 20 >> $O/ab_unfused.log 2>&1
done
for spec in "CORR 2048,2048" "COVAR 2048,2048" "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" \
            "SYRK 2048,2048" "SYR2K 2048,2048"; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$1.csv \
      python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
timeout 900 python tools/stencil_large.py > $O/stencil_large.jsonl 2> $O/stencil_large.err
ls -la $O
mkdir -p $O/prof
for k in stats_centre_coop sym_scatter tc_tma2_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $O/prof/prof_CORR_$k python tools/profile_kernels.py CORR 2048,2048 stage=2 2 > /dev/null 2>&1
done
for spec in "2MM 2048,2048,2048,2048 tc_tma2_kernel" "SYRK 2048,2048 tc_tma2_kernel" "2MM 2048,2048,2048,2048 f16_split"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o $O/prof/prof_$1_$3 python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
ls -la $O/prof
