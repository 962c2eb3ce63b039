# f16 debugging + the epilogue-staged scales: error localisation, A/B, launch lists, ncu of the prep kernels
O=gpurun_out/c4
mkdir -p $O/prof
timeout 600 python tools/f16_debug.py > $O/f16_debug.log 2>&1
for spec in "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048" \
            "CORR 2048,2048" "COVAR 2048,2048" "2MM 4096,4096,4096,4096" "SYRK 4096,4096" "3DCONV 512,512,512" "3DCONV 256,256,256"; do
  set -- $spec
  timeout 300 python tools/ab_time.py $1 $2 stage=2 20 >> $O/ab.log 2>&1
done
for spec in "CORR 2048,2048" "2MM 2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048"; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$1.csv \
      python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
for spec in "CORR 2048,2048 strip_stats_f16" "2MM 2048,2048,2048,2048 f16_split" "2MM 2048,2048,2048,2048 tc_tma2_kernel"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o $O/prof/prof_$1_$3 python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
ls -la $O $O/prof
