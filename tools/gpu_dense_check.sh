# Dense-set check on one GPU: parity (validation / TC tiles / config sizes /
# wide-range 3xFP16 / 3xTF32 subprocess), A/B timings, launch lists.
# usage: bash tools/gpu_dense_check.sh <outdir>
O=${1:-gpurun_out/dense}
mkdir -p $O
PF_PARITY_LOG=$O/parity.jsonl timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_parity.py \
    tests/test_gpu_tc_modes.py -m gpu -q -k "2MM or 3MM or SYRK or SYR2K or CORR or COVAR or GEMM or compare or wide or tf32" \
    > $O/parity.log 2>&1
echo "rc=$?" >> $O/parity.log
for spec in "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048" \
            "CORR 2048,2048" "COVAR 2048,2048" "2MM 4096,4096,4096,4096" "SYRK 4096,4096" "CORR 4096,4096"; do
  set -- $spec
  timeout 300 python tools/ab_time.py $1 $2 stage=2 20 >> $O/ab.log 2>&1
done
for spec in "CORR 2048,2048" "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048"; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$1.csv \
      python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
ls $O
