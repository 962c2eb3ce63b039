# Evidence pass (one GPU): full GPU suite + parity log, smoke, bench
# arms, all-variant report, ncu of the final dense kernels, dense A/B + launch lists.
O=gpurun_out/ev4
mkdir -p $O/prof
PF_PARITY_LOG=$O/parity_all.jsonl timeout 2400 python -m pytest tests -m gpu -q --durations=15 -rs > $O/gputest.log 2>&1
echo "pytest rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
bash tools/gpu_bench_only.sh $O
bash tools/gpu_dense_check.sh $O/dense
for spec in "2MM 2048,2048,2048,2048 tc_tma2_kernel" "2MM 2048,2048,2048,2048 f16_split" "3MM 2048,2048,2048,2048,2048 tc_tma2_kernel"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 2 \
      -o $O/prof/prof_$1_$3 python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
timeout 2400 python tools/variant_report.py --out $O/variant_report.json > $O/variant_report.md 2> $O/variant_report.err
ls -la $O $O/prof
