# Round-2 evidence pass 3 (one GPU): full GPU suite with parity log, smoke,
# bench arms (incl. torchrun N=1), all-variant report, ncu of the updated
# dense kernels, and the 15-kernel staging campaign on the final kernels.
O=gpurun_out/ev3
mkdir -p $O/prof
PF_PARITY_LOG=$O/parity_all.jsonl timeout 2400 python -m pytest tests -m gpu -q --durations=15 -rs > $O/gputest.log 2>&1
echo "pytest rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
bash tools/gpu_bench_only.sh $O
for spec in "2MM 2048,2048,2048,2048 tc_tma2_kernel" "CORR 2048,2048 tc_tma2_kernel" "CORR 2048,2048 strip_stats_f16" \
            "CORR 2048,2048 sym_scatter" "2MM 2048,2048,2048,2048 f16_split" "SYRK 2048,2048 tc_tma2_kernel"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o $O/prof/prof_$1_$3 python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
timeout 2400 python tools/variant_report.py --out $O/variant_report.json > $O/variant_report.md 2> $O/variant_report.err
timeout 2700 python tools/run_campaign.py --catalog staging --out $O/campaign_staging > $O/campaign_staging.log 2>&1
echo "campaign rc=$?" >> $O/campaign_staging.log
ls -la $O $O/prof
