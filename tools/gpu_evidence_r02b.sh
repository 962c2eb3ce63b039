# Round-2 evidence pass after the 3xFP16 / stencil work (one GPU): full GPU
# suite with per-case parity log, smoke, all-variant report at config sizes,
# bench arms, MMA-only rate of the kind::f16 pipeline, ncu of the dense set.
O=gpurun_out/ev2
mkdir -p $O/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
PF_PARITY_LOG=$O/parity_all.jsonl timeout 2400 python -m pytest tests -m gpu -q --durations=15 -rs > $O/gputest.log 2>&1
echo "pytest rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
PF_TC_DIAG=5 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/mma_only_2MM.csv \
    python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 2 > /dev/null 2>&1
for spec in "2MM 2048,2048,2048,2048 tc_tma2_kernel" "CORR 2048,2048 tc_tma2_kernel" "SYRK 2048,2048 tc_tma2_kernel" \
            "SYR2K 2048,2048 tc_tma2_kernel" "CORR 2048,2048 strip_stats_f16" "2MM 2048,2048,2048,2048 f16_split" \
            "3DCONV 512,512,512 conv3d_s2d" "2DCONV 8192,8192 conv2d_s2"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o $O/prof/prof_$1_$3 python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
timeout 2400 python tools/variant_report.py --out $O/variant_report.json > $O/variant_report.md 2> $O/variant_report.err
ls -la $O $O/prof
