# Round-2 pass 3: per-row-scaled 3xFP16 (one split launch), column-strip
# CORR/COVAR statistics, 3DCONV chunk-fastest grid; parity, A/B timings,
# launch lists, stencils beyond L2, full GPU suite, bench arms, Table-1 study.
O=gpurun_out/c3
mkdir -p $O
export PF_PARITY_LOG=$O/parity.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_parity.py tests/test_gpu_tc_modes.py -m gpu -q \
    -k "2MM or 3MM or SYRK or SYR2K or CORR or COVAR or GEMM or compare or wide or tf32" > $O/parity.log 2>&1
echo "rc=$?" >> $O/parity.log
unset PF_PARITY_LOG
for spec in "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048" \
            "CORR 2048,2048" "COVAR 2048,2048" "2MM 4096,4096,4096,4096" "SYRK 4096,4096" "GEMM 512,512,512"; do
  set -- $spec
  for f in 1 0; do PF_TC_F16=$f timeout 300 python tools/ab_time.py $1 $2 stage=2 20 >> $O/ab.log 2>&1; done
done
for spec in "CORR 2048,2048" "COVAR 2048,2048" "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" \
            "SYRK 2048,2048" "SYR2K 2048,2048"; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$1.csv \
      python tools/profile_kernels.py $1 $2 stage=2 2 > /dev/null 2>&1
done
timeout 900 python tools/stencil_large.py > $O/stencil_large.jsonl 2> $O/stencil_large.err
PF_C3_ZSLOW=1 timeout 300 python tools/stencil_large.py --stages 2 --cases 3DCONV:256,256,256 3DCONV:512,512,512 \
    > $O/stencil_zslow.jsonl 2>&1
for spec in "2DCONV 8192,8192 conv2d_s2" "3DCONV 512,512,512 conv3d_s2d" "2DCONV 4096,4096 conv2d_s2" "3DCONV 256,256,256 conv3d_s2d"; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:$3 --csv --log-file $O/dram_$1_$2.csv python tools/profile_kernels.py $1 $2 stage=2 3 > /dev/null 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q --durations=15 -rs > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 1200 python tools/run_study.py --kb profiles/r02_campaign_table1/kb.json --out $O/study_table1 > $O/study_table1.log 2>&1
echo "study rc=$?" >> $O/study_table1.log
ls -la $O
