# Round-1 session-2 GPU pass: CTA-pair tcgen05 parity first (short timeout),
# then the whole -m gpu suite, smoke, bench, launch list, ncu --set full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k tensor_core 2>&1 | tail -15
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -12
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --cpu-evals 0 > gpurun_out/bench_under_ncu.log 2>&1
for spec in "GESUMMV 16384 stage=2 gesummv_s2" "ATAX 16384,16384 stage=2 s2_fused" \
            "2MM 2048,2048,2048,2048 stage=2 tc_tma"; do
  set -- $spec
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 \
      -o gpurun_out/prof_$1_$4 python tools/profile_kernels.py $1 $2 $3 3 > gpurun_out/prof_$1_$4.log 2>&1
done
timeout 900 python tools/variant_report.py --out gpurun_out/variant_report_dense.json --benches GEMM 2MM 3MM SYRK SYR2K CORR COVAR 2>&1 | tail -12
ls -la gpurun_out
