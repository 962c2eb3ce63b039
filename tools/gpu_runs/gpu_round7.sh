set -x
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
python tools/variant_report.py --out gpurun_out/variant_report_dense.json --benches GEMM 2MM 3MM SYRK SYR2K 2>&1 | tail -7
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.json
ncu --set full --clock-control none --import-source on -k regex:tc_tma_kernel -s 1 -c 1 -o gpurun_out/prof_2MM_tc_tma python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 3 > gpurun_out/prof_tma.log 2>&1
