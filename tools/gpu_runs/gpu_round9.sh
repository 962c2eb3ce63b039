# clean-L2 flush re-measure (stencils, BLAS-2), tcgen05 bottleneck split, GEMM 512 launch list
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_toolchain.py -q 2>&1 | tail -3
timeout 600 python tools/variant_report.py --out gpurun_out/variant_report_hbm.json --benches 2DCONV 3DCONV ATAX BICG MVT GESUMMV FDTD-2D 2>&1 | tail -10
timeout 900 bash tools/tc_diag.sh 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gemm512_launches.csv \
    python tools/profile_kernels.py GEMM 512,512,512 stage=2 3 > /dev/null 2>&1
grep -v "^==" gpurun_out/gemm512_launches.csv | cut -d, -f5,9,15 | tail -12
