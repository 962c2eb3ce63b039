# 3DCONV TMA plane streaming + coalesced tcgen05 epilogue: parity, then timing
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stencil or tensor_core or 3DCONV or GEMM or 2MM or SYRK or CORR" 2>&1 | tail -15
timeout 600 python tools/variant_report.py --out gpurun_out/variant_report_r10.json --benches 3DCONV 2DCONV GEMM 2MM 3MM SYRK SYR2K CORR COVAR 2>&1 | tail -12
timeout 900 bash tools/tc_diag.sh 2>&1
for d in 8 14; do echo "pair=1 diag=$d $(PF_TC_DIAG=$d timeout 120 python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 10 2>&1 | tail -1)"; done
