# GRAMSCHM row-slice panels (PF_GS_W=3), CORR/COVAR 64-tile transposes + 4-deep column sums, GEMM split caps
set -x
PF_GS_W=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GRAMSCHM" 2>&1 | tail -3
for wd in 3 16; do echo "GRAMSCHM W=$wd $(PF_GS_W=$wd timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 5 2>&1 | tail -1)"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "CORR or COVAR" 2>&1 | tail -2
for b in CORR COVAR; do echo "$b $(timeout 120 python tools/profile_kernels.py $b 2048,2048 stage=2 10 2>&1 | tail -1)"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py CORR 2048,2048 stage=2 1 2>/dev/null | python tools/ncu_list.py | tail -8
for sp in 2 4 8; do echo "GEMM split<=$sp $(PF_TC_SPLITS=$sp timeout 120 python tools/profile_kernels.py GEMM 512,512,512 stage=2 10 2>&1 | tail -1)"; done
