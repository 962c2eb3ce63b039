# CORR/COVAR column statistics strip height
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "CORR or COVAR" 2>&1 | tail -1
for r in 32 16 8; do for b in CORR COVAR; do echo "$b rows=$r $(PF_CC_ROWS=$r timeout 120 python tools/profile_kernels.py $b 2048,2048 stage=2 10 2>&1 | tail -1)"; done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py CORR 2048,2048 stage=2 1 2>/dev/null | python tools/ncu_list.py | tail -8
