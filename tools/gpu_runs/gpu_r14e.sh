# GRAMSCHM spread columns + critical column first
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GRAMSCHM" 2>&1 | tail -2
PF_GS_W=8 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GRAMSCHM" 2>&1 | tail -1
for wd in 16 8; do echo "GRAMSCHM W=$wd $(PF_GS_W=$wd timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 5 2>&1 | tail -1)"; done
PF_GS_W=16 timeout 300 python tools/gs_trace.py 2048,2048 2>&1 | tail -17
