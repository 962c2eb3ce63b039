# GRAMSCHM scaling probe: per-panel cost vs rows (m) at n = 2048
set -x
for m in 2048 1024 512 128; do echo "GRAMSCHM m=$m $(timeout 300 python tools/profile_kernels.py GRAMSCHM $m,2048 stage=2,vec=1 3 2>&1 | tail -1)"; done
for n in 1024 512; do echo "GRAMSCHM n=$n $(timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,$n stage=2,vec=1 3 2>&1 | tail -1)"; done
echo "GRAMSCHM v1 m=512 $(PF_GS_PANEL=1 timeout 300 python tools/profile_kernels.py GRAMSCHM 512,2048 stage=2,vec=1 3 2>&1 | tail -1)"
