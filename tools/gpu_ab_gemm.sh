# A/B of the cluster split-K contraction (GEMM and the small 2MM/3MM products)
mkdir -p gpurun_out/r3
timeout 600 python -m pytest tests -m gpu -q -x -k "GEMM or 2MM or 3MM or smoke or config" > gpurun_out/r3/tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3/tests.log

for d in 512,512,512 256,256,256 384,384,384 128,128,128; do for sk in 1 0; do PF_TC_SK=$sk timeout 120 python tools/ab_time.py GEMM $d stage=2 30 >> gpurun_out/r3/ab.log 2>&1; done; done
PF_SK_TRACE=1 timeout 120 python tools/sk_trace.py GEMM 512,512,512 2 4 > gpurun_out/r3/sk_trace.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_splitk -s 2 -c 1 -o gpurun_out/r3/prof_GEMM_splitk python tools/profile_kernels.py GEMM 512,512,512 stage=2 3 > /dev/null 2>&1
for sk in 1 0; do PF_TC_SK=$sk timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3/launches_sk$sk.csv python tools/profile_kernels.py GEMM 512,512,512 stage=2 3 > /dev/null 2>&1; done
