bash tools/gpu_dense_check.sh gpurun_out/c17
bash tools/gpu_bench_only.sh gpurun_out/c17b
