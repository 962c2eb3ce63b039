# Round evidence: GPU tests, smoke, bench (plain + torchrun N=1 + reference arm), variant report, launch list, ncu captures
set -x
mkdir -p gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -10
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; tail -c 600 gpurun_out/bench_torchrun.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 1500 python tools/variant_report.py --out gpurun_out/variant_report.json 2>&1 | tail -17
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --cpu-evals 0 --num-sequences 200 > gpurun_out/bench_under_ncu.log 2>&1
for spec in "ATAX 16384,16384 stage=2 s2_fused" "GESUMMV 16384 stage=2 gesummv_s2" \
            "2MM 2048,2048,2048,2048 stage=2 tc_tma2_kernel" "3DCONV 256,256,256 stage=2 conv3d_s2d" \
            "2DCONV 4096,4096 stage=2 conv2d_s2" "FDTD-2D 2048,2048,24 stage=2 step_rt" "GEMM 512,512,512 stage=2 tc_tma_kernel" \
            "SYRK 2048,2048 stage=2 tc_tma2_kernel" "CORR 2048,2048 stage=2 tc_tma2_kernel"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 \
      -o gpurun_out/prof/prof_$1_$4 python tools/profile_kernels.py $1 $2 $3 3 > gpurun_out/prof/prof_$1.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gs_panel2 -c 1 \
   -o gpurun_out/prof/prof_GRAMSCHM_gs_panel2 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 1 > /dev/null 2>&1
ls -la gpurun_out/prof
