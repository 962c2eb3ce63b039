# bench arms only (one GPU): our arm, torchrun N=1, reference arm
O=${1:-gpurun_out/bench}
mkdir -p $O
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --sweep-orders 0 > $O/bench_torchrun.json 2> $O/bench_torchrun.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
