# The bench's N > 1 path on a one-GPU box: 2 and 4 ranks, all on cuda:0 with a
# gloo control plane (PF_DIST_ONE_DEVICE / PF_DIST_BACKEND test hooks).  The
# numbers are not scaling measurements (the ranks share one GPU); the point is
# that every rank runs, the line aggregates over ranks and the sweep shards.
O=gpurun_out/multirank
mkdir -p $O
export PF_DIST_ONE_DEVICE=1 PF_DIST_BACKEND=gloo
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + n)) bench.py --gpus $n --steps 3 --warmup 3 --e2e-steps 1 --sweep-orders 10 \
      > $O/bench_n$n.json 2> $O/bench_n$n.err
  echo "n=$n rc=$?" >> $O/rc.txt
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29610 + n)) bench.py --impl reference --gpus $n --steps 3 --warmup 3 \
      > $O/bench_ref_n$n.json 2> $O/bench_ref_n$n.err
  echo "ref n=$n rc=$?" >> $O/rc.txt
done
