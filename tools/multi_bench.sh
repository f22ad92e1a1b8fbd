set -x
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo rc=$? >> gpurun_out/bench_n$N.log
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --impl reference --steps 3 --warmup 3 > gpurun_out/ref_n4.log 2>&1; echo rc=$? >> gpurun_out/ref_n4.log
