# N=4 C3, developed flow (3000 untimed warm-up steps), default vs just-in-time kernel
for v in "" 43 "" 43; do
  SPLBCU_PLAIN_VARIANT=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --warmup 3000 --steps 50 --quick 2>/dev/null | grep '^{' | sed "s/^/variant=${v:-default} /" >> gpurun_out/devflow_n4.log
  SPLBCU_PLAIN_VARIANT=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 4 --warmup 3 --steps 50 --quick 2>/dev/null | grep '^{' | sed "s/^/rest variant=${v:-default} /" >> gpurun_out/devflow_n4.log
done
