# round-2 probe: host facts, NCCL two-ranks-on-one-GPU, C3 developed flow at N=1
mkdir -p gpurun_out
{ nproc; free -g; nvidia-smi -L; lscpu | grep -i 'model name'; } > gpurun_out/r02_host.txt 2>&1
cat > /tmp/dup.py <<'PY'
import os, torch, torch.distributed as td
td.init_process_group("nccl", device_id=torch.device("cuda", 0))
t = torch.ones(4, device="cuda:0") * (td.get_rank() + 1)
td.all_reduce(t)
print("rank", td.get_rank(), "allreduce", t.tolist(), flush=True)
td.destroy_process_group()
PY
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 /tmp/dup.py > gpurun_out/r02_nccl_dup.log 2>&1; echo "rc=$?" >> gpurun_out/r02_nccl_dup.log
for v in "" 43 59; do
  for w in 3 3000; do
    SPLBCU_PLAIN_VARIANT=$v timeout 900 python bench.py --warmup $w --steps 50 --quick --no-cpu 2>&1 | grep '^{' | sed "s/^/variant=${v:-default} warmup=$w /" >> gpurun_out/r02_devflow_n1.log
  done
done
