# C5 on 4 GPUs and C4 on 1 GPU with the current kernels (DESIGN table refresh)
set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --workload c5 --steps 10 > gpurun_out/bench_c5_n4.log 2>&1; echo rc=$? >> gpurun_out/bench_c5_n4.log
timeout 600 python bench.py --workload c4 --steps 20 --no-cpu --no-secondary > gpurun_out/bench_c4.log 2>&1; echo rc=$? >> gpurun_out/bench_c4.log
