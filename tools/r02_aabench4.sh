mkdir -p gpurun_out/aabench4
timeout 900 python bench.py --gpus 4 --storage aa > gpurun_out/aabench4/aa_n4.log 2>&1
timeout 900 python bench.py --gpus 4 > gpurun_out/aabench4/two_n4.log 2>&1
timeout 900 python bench.py --gpus 2 --storage aa > gpurun_out/aabench4/aa_n2.log 2>&1
timeout 900 python bench.py --gpus 2 > gpurun_out/aabench4/two_n2.log 2>&1
