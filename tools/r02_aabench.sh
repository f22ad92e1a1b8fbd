mkdir -p gpurun_out/aabench
timeout 900 python bench.py --storage aa > gpurun_out/aabench/aa_n1.log 2>&1
timeout 900 python bench.py > gpurun_out/aabench/two_n1.log 2>&1
timeout 900 python bench.py --storage aa --no-cpu --no-secondary > gpurun_out/aabench/aa_n1b.log 2>&1
