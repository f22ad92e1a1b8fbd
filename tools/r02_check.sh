# round-2 check: GPU tests, default bench (developed flow), AA developed
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r02_bench.log
timeout 600 python bench.py --steps 20 --warmup 5 --storage aa --quick > gpurun_out/r02_bench_aa.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_aa.log
