mkdir -p gpurun_out/check2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/check2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/check2/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/check2/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/check2/bench.log
bash tools/r02_sweep2.sh
