mkdir -p gpurun_out/check3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/check3/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/check3/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/check3/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/check3/bench.log
timeout 900 python profiles/sweep_variants.py --workload c2,c4 --variants 0 --pre 3000 --steps 20 > gpurun_out/check3/dev_c2c4_auto.jsonl 2>&1
