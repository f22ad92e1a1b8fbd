mkdir -p gpurun_out/final4
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final4/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final4/pytest_gpu.log
SPLBCU_LIB=$PWD/paper_2202_11770_b200/libsplbcu_tuning.so timeout 1200 python profiles/sweep_variants.py --workload c3 --variants 76,82,83,84,76 --pre 3000 --steps 20 > gpurun_out/final4/dyn_shapes.jsonl 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final4/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final4/bench.log
