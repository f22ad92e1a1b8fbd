mkdir -p gpurun_out/final2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final2/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final2/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final2/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final2/bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final2/ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/final2/ref.log
timeout 600 python bench.py --workload c3 --storage aa --steps 20 --warmup 5 --quick > gpurun_out/final2/aa_c3.log 2>&1
