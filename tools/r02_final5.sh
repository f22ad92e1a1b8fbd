# final state: GPU suite, smoke, default bench (N=1)
mkdir -p gpurun_out/final5
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final5/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final5/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/final5/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/final5/bench_n1.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/final5/bench_ref.log 2>&1
