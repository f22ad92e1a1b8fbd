mkdir -p gpurun_out/final3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final3/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final3/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final3/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final3/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final3/bench.log
timeout 900 python bench.py --steps 20 --warmup 5 --quick > gpurun_out/final3/bench_quick2.log 2>&1
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k regex:lbm_push_dyn --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/final3/c3_dev_dyn -f python tools/prof_target.py --workload c3 --variant 76 > gpurun_out/final3/ncu_dyn.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/final3/launches.csv python bench.py --steps 2 --warmup 3 --develop 0 --quick > gpurun_out/final3/ncu_launches.log 2>&1
