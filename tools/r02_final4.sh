# final check of the AA-default state: GPU suite, smoke, default bench, AA launch list
mkdir -p gpurun_out/final4
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final4/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final4/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/final4/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/final4/bench_n1.log 2>&1
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/final4/c3_dev_aa_launches.csv python tools/prof_target.py --workload c3 --storage aa --steps 2 > gpurun_out/final4/ncu_launches.log 2>&1
