# final single-GPU session: bench line, its ncu launch list, e2e A/B, pull and AA numbers, C2 run-table capture
mkdir -p gpurun_out/final1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final1/bench.log 2>&1; echo "rc=$?" >> gpurun_out/final1/bench.log
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/final1/launches.csv python bench.py --steps 2 --warmup 3 --develop 0 --quick > gpurun_out/final1/ncu_launches.log 2>&1
timeout 900 python tools/e2e_ab.py --workload c3 --observe 0 > gpurun_out/final1/e2e_c3_noobs.jsonl 2>&1
timeout 900 python tools/e2e_ab.py --workload c3 --observe 1 > gpurun_out/final1/e2e_c3_obs.jsonl 2>&1
timeout 900 python bench.py --workload c2 --scheme pull --steps 20 --warmup 5 --quick > gpurun_out/final1/pull_c2.log 2>&1
timeout 900 python bench.py --workload c3 --scheme pull --steps 10 --warmup 3 --develop 300 --quick > gpurun_out/final1/pull_c3.log 2>&1
timeout 900 python bench.py --workload c3 --storage aa --steps 20 --warmup 5 --quick > gpurun_out/final1/aa_c3.log 2>&1
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k regex:lbm_push_run --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/final1/c2_dev_run -f python tools/prof_target.py --workload c2 --variant 71 > gpurun_out/final1/ncu_c2run.log 2>&1
