mkdir -p gpurun_out/sweep2
export SPLBCU_LIB=$PWD/paper_2202_11770_b200/libsplbcu_tuning.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "variants" > gpurun_out/sweep2/pytest_variants.log 2>&1; echo "rc=$?" >> gpurun_out/sweep2/pytest_variants.log
timeout 1500 python profiles/sweep_variants.py --workload c3 --variants 59,67,68,69,70,43 --pre 3000 --steps 20 > gpurun_out/sweep2/dev_c3.jsonl 2>&1
timeout 600 python profiles/sweep_variants.py --workload c3 --variants 69,43 --steps 20 > gpurun_out/sweep2/rest_c3.jsonl 2>&1
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k regex:lbm_push_tmc --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/sweep2/c3_dev_v59 -f python tools/prof_target.py --workload c3 --variant 59 > gpurun_out/sweep2/ncu59.log 2>&1
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k regex:lbm_push_tmc --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/sweep2/c3_dev_v69 -f python tools/prof_target.py --workload c3 --variant 69 > gpurun_out/sweep2/ncu69.log 2>&1
