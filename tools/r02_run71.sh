mkdir -p gpurun_out/run71
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -m gpu -q -p no:cacheprovider -k "variants or chunked or full_size or online" > gpurun_out/run71/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/run71/pytest.log
SPLBCU_VERBOSE=1 timeout 1500 python profiles/sweep_variants.py --workload c3 --variants 71,0,71 --pre 3000 --steps 20 > gpurun_out/run71/dev_c3.jsonl 2> gpurun_out/run71/dev_c3.err
timeout 900 python profiles/sweep_variants.py --workload c2,c4 --variants 71,0 --pre 3000 --steps 20 > gpurun_out/run71/dev_c2c4.jsonl 2>&1
timeout 600 python profiles/sweep_variants.py --workload c3 --variants 71,43 --steps 20 > gpurun_out/run71/rest_c3.jsonl 2>&1
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k regex:lbm_push_run --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/run71/c3_dev_v71 -f python tools/prof_target.py --workload c3 --variant 71 > gpurun_out/run71/ncu71.log 2>&1
