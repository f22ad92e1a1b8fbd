mkdir -p gpurun_out/pushw
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "variants or chunked" > gpurun_out/pushw/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pushw/pytest.log
timeout 1500 python profiles/sweep_variants.py --workload c3 --variants 43,74,75,43,75 --pre 3000 --steps 20 > gpurun_out/pushw/dev_c3.jsonl 2>&1
timeout 900 python profiles/sweep_variants.py --workload c2,c4 --variants 43,75 --pre 3000 --steps 20 > gpurun_out/pushw/dev_c2c4.jsonl 2>&1
timeout 600 python profiles/sweep_variants.py --workload c3 --variants 43,75 --steps 20 > gpurun_out/pushw/rest_c3.jsonl 2>&1
