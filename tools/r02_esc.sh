mkdir -p gpurun_out/esc
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py tests/test_bench_geometries.py -m gpu -q -p no:cacheprovider -k "variants or chunked or full_size or online or aa_odd or bench_geom or c3_tree or c4_channel or c5_tree or c2_full" > gpurun_out/esc/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/esc/pytest.log
timeout 1500 python profiles/sweep_variants.py --workload c3 --variants 43,59,71,0 --pre 3000 --steps 20 > gpurun_out/esc/dev_c3.jsonl 2>&1
timeout 600 python profiles/sweep_variants.py --workload c3 --variants 43,59,71 --steps 20 > gpurun_out/esc/rest_c3.jsonl 2>&1
timeout 900 python profiles/sweep_variants.py --workload c2,c4 --variants 43,71 --pre 3000 --steps 20 > gpurun_out/esc/dev_c2c4.jsonl 2>&1
python tools/aa_split.py --workload c3 > gpurun_out/esc/aa_split_c3.json 2>&1
bash tools/r02_dbg.sh
