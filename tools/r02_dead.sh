mkdir -p gpurun_out/dead
timeout 900 python -m pytest tests/test_dist.py -m gpu -q -p no:cacheprovider -k "dead or nccl" > gpurun_out/dead/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/dead/pytest.log
