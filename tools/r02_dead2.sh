mkdir -p gpurun_out/dead2
SPLBCU_TRACE=1 timeout 600 python -m pytest tests/test_dist.py -m gpu -q -p no:cacheprovider -k "dead" > gpurun_out/dead2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/dead2/pytest.log
