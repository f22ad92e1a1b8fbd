# the whole GPU suite on a 4-GPU box at the final commit
mkdir -p gpurun_out/final_all4
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_all4/pytest_gpu_4.log 2>&1; echo "rc=$?" >> gpurun_out/final_all4/pytest_gpu_4.log
