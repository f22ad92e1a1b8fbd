# GPU check used during development: tests, N=1 bench, N=2/4 benches, reference arm
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
bash tools/multi_bench.sh
