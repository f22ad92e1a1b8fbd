mkdir -p gpurun_out/c2line
timeout 900 python bench.py --workload c2 --steps 50 --warmup 5 > gpurun_out/c2line/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/c2line/bench_c2.log
timeout 900 python bench.py --workload c2 --impl reference --steps 20 --warmup 5 > gpurun_out/c2line/ref_c2.log 2>&1; echo "rc=$?" >> gpurun_out/c2line/ref_c2.log
