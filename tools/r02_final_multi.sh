# final 4-GPU session: multi-GPU tests, C3 strong scaling, 8-GPU-slab size, C4 weak, C5, P2P edge-kernel ncu
mkdir -p gpurun_out/fmulti
timeout 1500 python -m pytest tests/test_dist.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
  -k "dist or nccl or dead or eight or multi or p2p or store_set" > gpurun_out/fmulti/pytest_multi.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fmulti/pytest_multi.log
for n in 2 4; do
  timeout 900 python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/fmulti/bench_c3_n$n.log 2>&1
done
timeout 900 python bench.py --gpus 4 --steps 50 --warmup 5 --scale 0.5 --quick > gpurun_out/fmulti/bench_c3half_n4.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 50 --warmup 5 --scale 0.5 --quick > gpurun_out/fmulti/bench_c3half_n1.log 2>&1
timeout 1200 python bench.py --gpus 4 --workload c5 --steps 20 --warmup 5 --quick > gpurun_out/fmulti/bench_c5_n4.log 2>&1
for n in 1 2 4; do
  timeout 1200 python bench.py --gpus $n --workload c4w --steps 20 --warmup 5 --develop 1000 --quick > gpurun_out/fmulti/bench_c4w_n$n.log 2>&1
done
/usr/local/cuda/bin/ncu --query-metrics > gpurun_out/fmulti/ncu_metrics.txt 2>&1
NVL=$(grep -oE "^nvl[a-z_]+__bytes" gpurun_out/fmulti/ncu_metrics.txt | sort -u | sed 's/$/.sum/' | paste -sd, -)
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k "regex:lbm_push_tma|lbm_push<" --set full --import-source on \
  --clock-control none -o gpurun_out/fmulti/c3_edge_p2p -f python tools/prof_edge.py c3 1000 > gpurun_out/fmulti/ncu_edge.log 2>&1
if [ -n "$NVL" ]; then
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k "regex:lbm_push_tma" --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,$NVL \
  --clock-control none --csv --log-file gpurun_out/fmulti/c3_edge_p2p_nvl.csv python tools/prof_edge.py c3 1000 > gpurun_out/fmulti/ncu_edge_nvl.log 2>&1
fi
