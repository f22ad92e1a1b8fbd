# after the sampler/barrier fix: dist series side stream A/B, N=2, N=1 default line
mkdir -p gpurun_out/side4b
for i in 1 2; do
  timeout 900 python bench.py --gpus 4 > gpurun_out/side4b/side_n4_$i.log 2>&1
  SPLBCU_SERIES_SIDE_OFF=1 timeout 900 python bench.py --gpus 4 --no-cpu > gpurun_out/side4b/off_n4_$i.log 2>&1
done
timeout 900 python bench.py --gpus 2 > gpurun_out/side4b/side_n2.log 2>&1
timeout 900 python bench.py > gpurun_out/side4b/n1.log 2>&1
