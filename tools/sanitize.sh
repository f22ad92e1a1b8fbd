# compute-sanitizer over small engine runs; logs -> gpurun_out/sanitizer/
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
for c in smoke p2p3 aa3 pull3; do
  for t in memcheck racecheck synccheck; do
    timeout 900 $CS --tool $t --print-limit 30 python tools/sanitize_cases.py $c > gpurun_out/sanitizer/${t}_${c}.log 2>&1
    echo "$t $c rc=$?" >> gpurun_out/sanitizer/summary.txt
  done
done
