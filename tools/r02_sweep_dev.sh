# developed-flow sweep of the bulk push kernel variants (tuning build), C3
mkdir -p gpurun_out/sweep
SPLBCU_LIB=$PWD/paper_2202_11770_b200/libsplbcu_tuning.so timeout 1500 python profiles/sweep_variants.py --workload c3 \
  --variants 43,59,49,56,57,58,47 --pre 3000 --steps 20 > gpurun_out/sweep/dev_c3.jsonl 2>&1
