#!/bin/bash
# usage (inside gpurun): tools/svd_sweep.sh "1024 256" "1024 512" ...   -- SVD kernel times per block width
cd "$(dirname "$0")/.."
for sn in "$@"; do
  for b in 2 4 8 16; do
    NSK_SVD_B=$b timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/svdb.csv python tools/svd_one.py $sn > /dev/null 2>&1
    echo "$sn b=$b $(timeout 30 python tools/launches.py gpurun_out/svdb.csv | grep -E 'jacobi|qr_kernel' | tail -2 | awk '{print $NF}' | tr '\n' ' ')"
  done
done
