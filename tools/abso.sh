#!/bin/bash
# usage (inside gpurun): tools/abso.sh <kind> <so-dir> [kernel regex]  -- bench <kind> with each prebuilt
# libnullsketch_b200.so under <so-dir>/*/ (and, with a regex, that kernel's DRAM bytes from a short ncu pass)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LIB=paper_2206_00975_b200/libnullsketch_b200.so
cp $LIB /tmp/orig.so
for d in $2/*/; do
  v=$(basename $d)
  cp $d/libnullsketch_b200.so $LIB
  timeout 300 python bench.py --kind $1 --steps 20 --warmup 5 --e2e-steps 1 --no-cpu > gpurun_out/abso_$v.log 2>&1
  echo "$v: $(tail -1 gpurun_out/abso_$v.log | timeout 10 python tools/bsum.py)"
  if [ -n "$3" ]; then
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"$3" -c 1 \
      python bench.py --kind $1 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/abso_ncu_$v.log 2>&1
    grep -E "gpu__time|dram__bytes" gpurun_out/abso_ncu_$v.log | sed 's/  */ /g'
  fi
done
cp /tmp/orig.so $LIB
