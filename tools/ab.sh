#!/bin/bash
# usage (inside gpurun): tools/ab.sh <kind> <ENVVAR> "<values>" -- kernel time of one bench kind per env value
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in $3; do
  env $2=$v timeout 300 python bench.py --kind $1 --steps 20 --warmup 5 --e2e-steps 1 --no-cpu > gpurun_out/ab_$1_$v.log 2>&1
  echo -n "$2=$v "; tail -1 gpurun_out/ab_$1_$v.log | timeout 10 python tools/bsum.py ab
done
