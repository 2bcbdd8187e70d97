#!/bin/bash
# usage (inside gpurun): tools/bench_all.sh [tag] -- one bench line per BASELINE config + the reference arm
cd "$(dirname "$0")/.."
TAG=${1:-r02}
mkdir -p gpurun_out
for k in srht countsketch gaussian srdct srft cfg0 cfg4; do
  timeout 900 python bench.py --kind $k --steps 20 --warmup 5 --e2e-steps 3 > gpurun_out/bench_${TAG}_$k.log 2>&1
  tail -1 gpurun_out/bench_${TAG}_$k.log | timeout 10 python tools/bsum.py $TAG
done
for k in srht countsketch srdct cfg0 cfg4; do
  timeout 900 python bench.py --impl reference --kind $k --steps 5 --warmup 1 > gpurun_out/bench_${TAG}_reference_$k.log 2>&1
  tail -1 gpurun_out/bench_${TAG}_reference_$k.log | cut -c1-200
done
