#!/bin/bash
# usage (inside gpurun): tools/profile_round.sh   -- tests, benches, launch list and ncu captures for profiles/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for k in srht countsketch gaussian srdct srft; do
  timeout 600 python bench.py --kind $k --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_$k.log 2>&1
  tail -1 gpurun_out/bench_$k.log | timeout 10 python tools/bsum.py
done
# launch list of the default bench command (this library's kernels only); ncu only after a clean run
timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/plain_default.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:nsk:: \
  -c 2000 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu \
  > gpurun_out/ncu_launch.log 2>&1
cap() {  # cap <name> <kernel regex> <bench args>
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o gpurun_out/prof_$1 \
    python bench.py $3 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_$1.log 2>&1
  echo "ncu $1: $(tail -1 gpurun_out/ncu_$1.log)"
}
cap srht srht_kernel "--kind srht"
cap countsketch countsketch_owner "--kind countsketch"
cap gaussian gaussian_sketch "--kind gaussian"
cap srft srft_ws_kernel "--kind srft"
cap srdct srdct_stream_kernel "--kind srdct"
cap svd cluster_svd_kernel "--kind srht"
