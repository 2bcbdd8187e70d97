#!/bin/bash
# usage (inside gpurun): tools/profile_round.sh [tag]   -- bench lines, launch list and ncu captures for profiles/
# Every ncu run follows a clean run of the same command; nothing timed here is read from a profiled run.
cd "$(dirname "$0")/.."
TAG=${1:-r02}
mkdir -p gpurun_out
for k in srht countsketch gaussian srdct srft cfg0 cfg4; do
  timeout 900 python bench.py --kind $k --steps 20 --warmup 5 --e2e-steps 3 > gpurun_out/bench_${TAG}_$k.log 2>&1
  tail -1 gpurun_out/bench_${TAG}_$k.log | timeout 10 python tools/bsum.py $TAG
done
timeout 600 python tools/tls_parts.py > gpurun_out/tls_parts_${TAG}.txt 2>&1
tail -4 gpurun_out/tls_parts_${TAG}.txt
timeout 600 python tools/svd_parts.py > gpurun_out/svd_parts_${TAG}.txt 2>&1
NSK_SVD_DEBUG=1 timeout 600 python tools/svd_parts.py >> gpurun_out/svd_parts_${TAG}.txt 2>&1
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_reference.log 2>&1
tail -1 gpurun_out/bench_${TAG}_reference.log | cut -c1-300
# launch list of the default bench command (this library's kernels only); ncu only after a clean run
timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/plain_default.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:nsk:: \
  -c 2000 --csv --log-file gpurun_out/launches_${TAG}_default.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu \
  > gpurun_out/ncu_launch.log 2>&1
cap() {  # cap <name> <kernel regex> <command...>
  local name=$1 rx=$2
  shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -c 1 -o gpurun_out/prof_${TAG}_$name \
    "$@" > gpurun_out/ncu_${TAG}_$name.log 2>&1
  echo "ncu $name: $(tail -1 gpurun_out/ncu_${TAG}_$name.log)"
}
cap srht srht_kernel python bench.py --kind srht --steps 1 --warmup 3 --no-cpu --e2e-steps 1
cap countsketch countsketch_owner python bench.py --kind countsketch --steps 1 --warmup 3 --no-cpu --e2e-steps 1
cap gaussian gaussian_sketch python bench.py --kind gaussian --steps 1 --warmup 3 --no-cpu --e2e-steps 1
cap srft srft_ws_kernel python bench.py --kind srft --steps 1 --warmup 3 --no-cpu --e2e-steps 1
cap srdct srdct_stream_kernel python bench.py --kind srdct --steps 1 --warmup 3 --no-cpu --e2e-steps 1
cap cfg4 gaussian_sketch python bench.py --kind cfg4 --steps 1 --warmup 3 --no-cpu --e2e-steps 1
cap svd cluster_svd_kernel python bench.py --kind srht --steps 1 --warmup 3 --no-cpu --e2e-steps 1
cap qr qr_reg_kernel python bench.py --kind srht --steps 1 --warmup 3 --no-cpu --e2e-steps 1
cap general srtt_gen_kernel python tools/srtt_general_time.py
cap shard srtt_fft_kernel python tools/srtt_general_time.py
ls -la gpurun_out/prof_${TAG}_*
