#!/bin/bash
# usage (inside gpurun): tools/bench_all.sh "<kinds>"  -- one bench line per kind into gpurun_out/bench_<kind>.log
cd "$(dirname "$0")/.."
for k in $1; do
  timeout 600 python bench.py --kind $k --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_$k.log 2>&1
  tail -1 gpurun_out/bench_$k.log | timeout 10 python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(k:=d['config']['kind'], 'value=%.4g'%d['value'], 'kernel_ms=', r['kernel_ms'], 'achieved=', r['achieved'], r['unit'], 'frac=', r['frac'], 'svd_ms=', d['breakdown']['svd_ms'], 'e2e_ms=', d['e2e']['ms'], 'cpu=', d['cpu_baseline']['value'])" 2>&1 | tail -1
done
