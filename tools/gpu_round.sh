#!/bin/bash
# usage: tools/gpu_round.sh "<kinds>" [pytest -k expression]   -- run inside gpurun
cd "$(dirname "$0")/.."
if [ -n "$2" ]; then
  timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "$2" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log
for k in $1; do
  timeout 400 python bench.py --kind $k --steps 20 --warmup 3 --e2e-steps 2 > gpurun_out/bench_$k.log 2>&1
  tail -1 gpurun_out/bench_$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['kind'], 'value=%.4g'%d['value'], 'kernel_ms=', r['kernel_ms'], 'achieved=', r['achieved'], r['unit'], 'frac=', r['frac'], 'svd_ms=', d['breakdown']['svd_ms'], 'e2e=%.4g'%d['e2e']['value'])" 2>&1 | tail -2
done
