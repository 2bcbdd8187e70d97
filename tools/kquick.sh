#!/bin/bash
# usage (inside gpurun): tools/kquick.sh <kind> <kernel regex> [pytest -k expr]
# Quick loop for one kernel: parity tests, a clean bench line, then a short ncu metric pass.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -n "$3" ]; then
  timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "$3" > gpurun_out/kq_pytest.log 2>&1
  tail -2 gpurun_out/kq_pytest.log
fi
timeout 400 python bench.py --kind $1 --steps 20 --warmup 5 --e2e-steps 1 --no-cpu > gpurun_out/kq_bench.log 2>&1
tail -1 gpurun_out/kq_bench.log | timeout 10 python tools/bsum.py kq
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum \
  --clock-control none -k regex:"$2" -c 1 python bench.py --kind $1 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/kq_ncu.log 2>&1
grep -E "gpu__time|dram__bytes|fp64|issue_active|registers|wavefronts|inst_executed" gpurun_out/kq_ncu.log | sed 's/  */ /g'
