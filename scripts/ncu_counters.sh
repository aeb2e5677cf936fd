#!/bin/bash
# Per-kernel ncu counters of a steady-state bench step, for each config:
#   bash scripts/ncu_counters.sh c3 c2 ...   -> gpurun_out/ncu_counters_<cfg>.csv
# then: python scripts/ncu_counters.py gpurun_out/ncu_counters_*.csv > profiles/traffic_r02.json
cd "$(dirname "$0")/.."
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
for cfg in "$@"; do
  timeout 900 ncu --metrics $M --clock-control none -s 80 -c 90 --csv --log-file gpurun_out/ncu_counters_$cfg.csv \
    python bench.py --config $cfg --steps 4 --warmup 4 --no-cpu --no-extras > gpurun_out/ncu_counters_$cfg.log 2>&1
  echo "ncu $cfg exit $?"
done
