# c3 counters + launch list after the depth-order heuristic change (global sort at config 3)
mkdir -p gpurun_out/ev3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none -s 80 -c 90 --csv --log-file gpurun_out/ev3/ncu_counters_c3.csv \
  python bench.py --config c3 --steps 4 --warmup 4 --no-cpu --no-extras > gpurun_out/ev3/ncu_counters_c3.log 2>&1
echo "ncu c3 $?"
cp gpurun_out/ev2/ncu_counters_c2.csv gpurun_out/ev2/ncu_counters_c1.csv gpurun_out/ev2/ncu_counters_c3b1.csv gpurun_out/ev2/ncu_counters_c4.csv gpurun_out/ev3/ 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev3/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extras > gpurun_out/ev3/ncu_launches.log 2>&1; echo "ncu launches $?"
