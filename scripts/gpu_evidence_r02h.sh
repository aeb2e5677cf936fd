# Round-2 final evidence run on one B200 (outputs under gpurun_out/ev8/; copied to profiles/ by hand)
set -x
mkdir -p gpurun_out/ev8
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/ev8/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev8/gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/ev8/gputests.log
tail -3 gpurun_out/ev8/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev8/smoke.log 2>&1; echo "smoke $?"
# per-config ncu counters first: the bench lines read profiles/traffic_r02.json
for cfg in c3 c2 c1 c3b1 c4; do
  M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
  timeout 900 ncu --metrics $M --clock-control none -s 80 -c 90 --csv --log-file gpurun_out/ev8/ncu_counters_$cfg.csv \
    python bench.py --config $cfg --steps 4 --warmup 4 --no-cpu --no-extras > gpurun_out/ev8/ncu_counters_$cfg.log 2>&1
  echo "ncu $cfg exit $?"
done
python scripts/ncu_counters.py gpurun_out/ev8/ncu_counters_*.csv > gpurun_out/ev8/traffic_r02.json && cp gpurun_out/ev8/traffic_r02.json profiles/traffic_r02.json
# launch list of the headline command
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev8/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extras > gpurun_out/ev8/ncu_launches.log 2>&1; echo "ncu launches $?"
# bench lines
timeout 900 python bench.py > gpurun_out/ev8/bench_c3.json 2> gpurun_out/ev8/bench_c3.err; echo "bench c3 $?"; tail -c 300 gpurun_out/ev8/bench_c3.json
for cfg in c1 c2 c3b1 c4 c5 views eval; do
  timeout 900 python bench.py --config $cfg > gpurun_out/ev8/bench_$cfg.json 2> gpurun_out/ev8/bench_$cfg.err; echo "bench $cfg $?"
done
timeout 900 python bench.py --config views --views-f32 > gpurun_out/ev8/bench_views_f32.json 2> gpurun_out/ev8/bench_views_f32.err; echo "bench views f32 $?"
timeout 1200 python bench.py --impl reference > gpurun_out/ev8/bench_reference.json 2> gpurun_out/ev8/bench_reference.err; echo "bench ref $?"
# full capture of the two blend kernels, one launch each, source-level
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"blend_forward|blend_backward" -s 6 -c 2 \
  -o gpurun_out/ev8/blend_r02 -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --no-extras > gpurun_out/ev8/ncu_blend.log 2>&1; echo "ncu full $?"
