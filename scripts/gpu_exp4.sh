set -x
bash scripts/compare_variants.sh variants/libgmr_f5.so variants/libgmr_f6b320.so
bash scripts/ncu_counters.sh c3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:blend_ -s 8 -c 2 -o gpurun_out/blend_r02a python bench.py --steps 1 --warmup 4 --no-cpu --no-extras > gpurun_out/ncu_blend.log 2>&1; echo ncu $?
