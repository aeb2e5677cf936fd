set -x
bash scripts/compare_variants.sh variants/libgmr_cw.so
GMR_LIB_PATH=$PWD/variants/libgmr_cw.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:blend_ -s 2 -c 2 -o gpurun_out/blend_cw python bench.py --steps 1 --warmup 1 --no-cpu --no-extras > gpurun_out/ncu_blend.log 2>&1; echo ncu $?
