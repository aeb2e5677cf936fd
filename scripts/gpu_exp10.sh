set -x
GMR_LIB_PATH=$PWD/variants/libgmr_lsort3.so timeout 600 python -m pytest tests -m gpu -x -q -k "parity or edges or stress or configs" > gpurun_out/tests_lsort3.log 2>&1; tail -3 gpurun_out/tests_lsort3.log
bash scripts/compare_variants.sh variants/libgmr_lsort3.so
GMR_LIB_PATH=$PWD/variants/libgmr_lsort3.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:list_depth_sort -s 6 -c 2 -o gpurun_out/lsort3 -f \
  python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --no-extras > gpurun_out/ncu_lsort3.log 2>&1; tail -2 gpurun_out/ncu_lsort3.log
