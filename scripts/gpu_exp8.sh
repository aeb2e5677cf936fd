set -x
bash scripts/compare_variants.sh variants/libgmr_bucket.so
GMR_LIB_PATH=$PWD/variants/libgmr_bucket.so timeout 600 python -m pytest tests -m gpu -x -q -k "parity or edges or configs" > gpurun_out/tests_bucket.log 2>&1; tail -3 gpurun_out/tests_bucket.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bin_depth_sort -s 3 -c 1 -o gpurun_out/depth_sort -f \
  python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --no-extras > gpurun_out/ncu_depth.log 2>&1; tail -2 gpurun_out/ncu_depth.log
